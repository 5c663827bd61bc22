#!/bin/bash
# knob A/B of the layers below 0.85 of peak in the VGG step (kernel time, L2 flushed, median of 7)
out=gpurun_out/${1:-knobs}; mkdir -p $out
L=vgg16/conv5_1,vgg16/conv1_2,vgg16/conv2_1,vgg16/conv3_1,vgg16/conv4_1
for env in "" "CLB_CTA_GROUP=1" "CLB_CTA_GROUP=2" "CLB_CTA_GROUP=2 CLB_BN=128" "CLB_CTA_GROUP=1 CLB_BN=128" \
           "CLB_MAX_SPLIT=1" "CLB_MAX_SPLIT=3" "CLB_PADDED_ROWS=1" "CLB_PADDED_ROWS=0" "CLB_BPS=1" "CLB_BPS=3" "CLB_SK_UNITS=0"; do
  env $env timeout 300 python tools/knob_sweep.py $L >> $out/knobs.txt 2>&1
done
