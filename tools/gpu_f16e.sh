#!/bin/bash
# accuracy vs K for the three fp32-faithful splits; traces + knob A/B of the layers furthest from peak
out=gpurun_out/${1:-f16e}; mkdir -p $out
for sp in 3xf16 mixed 3xtf32; do CLB_SPLIT=$sp timeout 300 python tools/acc_conv.py >> $out/acc.txt 2>&1; done
for L in vgg16/conv5_1 vgg16/conv1_2 vgg16/conv2_1 vgg16/conv4_1; do
  CLB_TRACE=1 timeout 120 python tools/prof_layer.py --layer $L --reps 1 >> $out/trace.txt 2>&1
done
L=vgg16/conv5_1,vgg16/conv1_2,vgg16/conv2_1,vgg16/conv3_1,vgg16/conv4_1,alexnet/conv3
for env in "" "CLB_CTA_GROUP=1" "CLB_CTA_GROUP=2" "CLB_BN=128" "CLB_PADDED_ROWS=1" "CLB_PADDED_ROWS=0" "CLB_MAX_SPLIT=1" "CLB_BPS=1" "CLB_MSUB=1" "CLB_MSUB=2" "CLB_SPLIT_ISSUE=0"; do
  env $env timeout 300 python tools/knob_sweep.py $L >> $out/knobs.txt 2>&1
done
