#!/bin/bash
# knob sweep on the VGG half-K and 14x14 layers (kernel ms, tools/knob_sweep.py)
out=gpurun_out/knobs5; mkdir -p $out
L=vgg16/conv2_1,vgg16/conv3_1,vgg16/conv4_1,vgg16/conv5_1
run() { env "$@" timeout 300 python tools/knob_sweep.py $L >> $out/t.txt 2>&1; }
run CLB_X=0
run CLB_PADDED_ROWS=1
run CLB_PADDED_ROWS=0
run CLB_BN=128
run CLB_BN=128 CLB_PADDED_ROWS=1
run CLB_BPS=1
run CLB_BPS=2
run CLB_CHUNK=2
run CLB_CHUNK=8
run CLB_MSUB=2
run CLB_MSUB=2 CLB_BN=128
run CLB_CTA_GROUP=1
run CLB_X=0
cat $out/t.txt
