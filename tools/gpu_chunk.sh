#!/bin/bash
# longer TMEM accumulation chunks: kernel times and accuracy
out=gpurun_out/${1:-chunk}; mkdir -p $out
L1=vgg16/conv1_2,vgg16/conv2_1,vgg16/conv2_2
L2=vgg16/conv3_2,vgg16/conv4_2,vgg16/conv5_1,vgg16/conv3_1
for env in "" "CLB_CHUNK=3" "CLB_CHUNK=4" "CLB_CHUNK=6"; do env $env timeout 300 python tools/knob_sweep.py $L1 >> $out/knobs.txt 2>&1; done
for env in "" "CLB_CHUNK=9" "CLB_CHUNK=12" "CLB_CHUNK=18"; do env $env timeout 300 python tools/knob_sweep.py $L2 >> $out/knobs.txt 2>&1; done
for c in 6 12 18 24; do CLB_CHUNK=$c CLB_SPLIT=3xf16 CLB_PADDED_ROWS=0 timeout 300 python tools/acc_conv.py | sed "s/^/chunk=$c /" >> $out/acc.txt 2>&1; done
for c in 2 4 6; do CLB_CHUNK=$c CLB_SPLIT=3xf16 CLB_PADDED_ROWS=1 timeout 300 python tools/acc_conv.py | sed "s/^/padded chunk=$c /" >> $out/acc.txt 2>&1; done
