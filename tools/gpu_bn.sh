#!/bin/bash
# tile N in the padded-row mode for the BN = 256 layers
mkdir -p gpurun_out
L=alexnet/conv2,alexnet/conv5,vgg16/conv5_1,vgg16/conv5_2,vgg16/conv4_2,vgg16/conv3_2
{
timeout 200 python tools/knob_sweep.py $L
for bn in 128 192 256; do CLB_PADDED_ROWS=1 CLB_BN=$bn timeout 200 python tools/knob_sweep.py $L; CLB_PADDED_ROWS=0 CLB_BN=$bn timeout 200 python tools/knob_sweep.py $L; done
} > gpurun_out/bn_sweep.txt 2>&1
