#!/bin/bash
# stage buffering: smem budget (CLB_SMEM_KB) x stage grouping (CLB_BPS), kernel times per layer
mkdir -p gpurun_out
L=alexnet/conv2,alexnet/conv3,alexnet/conv4,alexnet/conv5,vgg16/conv1_2,vgg16/conv2_1,vgg16/conv2_2,vgg16/conv3_2,vgg16/conv4_2,vgg16/conv5_2
for kb in 200 216 227; do for b in 1 2; do CLB_SMEM_KB=$kb CLB_BPS=$b timeout 200 python tools/knob_sweep.py $L; done; done > gpurun_out/smem_sweep.txt 2>&1
