#!/bin/bash
# accumulation chunk length (CLB_CHUNK, k-iterations) x stage grouping (CLB_BPS): speed + accuracy
A=alexnet/conv2,alexnet/conv3,alexnet/conv4,alexnet/conv5,vgg16/conv3_1,vgg16/conv3_2,vgg16/conv4_1,vgg16/conv4_2,vgg16/conv5_1,vgg16/conv5_2
P=vgg16/conv1_2,vgg16/conv2_1,vgg16/conv2_2
mkdir -p gpurun_out
{
for b in 1 2; do for c in 8 12 16; do CLB_BPS=$b CLB_CHUNK=$c timeout 200 python tools/knob_sweep.py $A; done; done
for b in 1 2 3; do for c in 2 3 4 6; do CLB_BPS=$b CLB_CHUNK=$c timeout 200 python tools/knob_sweep.py $P; done; done
} > gpurun_out/chunk_speed.txt 2>&1
for c in 8 12 16 32; do echo "== CLB_CHUNK=$c (16 K-elements per iteration)"; CLB_CHUNK=$c timeout 200 python tools/acc_sweep.py; done > gpurun_out/chunk_acc.txt 2>&1
