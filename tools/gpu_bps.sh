#!/bin/bash
# stage-grouping / spin-wait experiment: every tensor-core layer of both workloads under
# CLB_BPS x CLB_SPIN (kernel times)
A=alexnet/conv2,alexnet/conv3,alexnet/conv4,alexnet/conv5
V=vgg16/conv1_2,vgg16/conv2_1,vgg16/conv2_2,vgg16/conv3_1,vgg16/conv3_2,vgg16/conv4_1,vgg16/conv4_2,vgg16/conv5_1,vgg16/conv5_2
mkdir -p gpurun_out
for sp in 0 1; do for b in 1 2 3; do CLB_SPIN=$sp CLB_BPS=$b timeout 300 python tools/knob_sweep.py $A,$V; done; done > gpurun_out/bps_spin.txt 2>&1
