#!/bin/bash
# Two-sub-tile mode (CLB_MSUB=2) on the padded-row layers: kernel time A/B, trace.
mkdir -p gpurun_out/msub
L=${1:-vgg16/conv1_2,vgg16/conv2_1,vgg16/conv2_2,vgg16/conv3_1,googlenet/3a_3x3,c1}
for r in 1 2; do
for m in 1 2; do
  CLB_MSUB=$m timeout 300 python tools/knob_sweep.py $L >> gpurun_out/msub/times2.txt 2>&1
done
done
CLB_MSUB=2 CLB_TRACE=1 timeout 120 python tools/knob_sweep.py vgg16/conv2_1 > gpurun_out/msub/trace2_21.txt 2>&1
cat gpurun_out/msub/times2.txt
