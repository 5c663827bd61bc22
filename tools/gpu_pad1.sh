#!/bin/bash
# shared-padding padded-row mode with CTA-pair sizing: parity under forced padded, kernel times auto / forced / off
mkdir -p gpurun_out
CLB_PADDED_ROWS=1 timeout 600 python -m pytest tests/test_fuzz_gpu.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pad3_pytest_forced.txt 2>&1; echo "rc=$?" >> gpurun_out/pad3_pytest_forced.txt
L=alexnet/conv2,alexnet/conv3,alexnet/conv4,alexnet/conv5,vgg16/conv1_2,vgg16/conv2_1,vgg16/conv2_2,vgg16/conv3_1,vgg16/conv3_2,vgg16/conv4_1,vgg16/conv4_2,vgg16/conv5_1,vgg16/conv5_2,googlenet/3a_3x3,googlenet/3a_5x5,googlenet/4a_3x3,googlenet/4a_5x5,googlenet/5b_3x3,googlenet/5b_5x5
{
timeout 300 python tools/knob_sweep.py $L
CLB_PADDED_ROWS=1 timeout 300 python tools/knob_sweep.py $L
CLB_PADDED_ROWS=0 timeout 300 python tools/knob_sweep.py $L
} > gpurun_out/pad3_sweep.txt 2>&1
