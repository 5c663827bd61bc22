#!/bin/bash
# A / B TMA issue from two warps (CLB_SPLIT_ISSUE=1): parity + kernel times
mkdir -p gpurun_out
CLB_SPLIT_ISSUE=1 timeout 600 python -m pytest tests/test_fuzz_gpu.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/si_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/si_pytest.txt
L=alexnet/conv2,alexnet/conv3,alexnet/conv4,alexnet/conv5,vgg16/conv1_2,vgg16/conv2_2,vgg16/conv3_2,vgg16/conv4_2,vgg16/conv5_2
{ timeout 200 python tools/knob_sweep.py $L; CLB_SPLIT_ISSUE=1 timeout 200 python tools/knob_sweep.py $L; } > gpurun_out/si_sweep.txt 2>&1
