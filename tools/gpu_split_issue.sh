#!/bin/bash
# TMA issue split levels (CLB_SPLIT_ISSUE=0|1|2): parity at the default, kernel times, A/B bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/si_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/si_pytest.txt
L=alexnet/conv2,alexnet/conv3,alexnet/conv4,alexnet/conv5,vgg16/conv1_2,vgg16/conv3_2,vgg16/conv5_2,googlenet/4a_3x3
{ for si in 1 2; do CLB_SPLIT_ISSUE=$si timeout 200 python tools/knob_sweep.py $L; done; } > gpurun_out/si_sweep.txt 2>&1
for si in 1 2 1 2; do CLB_SPLIT_ISSUE=$si timeout 300 python bench.py --steps 30 --warmup 5 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print('split', $si, round(d['value'],1), d['ms_per_step'])"; done > gpurun_out/ab.txt 2>&1
