#!/bin/bash
# Weight-stationary B: parity (padded/stacked subprocess tests + full GPU suite) and A/B timing.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/bres
O=gpurun_out/bres
L=c1,vgg16/conv1_2,vgg16/conv2_1,googlenet/3a_5x5,googlenet/4a_5x5,googlenet/4a_3x3,googlenet/3a_1x1,sweep/k5,sweep/k3
for br in 0 -1; do for st in 0 1; do
  env CLB_B_RESIDENT=$br CLB_STACKED=$st timeout 300 python tools/knob_sweep.py $L >> $O/ab.txt 2>&1
done; done
CLB_STACKED=1 CLB_TRACE=1 timeout 300 python tools/knob_sweep.py vgg16/conv1_2 2>&1 | grep -v slowest | tail -n 2 > $O/trace.txt
CLB_STACKED=0 CLB_TRACE=1 timeout 300 python tools/knob_sweep.py vgg16/conv1_2 2>&1 | grep -v slowest | tail -n 2 >> $O/trace.txt
timeout 900 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
