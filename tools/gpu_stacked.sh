#!/bin/bash
# Tap-stacked mode: parity tests (forced on / off) and per-layer A/B kernel times.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/stacked
O=gpurun_out/stacked
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tap_shared" > $O/pytest_padded.txt 2>&1; echo "rc=$?" >> $O/pytest_padded.txt
L=c1,vgg16/conv1_2,googlenet/3a_5x5,googlenet/4a_5x5,vgg16/conv2_1
for st in 0 1; do
  env CLB_STACKED=$st timeout 300 python tools/knob_sweep.py $L >> $O/ab.txt 2>&1
done
CLB_STACKED=1 CLB_TRACE=1 timeout 300 python tools/knob_sweep.py vgg16/conv1_2 > $O/trace_conv1_2.txt 2>&1
CLB_STACKED=0 CLB_TRACE=1 timeout 300 python tools/knob_sweep.py vgg16/conv1_2 >> $O/trace_conv1_2.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
