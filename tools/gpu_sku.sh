#!/bin/bash
# Stream-K unit count model (CLB_SK_UNITS): A/B over stream-K-heavy layers + GPU suite.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/sku
O=gpurun_out/sku
L=vgg16/conv5_1,vgg16/conv4_1,vgg16/conv3_1,alexnet/conv3,alexnet/conv5,googlenet/3a_3x3,googlenet/4a_1x1,googlenet/5b_3x3,c1,sweep/k7,sweep/k11
for rep in 1 2; do for sk in 0 1; do
  env CLB_SK_UNITS=$sk timeout 300 python tools/knob_sweep.py $L >> $O/ab.txt 2>&1
done; done
CLB_TRACE=1 timeout 300 python tools/knob_sweep.py vgg16/conv5_1 2>&1 | grep -v slowest | tail -n 2 | cut -c1-300 > $O/trace.txt
timeout 900 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
