#!/bin/bash
# A loads from two warps (alternate stages): A/B per layer, then parity with it forced on.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/aiss
O=gpurun_out/aiss
L=alexnet/conv2,alexnet/conv3,alexnet/conv4,alexnet/conv5,vgg16/conv5_1,vgg16/conv4_2,vgg16/conv1_2,vgg16/conv2_2,googlenet/3a_3x3
for rep in 1 2; do for ai in 1 2; do
  env CLB_A_ISSUERS=$ai timeout 300 python tools/knob_sweep.py $L >> $O/ab.txt 2>&1
done; done
CLB_A_ISSUERS=2 timeout 900 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
