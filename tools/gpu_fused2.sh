#!/bin/bash
# Fused prepass auto rule (<= 2 MB inputs): GPU suite + batch-1 forward times auto vs off.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/fused2
O=gpurun_out/fused2
timeout 900 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
L=c1,sweep/k1,sweep/k3,sweep/k5,sweep/k7,sweep/k11,googlenet/4a_5x5,googlenet/5b_5x5
for rep in 1 2; do for fu in 0 auto; do
  if [ $fu = auto ]; then env -u CLB_FUSED_PREPASS timeout 300 python tools/fwd_time.py $L >> $O/fwd.txt 2>&1;
  else CLB_FUSED_PREPASS=0 timeout 300 python tools/fwd_time.py $L >> $O/fwd.txt 2>&1; fi
done; done
for rep in 1 2; do for fu in 0 auto; do
  if [ $fu = auto ]; then env -u CLB_FUSED_PREPASS timeout 300 python tools/fwd_time.py alexnet/conv2,alexnet/conv3,alexnet/conv4,alexnet/conv5 --batch 1 >> $O/fwd_b1.txt 2>&1;
  else CLB_FUSED_PREPASS=0 timeout 300 python tools/fwd_time.py alexnet/conv2,alexnet/conv3,alexnet/conv4,alexnet/conv5 --batch 1 >> $O/fwd_b1.txt 2>&1; fi
done; done
