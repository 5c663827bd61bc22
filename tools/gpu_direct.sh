#!/bin/bash
# Parameter-weight direct kernel (CLB_DIRECT_PARAM) vs shared-memory weights: parity + VGG conv1_1 time.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/direct
O=gpurun_out/direct
timeout 900 python -m pytest tests -q -m gpu -x -k "direct or selector or smoke or guard or fixtures or border or grid" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
for rep in 1 2; do for dp in 0 1; do
  env CLB_DIRECT_PARAM=$dp timeout 300 python tools/knob_sweep.py vgg16/conv1_1 >> $O/ab.txt 2>&1
done; done
