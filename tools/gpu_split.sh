#!/bin/bash
# Stream-K split cap sweep on small / latency-bound layers (kernel time, tools/knob_sweep.py).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
out=gpurun_out/split.txt; : > $out
L=c1,sweep/k1,sweep/k3,sweep/k7,googlenet/3a_1x1,googlenet/3a_3x3,googlenet/3a_5x5,googlenet/4a_3x3,googlenet/5b_1x1,googlenet/5b_3x3,googlenet/5b_5x5,vgg16/conv5_1,alexnet/conv5
for s in 1 2 3 4 6; do env CLB_MAX_SPLIT=$s timeout 300 python tools/knob_sweep.py $L >> $out 2>&1; done
for b in 1; do for s in 1 2 3 4 6; do env CLB_MAX_SPLIT=$s timeout 300 python tools/knob_sweep.py alexnet/conv2,alexnet/conv3 --batch 1 >> $out 2>&1; done; done
