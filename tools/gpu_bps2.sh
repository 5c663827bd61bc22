#!/bin/bash
# k-iterations per stage (CLB_BPS 1 / 2) x tap-stacked on conv1_2 and the padded-row layers.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/bps2
O=gpurun_out/bps2
L=vgg16/conv1_2,vgg16/conv2_1,vgg16/conv2_2,vgg16/conv3_2,alexnet/conv3,alexnet/conv4,c1
for rep in 1 2; do for b in 1 2; do for st in 0 1; do
  env CLB_BPS=$b CLB_STACKED=$st timeout 300 python tools/knob_sweep.py $L >> $O/ab.txt 2>&1
done; done; done
