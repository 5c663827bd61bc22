#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
L=${1:-vgg16/conv5_1,alexnet/conv3,alexnet/conv4,alexnet/conv5,vgg16/conv3_1,vgg16/conv2_2}
out=gpurun_out/knobs2.txt; : > $out
for cg in 0 1 2; do for bn in 0 128 192 256; do
  env CLB_CTA_GROUP=$cg CLB_BN=$bn timeout 300 python tools/knob_sweep.py $L >> $out 2>&1
done; done
