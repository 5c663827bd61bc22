#!/bin/bash
# Shared-memory budget sweep (more pipeline bytes in flight): kernel time per layer.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/smem
O=gpurun_out/smem
L=vgg16/conv1_2,c1,vgg16/conv2_1,vgg16/conv3_1,vgg16/conv4_2,vgg16/conv5_1,alexnet/conv2,alexnet/conv3,alexnet/conv4,alexnet/conv5,googlenet/4a_5x5
for kb in 200 212 224; do for st in 0 1; do
  env CLB_SMEM_KB=$kb CLB_STACKED=$st timeout 300 python tools/knob_sweep.py $L >> $O/ab.txt 2>&1
done; done
