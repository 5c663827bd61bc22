#!/bin/bash
# Role-wait traces of the mid-size VGG layers.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/tracevgg
O=gpurun_out/tracevgg
for L in vgg16/conv2_1 vgg16/conv2_2 vgg16/conv3_1 vgg16/conv4_2 alexnet/conv4; do
  CLB_TRACE=1 timeout 300 python tools/knob_sweep.py $L 2>&1 | grep -v slowest | tail -n 2 | cut -c1-520 >> $O/trace.txt
done
