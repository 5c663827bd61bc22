#!/bin/bash
# Role wait-time traces (CLB_TRACE=1) of the implicit kernel on representative layers.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
out=gpurun_out/trace.txt; : > $out
for L in vgg16/conv1_2 vgg16/conv2_1 vgg16/conv2_2 vgg16/conv3_1 vgg16/conv4_1 vgg16/conv5_1 alexnet/conv3; do
  echo "== $L" >> $out
  CLB_TRACE=1 timeout 120 python tools/prof_layer.py --layer $L --reps 1 2>&1 | grep -E "clb-trace|ok|Error" | tail -2 >> $out
done
for cg in 1 2; do
  echo "== vgg16/conv1_2 CLB_CTA_GROUP=$cg" >> $out
  CLB_CTA_GROUP=$cg CLB_TRACE=1 timeout 120 python tools/prof_layer.py --layer vgg16/conv1_2 --reps 1 2>&1 | grep -E "clb-trace" | tail -1 >> $out
done
echo "== vgg16/conv1_2 padded" >> $out
CLB_PADDED_ROWS=1 CLB_TRACE=1 timeout 120 python tools/prof_layer.py --layer vgg16/conv1_2 --reps 1 2>&1 | grep -E "clb-trace" | tail -1 >> $out
