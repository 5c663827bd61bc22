#!/bin/bash
# Per-CTA timelines (CLB_TRACE_DUMP) of the short layers: where the fixed cost of a launch goes.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/trace5
O=gpurun_out/trace5
for L in vgg16/conv5_1 alexnet/conv5 alexnet/conv3; do
  n=$(echo $L | tr '/' '_')
  CLB_TRACE=1 CLB_TRACE_DUMP=$O/dump_$n.txt timeout 300 python tools/knob_sweep.py $L > $O/trace_$n.txt 2>&1
done
timeout 300 python tools/knob_sweep.py vgg16/conv5_1 --batch 128 > $O/b128.txt 2>&1
timeout 300 python tools/knob_sweep.py alexnet/conv5 --batch 512 >> $O/b128.txt 2>&1
