#!/bin/bash
# Padded rows with one tap per stage (tiled A boxes, no k-tap B stage) vs the defaults, and role traces.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/tps1
O=gpurun_out/tps1
L=alexnet/conv2,alexnet/conv3,alexnet/conv4,alexnet/conv5,vgg16/conv4_2,vgg16/conv5_1,vgg16/conv3_2,c1,sweep/k5
timeout 300 python tools/knob_sweep.py $L > $O/ab.txt 2>&1
CLB_PADDED_ROWS=1 CLB_TPS1=1 timeout 300 python tools/knob_sweep.py $L >> $O/ab.txt 2>&1
CLB_PADDED_ROWS=1 timeout 300 python tools/knob_sweep.py $L >> $O/ab.txt 2>&1
CLB_TRACE=1 timeout 300 python tools/knob_sweep.py alexnet/conv2,alexnet/conv3,alexnet/conv5 2>&1 | grep -v slowest | awk 'NR%8==0 || /TF/' > $O/trace_default.txt
CLB_PADDED_ROWS=1 CLB_TPS1=1 CLB_TRACE=1 timeout 300 python tools/knob_sweep.py alexnet/conv2,alexnet/conv3,alexnet/conv5 2>&1 | grep -v slowest | awk 'NR%8==0 || /TF/' > $O/trace_tps1.txt
