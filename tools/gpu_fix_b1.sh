#!/bin/bash
# Batch-1 layers: staged (smem) vs global-load stream-K fixup, CUDA-graph forward times (tools/report.py).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/fixb1
O=gpurun_out/fixb1
for rep in 1 2; do for fx in 0 1; do
  CLB_FIXUP_SMEM=$fx timeout 900 python tools/report.py --workloads c1,alexnet-b1,sweep,googlenet --no-cpu > $O/rep_fix$fx\_$rep.json 2> /dev/null
done; done
