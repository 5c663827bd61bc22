#!/bin/bash
# Role-wait traces of batch-1 / small layers (latency regime).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
out=gpurun_out/trace_small.txt; : > $out
run() {   # layer [batch]
  echo "== $*" >> $out
  CLB_TRACE=1 timeout 120 python tools/prof_layer.py --layer $1 ${2:+--batch $2} --reps 2 2>&1 | grep -E "clb-trace|Error" | tail -1 >> $out
}
run c1; run alexnet/conv3 1; run alexnet/conv2 1; run sweep/k3; run sweep/k11; run googlenet/3a_3x3
