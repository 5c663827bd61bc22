#!/bin/bash
# CLB_TRACE role waits of several layers under the current defaults
out=gpurun_out/${1:-trl}; mkdir -p $out; shift
for L in "$@"; do
  echo "== $L" >> $out/trace.txt
  CLB_TRACE=1 timeout 120 python tools/prof_layer.py --layer $L --reps 1 2>&1 | grep "clb-trace" | tail -2 >> $out/trace.txt
done
