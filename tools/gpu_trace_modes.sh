#!/bin/bash
# CLB_TRACE role waits of one layer under several mode settings
out=gpurun_out/${1:-trm}; L=${2:-vgg16/conv1_2}; mkdir -p $out; shift 2
for env in "$@"; do
  echo "== $env" >> $out/trace.txt
  env CLB_TRACE=1 $env timeout 120 python tools/prof_layer.py --layer $L --reps 1 2>&1 | grep "clb-trace" | tail -2 >> $out/trace.txt
done
