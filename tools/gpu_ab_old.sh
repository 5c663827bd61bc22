#!/bin/bash
# A/B of the current build against the round-2 pre-fp16 build (tools/_ab/old) on small mixed-split layers
out=gpurun_out/${1:-abold}; mkdir -p $out
L=${2:-c1,alexnet/conv3,alexnet/conv4,googlenet/3a_1x1,googlenet/4a_5x5,sweep/k3}
for r in 1 2; do
  CLB_SPLIT=mixed timeout 300 python tools/knob_sweep.py $L | sed 's/^/NEW /' >> $out/ab.txt 2>&1
  CLB_SPLIT=mixed timeout 300 python tools/_ab/old/tools/knob_sweep.py $L | sed 's/^/OLD /' >> $out/ab.txt 2>&1
done
