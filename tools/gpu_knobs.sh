#!/bin/bash
# kernel times (tools/knob_sweep.py) of the given layers under each CLB_* setting, two passes
# usage (gpurun): bash tools/gpu_knobs.sh <tag> "<layer,layer,...>" "" "CLB_X=1" "CLB_X=0 CLB_Y=2" ...
tag=$1; L=$2; shift 2
out=gpurun_out/$tag; mkdir -p $out
for r in 1 2; do for env in "$@"; do
  env $env timeout 600 python tools/knob_sweep.py $L >> $out/knobs.txt 2>&1
done; done
