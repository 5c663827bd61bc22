#!/bin/bash
# A/B of library variants (tools/_ab/lib_<name>.so, same ABI) and the pre-fp16 build (tools/_ab/old)
# usage: bash tools/gpu_ab_variants.sh <tag> "<layers>" "<env>" <variant>...
tag=$1; L=$2; E=$3; shift 3
out=gpurun_out/$tag; mkdir -p $out
cp paper_1704_04428_b200/libconvlab_b200.so /tmp/keep.so
for r in 1 2; do
  for v in "$@"; do
    cp tools/_ab/lib_$v.so paper_1704_04428_b200/libconvlab_b200.so
    env $E timeout 300 python tools/knob_sweep.py $L | sed "s/^/$v /" >> $out/ab.txt 2>&1
  done
  env $E timeout 300 python tools/_ab/old/tools/knob_sweep.py $L | sed 's/^/old /' >> $out/ab.txt 2>&1
done
cp /tmp/keep.so paper_1704_04428_b200/libconvlab_b200.so
