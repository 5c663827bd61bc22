#!/bin/bash
# A/B of library builds (tools/_ab/lib_<name>.so, same ABI) on kernel times of the given layers
# usage: bash tools/gpu_ab_libs.sh <tag> "<layers>" <variant>...
tag=$1; L=$2; shift 2
out=gpurun_out/$tag; mkdir -p $out
cp paper_1704_04428_b200/libconvlab_b200.so /tmp/keep.so
for r in 1 2; do for v in "$@"; do
  cp tools/_ab/lib_$v.so paper_1704_04428_b200/libconvlab_b200.so
  timeout 300 python tools/knob_sweep.py $L | sed "s/^/$v /" >> $out/ab.txt 2>&1
done; done
cp /tmp/keep.so paper_1704_04428_b200/libconvlab_b200.so
