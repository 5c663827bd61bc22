#!/bin/bash
# A/B of one CLB_* environment setting on the default bench line, alternating on one box.
# usage: bash tools/gpu_ab_env.sh <tag> "<env A>" "<env B>" [reps] [bench args...]
tag=$1; A=$2; B=$3; reps=${4:-2}; shift 4
out=gpurun_out/$tag; mkdir -p $out
for r in $(seq 1 $reps); do
  env $A timeout 600 python bench.py "$@" > $out/a_$r.json 2> $out/a_$r.err
  env $B timeout 600 python bench.py "$@" > $out/b_$r.json 2> $out/b_$r.err
done
python tools/ab_summary.py $out $reps
