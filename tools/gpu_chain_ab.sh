#!/bin/bash
# chained-prepass heuristics A/B: sequential vs chain (heuristic) vs chain (host every eligible prepass)
tag=${1:-chainab}; out=gpurun_out/$tag; mkdir -p $out
for wl in vgg16 alexnet googlenet scale; do
  for mode in seq chain force; do
    extra=""; envs=""
    [ $mode = chain ] && extra="--chain"
    [ $mode = force ] && extra="--chain" && envs="CLB_CHAIN_FORCE=1"
    env $envs timeout 600 python bench.py --workload $wl --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 $extra > $out/${wl}_$mode.json 2> $out/${wl}_$mode.err
  done
  echo "$wl done"
done
