#!/bin/bash
# alternating repetitions: sequential vs chained (host every eligible prepass) on VGG-16
tag=${1:-chainrep}; out=gpurun_out/$tag; mkdir -p $out
for r in 1 2 3; do
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $out/seq_$r.json 2>/dev/null
  CLB_CHAIN_FORCE=1 timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 --chain > $out/force_$r.json 2>/dev/null
  CLB_CHAIN_MIN_MB=0 timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 --chain > $out/min0_$r.json 2>/dev/null
done
