#!/bin/bash
mkdir -p gpurun_out
for si in 0 1 0 1; do CLB_SPLIT_ISSUE=$si timeout 300 python bench.py --steps 30 --warmup 5 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print('split', $si, round(d['value'],1), d['ms_per_step'])"; done > gpurun_out/ab.txt 2>&1
