#!/bin/bash
# PDL on the prepass (overlap with the previous layer's contraction): bench A/B (alternating) + GPU suite.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/pdl
O=gpurun_out/pdl
timeout 900 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
for rep in 1 2; do for pdl in 0 1; do
  echo "CLB_PDL_PREPASS=$pdl alexnet $(CLB_PDL_PREPASS=$pdl timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"],4), d["roofline"]["kernel_ms_per_step"])')" >> $O/ab.txt
  echo "CLB_PDL_PREPASS=$pdl vgg16 $(CLB_PDL_PREPASS=$pdl timeout 300 python bench.py --workload vgg16 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"],4), d["roofline"]["kernel_ms_per_step"])')" >> $O/ab.txt
done; done
