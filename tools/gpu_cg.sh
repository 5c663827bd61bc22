#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for cg in 1 2; do
CLB_CTA_GROUP=$cg timeout 600 python bench.py --per-layer --no-cpu-baseline > gpurun_out/bench_alexnet_cg$cg.json 2> gpurun_out/bench_alexnet_cg$cg.err
CLB_CTA_GROUP=$cg timeout 600 python bench.py --workload vgg16 --steps 20 --warmup 3 --per-layer --no-cpu-baseline > gpurun_out/bench_vgg_cg$cg.json 2> gpurun_out/bench_vgg_cg$cg.err
done
