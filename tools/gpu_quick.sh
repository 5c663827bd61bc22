#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 300 ./tools/tma_probe > gpurun_out/tma_probe4.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --per-layer --no-cpu-baseline > gpurun_out/bench_alexnet.json 2> gpurun_out/bench_alexnet.err
timeout 600 python bench.py --workload vgg16 --steps 20 --warmup 3 --per-layer --no-cpu-baseline > gpurun_out/bench_vgg.json 2> gpurun_out/bench_vgg.err
