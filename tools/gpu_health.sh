#!/bin/bash
# Health check after a rebuild: GPU tests, smoke, AlexNet + VGG16 bench lines (per layer).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/health
O=gpurun_out/health
timeout 900 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 600 python bench.py --steps 30 --warmup 5 --per-layer --no-cpu-baseline > $O/bench_alexnet.json 2> $O/bench_alexnet.err
timeout 600 python bench.py --workload vgg16 --steps 20 --warmup 3 --per-layer --no-cpu-baseline > $O/bench_vgg.json 2> $O/bench_vgg.err
