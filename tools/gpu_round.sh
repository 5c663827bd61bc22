#!/bin/bash
# One GPU session: build check, tests, smoke, facade/plugin programs, short bench.
set -x
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python tools/acc_sweep.py > gpurun_out/acc_sweep.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 300 ./tests/cpp/facade_test gpu > gpurun_out/facade_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/facade_gpu.txt
timeout 300 ./tests/cpp/ref_plugin_test > gpurun_out/ref_plugin.txt 2>&1; echo "rc=$?" >> gpurun_out/ref_plugin.txt
timeout 600 python bench.py --per-layer > gpurun_out/bench_alexnet.json 2> gpurun_out/bench_alexnet.err; echo "bench rc=$?"
timeout 600 python bench.py --workload vgg16 --steps 20 --warmup 3 --per-layer --no-cpu-baseline > gpurun_out/bench_vgg.json 2> gpurun_out/bench_vgg.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
