#!/bin/bash
# Round-end evidence (no profiler): tests, smoke, C++ programs, benches, reference arm, report.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 900 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 300 ./tests/cpp/facade_test gpu > $O/facade_gpu.txt 2>&1; echo "rc=$?" >> $O/facade_gpu.txt
timeout 300 ./tests/cpp/ref_plugin_test > $O/ref_plugin.txt 2>&1; echo "rc=$?" >> $O/ref_plugin.txt
timeout 900 python bench.py > $O/bench_alexnet.json 2> $O/bench_alexnet.err; echo "bench rc=$?" >> $O/bench_alexnet.err
timeout 900 python bench.py --workload vgg16 --steps 20 --warmup 3 --per-layer --no-cpu-baseline > $O/bench_vgg.json 2> $O/bench_vgg.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 2400 python tools/report.py > $O/report_all.json 2> $O/report_all.err
