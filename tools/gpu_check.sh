#!/bin/bash
# round-2 GPU check: GPU test suite, smoke, default bench (VGG-16), other workloads.
# usage (gpurun): bash tools/gpu_r2.sh <tag> [pytest-args...]
tag=${1:-r2}; shift
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf "$@" > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
tail -3 $out/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
tail -2 $out/smoke.log
timeout 900 python bench.py > $out/bench_vgg16.json 2> $out/bench_vgg16.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref rc=$?"
