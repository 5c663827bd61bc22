#!/bin/bash
# raw-input A: correctness + VGG A/B against the prepass path
tag=${1:-raw}; out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -rf -x -k "raw_input or tap_shared or concurrent or baseline_shapes or graph" > $out/pytest_raw.log 2>&1; echo "pytest rc=$?" >> $out/pytest_raw.log
tail -3 $out/pytest_raw.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $out/bench_vgg_raw.json 2> $out/bench_vgg_raw.err; echo "raw bench rc=$?"
CLB_RAW_A=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $out/bench_vgg_prepass.json 2> $out/bench_vgg_prepass.err; echo "prepass bench rc=$?"
CLB_RAW_SLOTS=3 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $out/bench_vgg_raw3.json 2> $out/bench_vgg_raw3.err; echo "raw3 bench rc=$?"
timeout 900 python -m pytest tests/test_full_parity.py -m gpu -q -p no:cacheprovider -rf -k "vgg16 and fp32_faithful" > $out/pytest_full_vgg.log 2>&1; echo "full rc=$?" >> $out/pytest_full_vgg.log
tail -3 $out/pytest_full_vgg.log
