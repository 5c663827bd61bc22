#!/bin/bash
# bench lines (VGG default, AlexNet) + the ncu launch list of the default bench
out=gpurun_out/${1:-f16d}; mkdir -p $out
timeout 900 python bench.py --no-cpu-baseline > $out/bench_vgg16.json 2> $out/bench_vgg16.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $out/ncu.log 2>&1; echo "ncu rc=$?"
