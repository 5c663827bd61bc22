#!/bin/bash
out=gpurun_out/${1:-spec}; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -rf -k "f16_split or operand_split or padded_row or nhwc or graph or host" > $out/pytest_new.log 2>&1; echo "rc=$?" >> $out/pytest_new.log
tail -3 $out/pytest_new.log
timeout 900 python bench.py --no-cpu-baseline > $out/bench_vgg16.json 2> $out/bench_vgg16.err; echo "bench rc=$?"
CLB_F16_SPEC=0 timeout 900 python bench.py --no-cpu-baseline > $out/bench_vgg16_twopass.json 2> /dev/null; echo "bench2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $out/ncu.log 2>&1; echo "ncu rc=$?"
