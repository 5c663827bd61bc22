#!/bin/bash
# GPU test suite + bench lines of every workload (no CPU baseline)
# usage (gpurun): bash tools/gpu_suite_benches.sh <tag>
out=gpurun_out/${1:-suite}; mkdir -p $out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
tail -3 $out/pytest.log
timeout 900 python bench.py --no-cpu-baseline > $out/bench_vgg16.json 2> $out/bench_vgg16.err; echo "bench rc=$?"
for wl in alexnet googlenet c1 sweep alexnet-b1 scale; do
timeout 900 python bench.py --workload $wl --no-cpu-baseline > $out/bench_$wl.json 2> $out/bench_$wl.err; echo "$wl rc=$?"
done
