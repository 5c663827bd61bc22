#!/bin/bash
# round-end evidence: GPU suite, smoke, C++ boundary, default bench + reference arm, every
# workload (sequential / concurrent / chain), fast modes, method table, per-layer report.
tag=${1:-final}; out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $out/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
tail -2 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench_vgg16.json 2> $out/bench_vgg16.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $out/bench_reference.json 2> $out/bench_reference.err; echo "ref rc=$?"
timeout 900 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > $out/bench_vgg16_100steps.json 2> /dev/null
timeout 900 python bench.py --chain --steps 30 --warmup 5 --no-cpu-baseline > $out/bench_vgg16_chain.json 2> /dev/null
for p in tf32 bf16; do timeout 900 python bench.py --precision $p --steps 30 --warmup 5 --no-cpu-baseline > $out/bench_vgg16_$p.json 2> /dev/null; done
CLB_SPLIT=3xtf32 timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $out/bench_vgg16_3xtf32.json 2> /dev/null
for wl in alexnet scale googlenet c1 alexnet-b1 sweep; do
  timeout 900 python bench.py --workload $wl --steps 30 --warmup 5 > $out/bench_$wl.json 2> /dev/null
done
for wl in googlenet c1 alexnet-b1 sweep; do
  timeout 900 python bench.py --workload $wl --steps 30 --warmup 5 --no-cpu-baseline --concurrent > $out/bench_${wl}_concurrent.json 2> /dev/null
done
timeout 900 python bench.py --workload c1 --shard channels --steps 30 --warmup 5 --no-cpu-baseline > $out/bench_c1_mshard.json 2> /dev/null
echo benches done
timeout 1500 python tools/method_table.py > $out/method_table.json 2> /dev/null; echo "table rc=$?"
timeout 2400 python tools/report.py > $out/report.json 2> $out/report.err; echo "report rc=$?"
