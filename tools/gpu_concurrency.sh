#!/bin/bash
# new GPU tests + concurrency benches
tag=${1:-r2b}; out=gpurun_out/$tag; mkdir -p $out
timeout 1200 python -m pytest tests/test_cpp_gpu.py tests/test_mshard_gpu.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -rf -k "cpp or mshard or graph_replay_sees or bad_buffers or chain" > $out/pytest_new.log 2>&1; echo "pytest rc=$?" >> $out/pytest_new.log
tail -3 $out/pytest_new.log
for wl in googlenet c1 alexnet-b1 sweep; do
  timeout 600 python bench.py --workload $wl --steps 30 --warmup 5 --no-cpu-baseline > $out/bench_${wl}_seq.json 2> $out/bench_${wl}_seq.err
  timeout 600 python bench.py --workload $wl --steps 30 --warmup 5 --no-cpu-baseline --concurrent > $out/bench_${wl}_conc.json 2> $out/bench_${wl}_conc.err
  echo "$wl rc done"
done
timeout 600 python bench.py --workload c1 --shard channels --steps 20 --warmup 3 --no-cpu-baseline > $out/bench_c1_mshard.json 2> $out/bench_c1_mshard.err; echo "mshard rc=$?"
