#!/bin/bash
# full GPU suite + method table (with the timing-cache selector) + default bench
tag=${1:-r2d}; out=gpurun_out/$tag; mkdir -p $out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
tail -3 $out/pytest.log
timeout 1500 python tools/method_table.py > $out/method_table.json 2> $out/method_table.err; echo "table rc=$?"
timeout 900 python bench.py > $out/bench_vgg16.json 2> $out/bench_vgg16.err; echo "bench rc=$?"
for wl in alexnet googlenet scale c1 alexnet-b1 sweep; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline --e2e-steps 3 > $out/bench_$wl.json 2> $out/bench_$wl.err; echo "$wl rc=$?"
done
