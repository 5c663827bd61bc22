#!/bin/bash
# chained prepass: correctness + A/B benches
tag=${1:-chain}; out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -rf -k "chain or concurrent or graph_capture" > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
tail -3 $out/pytest.log
for wl in vgg16 alexnet googlenet; do
  timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > $out/${wl}_seq.json 2> $out/${wl}_seq.err
  timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --chain > $out/${wl}_chain.json 2> $out/${wl}_chain.err
  echo "$wl done"
done
CLB_CHAIN_MIN_MB=0 timeout 600 python bench.py --workload vgg16 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --chain > $out/vgg16_chain_all.json 2>&1
