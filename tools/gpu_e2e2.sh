#!/bin/bash
# Shared per-device copy streams (CLB_HOST_SHARED_STREAMS) vs per-plan: e2e A/B (alternating), host trace, tests.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/e2e2
O=gpurun_out/e2e2
for rep in 1 2; do for sh in 0 1; do
  echo "CLB_HOST_SHARED_STREAMS=$sh alexnet $(CLB_HOST_SHARED_STREAMS=$sh timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 20 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["e2e"]["value"],2))')" >> $O/ab.txt
  echo "CLB_HOST_SHARED_STREAMS=$sh vgg16 $(CLB_HOST_SHARED_STREAMS=$sh timeout 300 python bench.py --workload vgg16 --steps 3 --warmup 3 --e2e-steps 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["e2e"]["value"],2))')" >> $O/ab.txt
done; done
timeout 900 python -m pytest tests -q -m gpu -x -k "host or graph or shared or async" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 300 ./tests/cpp/facade_test gpu > $O/facade.txt 2>&1; echo "rc=$?" >> $O/facade.txt
