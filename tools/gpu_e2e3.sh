#!/bin/bash
# VGG16 / AlexNet e2e with the fused prepass auto rule vs off (host-pipeline chunks are sub-batches).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/e2e3
O=gpurun_out/e2e3
for rep in 1 2; do for fu in 0 auto; do
  if [ $fu = auto ]; then E="env -u CLB_FUSED_PREPASS"; else E="env CLB_FUSED_PREPASS=0"; fi
  echo "fused=$fu vgg16 $($E timeout 300 python bench.py --workload vgg16 --steps 10 --warmup 3 --e2e-steps 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["e2e"]["value"],2))')" >> $O/ab.txt
  echo "fused=$fu alexnet $($E timeout 300 python bench.py --steps 30 --warmup 5 --e2e-steps 10 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["e2e"]["value"],2))')" >> $O/ab.txt
done; done
