#!/bin/bash
# Fused prepass (phase 0 of the contraction) vs standalone prepass: parity, per-layer forward time, bench.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/fused
O=gpurun_out/fused
timeout 900 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
L=alexnet/conv2,alexnet/conv3,alexnet/conv4,alexnet/conv5,vgg16/conv1_2,vgg16/conv2_2,vgg16/conv3_2,vgg16/conv4_2,vgg16/conv5_1,googlenet/3a_1x1,googlenet/4a_3x3,c1
for rep in 1 2; do for fu in 0 1; do
  env CLB_FUSED_PREPASS=$fu timeout 300 python tools/fwd_time.py $L >> $O/fwd.txt 2>&1
done; done
for rep in 1 2; do for fu in 0 1; do
  echo "CLB_FUSED_PREPASS=$fu alexnet $(CLB_FUSED_PREPASS=$fu timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"],4), round(d["roofline"]["kernel_ms_per_step"],4), round(d["e2e"]["value"],2), d["gpu_launches"])')" >> $O/bench.txt
  echo "CLB_FUSED_PREPASS=$fu vgg16 $(CLB_FUSED_PREPASS=$fu timeout 300 python bench.py --workload vgg16 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"],4), round(d["roofline"]["kernel_ms_per_step"],4), round(d["e2e"]["value"],2), d["gpu_launches"])')" >> $O/bench.txt
done; done
