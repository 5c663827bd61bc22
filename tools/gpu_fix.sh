#!/bin/bash
# Stream-K finisher staging partner partials in smem (CLB_FIXUP_SMEM): A/B + trace + GPU suite.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/fix
O=gpurun_out/fix
timeout 900 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
L=alexnet/conv3,alexnet/conv4,alexnet/conv5,vgg16/conv5_1,vgg16/conv4_1,googlenet/3a_3x3,googlenet/5b_3x3,c1,sweep/k7,sweep/k11,alexnet/conv2
for rep in 1 2; do for fx in 0 1; do
  env CLB_FIXUP_SMEM=$fx timeout 300 python tools/knob_sweep.py $L >> $O/ab.txt 2>&1
done; done
CLB_TRACE=1 CLB_TRACE_DUMP=$O/dump_conv5.txt timeout 300 python tools/knob_sweep.py alexnet/conv5 > /dev/null 2>&1
for rep in 1 2; do for fx in 0 1; do
  echo "CLB_FIXUP_SMEM=$fx alexnet $(CLB_FIXUP_SMEM=$fx timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],1), round(d["ms_per_step"],4))')" >> $O/bench.txt
done; done
