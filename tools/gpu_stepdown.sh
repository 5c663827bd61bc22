#!/bin/bash
# Per-step device times of a 150-step AlexNet bench + nvidia-smi samples (SM/mem clock, power, temps).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/stepdown
O=gpurun_out/stepdown
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,temperature.memory,clocks_throttle_reasons.active --format=csv -lms 100 > $O/smi.csv 2>&1 &
SMI=$!
CLB_BENCH_STEP_MS=1 timeout 600 python bench.py --steps 150 --warmup 10 --no-cpu-baseline --e2e-steps 1 > $O/bench.json 2> $O/steps.txt
CLB_FLUSH_MB=0 CLB_BENCH_STEP_MS=1 timeout 600 python bench.py --steps 150 --warmup 10 --no-cpu-baseline --e2e-steps 1 > $O/bench_noflush.json 2> $O/steps_noflush.txt
kill $SMI
