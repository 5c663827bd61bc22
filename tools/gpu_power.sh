#!/bin/bash
# power limits of the box + SM clock / power draw sampled every 50 ms during the two benches
mkdir -p gpurun_out
nvidia-smi -q -d POWER,CLOCK,PERFORMANCE > gpurun_out/power_q.txt 2>&1
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv -lms 50 > gpurun_out/power_trace.csv 2>&1 &
SMI=$!
sleep 1
echo "alexnet start $(date +%T.%N)" > gpurun_out/power_marks.txt
timeout 300 python bench.py --steps 100 --warmup 5 > gpurun_out/power_bench.txt 2>/dev/null
echo "vgg start $(date +%T.%N)" >> gpurun_out/power_marks.txt
timeout 300 python bench.py --steps 100 --warmup 5 --workload vgg16 >> gpurun_out/power_bench.txt 2>/dev/null
echo "end $(date +%T.%N)" >> gpurun_out/power_marks.txt
sleep 1; kill $SMI
