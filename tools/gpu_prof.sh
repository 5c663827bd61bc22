#!/bin/bash
# ncu pass for the committed evidence: (1) launch list of the bench command, (2) one
# --set full capture of the 4 tc_conv_kernel launches of one timed bench step.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$B > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_alexnet.csv $B > gpurun_out/ncu_launch.log 2>&1
B1="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$B1 > gpurun_out/plain_bench1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc_conv_kernel -s 4 -c 4 -o gpurun_out/prof_alexnet_step $B1 > gpurun_out/ncu_full.log 2>&1
python tools/prof_layer.py --layer vgg16/conv1_2 --reps 1 > gpurun_out/plain_c12.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc_conv_kernel -s 1 -c 1 -o gpurun_out/prof_vgg16_conv1_2 python tools/prof_layer.py --layer vgg16/conv1_2 --reps 1 > gpurun_out/ncu_c12.log 2>&1
