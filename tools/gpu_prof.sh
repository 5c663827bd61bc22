#!/bin/bash
# ncu pass: launch list of the bench command + full capture of tc_conv_kernel on key layers.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$B > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_alexnet.csv $B > gpurun_out/ncu_launch.log 2>&1
for L in vgg16/conv1_2 vgg16/conv4_2 alexnet/conv3; do
  tag=$(echo $L | tr '/' '_')
  python tools/prof_layer.py --layer $L --reps 1 > gpurun_out/plain_$tag.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:tc_conv_kernel -s 1 -c 1 -o gpurun_out/prof_$tag python tools/prof_layer.py --layer $L --reps 1 > gpurun_out/ncu_$tag.log 2>&1
done
