#!/bin/bash
# ncu evidence for the default bench (VGG-16 b32): (1) launch list of the bench command,
# (2) one --set full capture of the 12 tc_conv_kernel launches of one timed step (traffic).
# usage (gpurun): bash tools/gpu_prof_vgg.sh <tag> [extra bench args]
tag=${1:-prof}; shift
out=gpurun_out/$tag; mkdir -p $out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 $*"
$B > $out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $out/launches.csv $B > $out/ncu_launch.log 2>&1
echo "launch list rc=$?"
B1="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 $*"
$B1 > $out/plain_bench1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc_conv_kernel -s 12 -c 12 -o $out/step $B1 > $out/ncu_full.log 2>&1
echo "full rc=$?"
