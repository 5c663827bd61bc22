#!/bin/bash
# conv1_2: stage grouping (CLB_BPS) vs accumulation chunk length (CLB_CHUNK, k-iterations)
mkdir -p gpurun_out
for cfg in "1 2" "1 3" "2 2" "3 3" "1 4" "2 4"; do
  set -- $cfg
  CLB_BPS=$1 CLB_CHUNK=$2 timeout 120 python tools/knob_sweep.py vgg16/conv1_2,vgg16/conv2_1,vgg16/conv2_2
done > gpurun_out/bps_chunk.txt 2>&1
