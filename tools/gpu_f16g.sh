#!/bin/bash
out=gpurun_out/${1:-f16g}; mkdir -p $out
L=vgg16/conv1_2,vgg16/conv2_1,vgg16/conv2_2,vgg16/conv3_1,vgg16/conv3_2,vgg16/conv4_1,vgg16/conv4_2,vgg16/conv5_1,alexnet/conv2,alexnet/conv3,alexnet/conv4,alexnet/conv5,googlenet/3a_1x1,googlenet/3a_3x3,googlenet/3a_5x5,googlenet/4a_1x1,googlenet/4a_3x3,googlenet/4a_5x5,googlenet/5b_1x1,googlenet/5b_3x3,googlenet/5b_5x5,sweep/k1,sweep/k3,sweep/k5,sweep/k7,sweep/k11,c1
for env in "" "CLB_SPLIT=mixed" "CLB_CHUNK=1"; do
  env $env timeout 600 python tools/knob_sweep.py $L >> $out/knobs.txt 2>&1
done
timeout 900 python bench.py --no-cpu-baseline > $out/bench_vgg16.json 2> $out/bench_vgg16.err; echo "bench rc=$?"
