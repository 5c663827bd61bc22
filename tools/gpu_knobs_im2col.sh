#!/bin/bash
out=gpurun_out/${1:-kim}; mkdir -p $out
L=vgg16/conv3_1,vgg16/conv3_2,vgg16/conv4_1,vgg16/conv4_2,vgg16/conv5_1,scale,alexnet/conv3,alexnet/conv4,alexnet/conv5,alexnet/conv2
for r in 1 2; do for env in "" "CLB_BPS=1" "CLB_SMEM_KB=220" "CLB_BPS=1 CLB_SMEM_KB=220" "CLB_BPS=3"; do
  env $env timeout 600 python tools/knob_sweep.py $L >> $out/knobs.txt 2>&1
done; done
for env in "" "CLB_BPS=1" "CLB_BPS=1 CLB_SMEM_KB=220"; do
  echo "== conv3_2 $env" >> $out/trace.txt
  env CLB_TRACE=1 $env timeout 120 python tools/prof_layer.py --layer vgg16/conv3_2 --reps 1 2>&1 | grep "clb-trace" | tail -2 >> $out/trace.txt
done
