#!/bin/bash
# effective SM clock inside the tcgen05 kernel (CTA clock64 cycles / globaltimer ns), per layer
mkdir -p gpurun_out
for L in alexnet/conv2 alexnet/conv3 alexnet/conv4 alexnet/conv5 vgg16/conv1_2 vgg16/conv2_2 vgg16/conv4_2 vgg16/conv5_1; do
  echo "== $L"; CLB_TRACE=1 timeout 120 python tools/prof_layer.py --layer $L --reps 20 2>&1 | grep "clb-trace\] rows" | tail -1
done > gpurun_out/trace_clock.txt 2>&1
timeout 60 ./tools/mma_probe > gpurun_out/trace_clock_mma_probe.txt 2>&1
