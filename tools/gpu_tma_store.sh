#!/bin/bash
out=gpurun_out/${1:-tms}; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -rf -k "tma_store" > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
tail -2 $out/pytest.log
L=vgg16/conv3_1,vgg16/conv3_2,vgg16/conv4_1,vgg16/conv4_2,vgg16/conv5_1,scale,googlenet/3a_1x1,googlenet/4a_1x1,googlenet/4a_3x3
for r in 1 2; do for env in "CLB_TMA_STORE=0" "CLB_TMA_STORE=1"; do
  env $env timeout 600 python tools/knob_sweep.py $L >> $out/knobs.txt 2>&1
done; done
for L in vgg16/conv3_2 vgg16/conv5_1; do for env in "CLB_TMA_STORE=0" "CLB_TMA_STORE=1"; do
  echo "== $L $env" >> $out/trace.txt
  env CLB_TRACE=1 $env timeout 120 python tools/prof_layer.py --layer $L --reps 1 2>&1 | grep "clb-trace" | tail -2 >> $out/trace.txt
done; done
