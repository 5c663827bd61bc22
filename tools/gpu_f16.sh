#!/bin/bash
# fp16 split: GPU suite + kernel times of every VGG-16 / AlexNet layer, default vs the mixed split
out=gpurun_out/${1:-f16}; mkdir -p $out
L=vgg16/conv1_2,vgg16/conv2_1,vgg16/conv2_2,vgg16/conv3_1,vgg16/conv3_2,vgg16/conv4_1,vgg16/conv4_2,vgg16/conv5_1,alexnet/conv2,alexnet/conv3,alexnet/conv4,alexnet/conv5
for env in "" "CLB_MSUB=1" "CLB_SPLIT=mixed"; do
  env $env timeout 300 python tools/knob_sweep.py $L >> $out/times.txt 2>&1
done
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
tail -3 $out/pytest.log
