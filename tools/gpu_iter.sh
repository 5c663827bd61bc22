#!/bin/bash
# one iteration: GPU parity suite, per-layer kernel times, AlexNet + VGG16 bench (30 steps)
mkdir -p gpurun_out
A=alexnet/conv2,alexnet/conv3,alexnet/conv4,alexnet/conv5
V=vgg16/conv1_2,vgg16/conv2_1,vgg16/conv2_2,vgg16/conv3_1,vgg16/conv3_2,vgg16/conv3_3,vgg16/conv4_1,vgg16/conv4_2,vgg16/conv4_3,vgg16/conv5_1,vgg16/conv5_2,vgg16/conv5_3
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/iter_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/iter_pytest.txt
timeout 300 python tools/knob_sweep.py $A,$V > gpurun_out/iter_layers.txt 2>&1
if [ "${ITER_BENCH:-1}" = 1 ]; then
{ timeout 300 python bench.py --steps 30 --warmup 5; timeout 300 python bench.py --steps 30 --warmup 5 --workload vgg16; } > gpurun_out/iter_bench.txt 2> gpurun_out/iter_bench.err
fi
