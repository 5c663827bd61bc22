#!/bin/bash
# L2 prefetch of the next piece's A rows: A/B on the padded-row layers, stacked on/off.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/prefetch
O=gpurun_out/prefetch
L=c1,vgg16/conv1_2,vgg16/conv2_1,vgg16/conv2_2,vgg16/conv3_1,vgg16/conv3_2,vgg16/conv4_1,vgg16/conv4_2,vgg16/conv5_1,googlenet/3a_5x5,googlenet/4a_3x3,alexnet/conv3,alexnet/conv4
for pf in 0 1; do for st in 0 1; do
  env CLB_L2_PREFETCH=$pf CLB_STACKED=$st timeout 300 python tools/knob_sweep.py $L >> $O/ab.txt 2>&1
done; done
CLB_STACKED=1 CLB_TRACE=1 timeout 300 python tools/knob_sweep.py vgg16/conv1_2 2>&1 | grep -v slowest | tail -n 2 > $O/trace.txt
CLB_STACKED=0 CLB_TRACE=1 timeout 300 python tools/knob_sweep.py vgg16/conv1_2 2>&1 | grep -v slowest | tail -n 2 >> $O/trace.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tap_shared" > $O/pytest_padded.txt 2>&1; echo "rc=$?" >> $O/pytest_padded.txt
