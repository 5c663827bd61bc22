#!/bin/bash
# ncu --set full of the padded NCHW -> split prepass (VGG conv1_2) + the knob-path parity tests.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/prep
O=gpurun_out/prep
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tap_shared" > $O/pytest_padded.txt 2>&1; echo "rc=$?" >> $O/pytest_padded.txt
python tools/prof_layer.py --layer vgg16/conv1_2 --reps 1 > $O/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nchw_to -s 1 -c 1 -o $O/prof_prepass_c12 python tools/prof_layer.py --layer vgg16/conv1_2 --reps 1 > $O/ncu.log 2>&1
timeout 300 python tools/fwd_time.py vgg16/conv1_2,vgg16/conv2_2,vgg16/conv3_2,alexnet/conv2,alexnet/conv3 > $O/fwd.txt 2>&1
timeout 300 python tools/knob_sweep.py vgg16/conv1_2,vgg16/conv2_2,vgg16/conv3_2,alexnet/conv2,alexnet/conv3 > $O/kern.txt 2>&1
