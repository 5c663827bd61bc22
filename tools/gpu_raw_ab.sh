#!/bin/bash
# raw-input A bisection: whole-forward time of VGG layers under CLB_RAW_* variants
L=${1:-vgg16/conv1_2,vgg16/conv2_2,vgg16/conv3_2,vgg16/conv4_2}
python tools/fwd_time.py $L
CLB_RAW_A=0 python tools/fwd_time.py $L
CLB_RAW_DBG=1 python tools/fwd_time.py $L
CLB_RAW_DBG=2 python tools/fwd_time.py $L
CLB_RAW_SLOTS=8 python tools/fwd_time.py $L
CLB_TRACE=1 python tools/fwd_time.py $L 2>&1 | grep -E "clb-trace\]  |fwd" | head -8
