#!/bin/bash
# A/B of the current library against tools/_ab/libconvlab_b200_before.so on the given layers
L=${1:-vgg16/conv1_1}
python tools/fwd_time.py $L
cp paper_1704_04428_b200/libconvlab_b200.so /tmp/after.so
cp tools/_ab/libconvlab_b200_before.so paper_1704_04428_b200/libconvlab_b200.so
python tools/fwd_time.py $L | sed 's/^/BEFORE /'
cp /tmp/after.so paper_1704_04428_b200/libconvlab_b200.so
