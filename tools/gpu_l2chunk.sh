#!/bin/bash
# L2-chunked forward: whole-forward time per layer vs chunk budget; parity of the chunked path.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/l2chunk
O=gpurun_out/l2chunk
L=vgg16/conv1_2,vgg16/conv2_1,vgg16/conv2_2,vgg16/conv3_1,vgg16/conv3_2,vgg16/conv4_2,vgg16/conv5_1,alexnet/conv2,alexnet/conv3,alexnet/conv4,alexnet/conv5
for mb in 0 16 32 48 80; do
  env CLB_L2_CHUNK_MB=$mb timeout 300 python tools/fwd_time.py $L >> $O/fwd.txt 2>&1
done
CLB_L2_CHUNK_MB=32 timeout 900 python -m pytest tests -q -m gpu -x > $O/pytest_gpu_chunk32.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu_chunk32.txt
