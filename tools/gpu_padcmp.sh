#!/bin/bash
# Tap-shared padded-row mode on/off: GPU tests + VGG16/AlexNet per-layer report for each.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
tail -2 gpurun_out/pytest_gpu.txt
for pr in 0 1; do
  echo "== CLB_PADDED_ROWS=$pr"
  CLB_PADDED_ROWS=$pr timeout 600 python tools/report.py --workloads vgg16,alexnet,c1 --no-cpu --reps 5 > gpurun_out/rep_pr$pr.txt 2>&1
  python tools/rep_table.py gpurun_out/rep_pr$pr.txt
done
./tools/trace_layers.sh; grep -v "^ok" gpurun_out/trace.txt
