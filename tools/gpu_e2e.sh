#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python tools/pcie_probe.py > gpurun_out/pcie.txt 2>&1
for c in 1 2 4 8; do
CLB_HOST_CHUNKS=$c timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_alex_c$c.json 2>&1
CLB_HOST_CHUNKS=$c timeout 600 python bench.py --workload vgg16 --steps 5 --warmup 2 --no-cpu-baseline --e2e-steps 3 > gpurun_out/e2e_vgg_c$c.json 2>&1
done
