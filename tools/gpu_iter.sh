#!/bin/bash
# One iteration: full GPU parity suite, traces, per-layer report for VGG16 + AlexNet, bench.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
tail -2 gpurun_out/pytest_gpu.txt
./tools/trace_layers.sh
timeout 600 python tools/report.py --workloads vgg16,alexnet --no-cpu --reps 5 > gpurun_out/rep.txt 2>&1
python tools/rep_table.py gpurun_out/rep.txt
: <<'PY'
import json
for l in open("gpurun_out/rep.txt"):
    l = l.strip()
    if l.startswith("{"):
        d = json.loads(l)
        if "layer" in d and "kernel_ms" in d:
            print(f'{d["layer"]:18s} {d["method"]:12s} {d["kernel_ms"]:8.3f} ms  {d["kernel_tflops"]:7.1f} TF  frac {d["frac_of_layer_roofline"]:.2f}')
PY
timeout 600 python bench.py --no-cpu-baseline --steps 30 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; cut -c1-300 gpurun_out/bench.json
timeout 600 python bench.py --workload vgg16 --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/bench_vgg.json 2> gpurun_out/bench_vgg.err; cut -c1-300 gpurun_out/bench_vgg.json
