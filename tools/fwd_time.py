"""Whole-forward time (prepass + contraction, events around plan.forward) of selected layers
under the current CLB_* environment, L2 flushed before each timed call, median of 9.
Driven by tools/gpu_*.sh scripts that re-run it under different knob settings."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1704_04428_b200 as clb
from paper_1704_04428_b200 import rng, workloads

layers = sys.argv[1].split(",")
batch = int(sys.argv[sys.argv.index("--batch") + 1]) if "--batch" in sys.argv else None
tag = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("CLB_"))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name in layers:
    group = name.split("/")[0]
    layer = [l for l in workloads.workload(group, batch) if l.name in (name, group)][0]
    x, w = rng.make_problem(layer.batch, layer.channels, layer.height, layer.width, layer.kernel_count,
                            layer.kernel_size)
    with clb.ConvPlan(layer, "auto", "fp32") as plan:
        plan.set_weights(w)
        y = plan.forward(x)
        torch.cuda.synchronize()
        ts = []
        for _ in range(9):
            flush.zero_()
            b, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            b.record()
            plan.forward(x, y)
            e.record()
            torch.cuda.synchronize()
            ts.append(b.elapsed_time(e))
        launches = plan.launch_count()
    ts.sort()
    ms = ts[len(ts) // 2]
    print(f"{name:16s} {tag:40s} fwd {ms:7.3f} ms {layer.flops() / ms / 1e9:7.1f} TF launches {launches}", flush=True)
