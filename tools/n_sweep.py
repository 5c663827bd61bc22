"""Steady-state tcgen05 conv-kernel throughput vs output channels M (= tile N) and CTA group,
timed with the library's profile events around the contraction only."""
import os, sys, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1704_04428_b200 as clb
from paper_1704_04428_b200 import _lib, rng

CASES = [(64, 256, 56, m) for m in (64, 128, 192, 256, 384, 512)] + [(128, 256, 13, 384), (128, 384, 13, 256)]
if len(sys.argv) > 1:
    CASES = [tuple(int(v) for v in c.split(",")) for c in sys.argv[1:]]
for (N, C, H, M) in CASES:
    layer = clb.LayerConfig("s", C, H, H, M, 3, batch=N)
    x, w = rng.make_problem(N, C, H, H, M, 3)
    with clb.ConvPlan(layer, "kn2row-gpu") as plan:
        plan.set_weights(w)
        y = plan.forward(x)
        ws = torch.empty(plan.workspace_bytes(), dtype=torch.uint8, device="cuda")
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
        for b, e in evs:
            b.record(); e.record()
        torch.cuda.synchronize()
        for b, e in evs:
            _lib.lib().cl_conv_set_profile_events(plan._h, b.cuda_event, e.cuda_event)
            plan.forward(x, y, ws)
        torch.cuda.synchronize()
        ms = min(b.elapsed_time(e) for b, e in evs)
    tf = layer.flops() / ms / 1e9
    print(json.dumps({"N": N, "C": C, "HW": H, "M": M, "cg": os.environ.get("CLB_CTA_GROUP", "auto"),
                      "kernel_ms": round(ms, 3), "TFLOPs": round(tf, 1), "frac": round(tf / 277.8, 3)}), flush=True)
