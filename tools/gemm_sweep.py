"""Steady-state tcgen05 engine throughput vs N (and CTA group): large M, long K, many tiles."""
import os, sys, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1704_04428_b200 as clb

M, K = 148 * 256 * 4, 2304
res = []
for N in (64, 128, 192, 256, 384, 512):
    a = torch.rand(M, K, device="cuda") - 0.5
    b = torch.rand(K, N, device="cuda") - 0.5
    c = clb.gemm(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        clb.gemm(a, b, out=c)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    tf = 2 * M * N * K / ms / 1e9
    res.append({"N": N, "cg": os.environ.get("CLB_CTA_GROUP", "auto"), "ms": round(ms, 3), "TFLOPs": round(tf, 1),
                "frac_of_277.8": round(tf / 277.8, 3)})
    print(json.dumps(res[-1]), flush=True)
