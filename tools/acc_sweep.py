"""Accuracy vs K of the 3xTF32 contraction (accumulator rounding study)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from oracle import oracle as O
import paper_1704_04428_b200 as clb
for k in (16, 64, 256, 1024, 4096, 16384):
    m, n = 256, 256
    a = O.fill(m * k, 1).reshape(m, k); b = O.fill(k * n, 2).reshape(k, n)
    ref = a.astype(np.float64) @ b.astype(np.float64)
    c = clb.gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
    cf = (a @ b)  # numpy fp32 (pairwise/blas) for scale
    e = O.parity_metrics(c, ref); ef = O.parity_metrics(cf, ref)
    bias = float(np.mean((c - ref) / np.abs(ref).max()))
    print(f"K={k:6d} gpu rel_l2={e['rel_l2']:.2e} max_rel={e['max_rel']:.2e} bias={bias:+.2e} | numpy-fp32 rel_l2={ef['rel_l2']:.2e}")
