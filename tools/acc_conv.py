"""fp32-faithful accuracy of the implicit kn2row kernel vs K = 9 C, against an fp64 reference,
for the operand split in force (CLB_SPLIT=3xf16 / mixed / 3xtf32); the reference's own fp32
conv_mcmk_sum (oracle) beside it for scale.  One line per C."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from oracle import oracle as O
import paper_1704_04428_b200 as clb


def conv64(x, w):   # x [C,H,W], w [M,k,k,C] -> [M,H,W] in float64, zero padding k//2
    C, H, W = x.shape
    M, k, _, _ = w.shape
    p = k // 2
    xp = np.zeros((C, H + 2 * p, W + 2 * p))
    xp[:, p:p + H, p:p + W] = x
    out = np.zeros((M, H, W))
    for i in range(k):
        for j in range(k):
            out += np.tensordot(w[:, i, j, :].astype(np.float64), xp[:, i:i + H, j:j + W], axes=([1], [0]))
    return out


split = os.environ.get("CLB_SPLIT", "auto")
for C in (32, 128, 512, 2048, 4096):
    H = W = 8
    M, k = 64, 3
    x, w = O.make_problem(1, C, H, W, M, k, 11 + C)
    ref = conv64(x[0], w)
    layer = clb.LayerConfig("acc", C, H, W, M, k, batch=1)
    with clb.ConvPlan(layer, "kn2row-gpu", "fp32") as plan:
        plan.set_weights(torch.from_numpy(w).cuda())
        y = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy()[0]
        used = plan.split
    yo = O.conv_batch(x, w)[0]
    e = O.parity_metrics(y, ref)
    eo = O.parity_metrics(yo, ref)
    print(f"split={split:6s} ({used}) K={9 * C:6d} gpu rel_l2={e['rel_l2']:.2e} max_rel={e['max_rel']:.2e} | "
          f"reference fp32 conv_mcmk_sum rel_l2={eo['rel_l2']:.2e} max_rel={eo['max_rel']:.2e}", flush=True)
