"""Runs ONE GPU case and prints a JSON line (used by tools/diag_gpu.py, one process per
case so a device fault cannot poison the others)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from oracle import oracle as O
import paper_1704_04428_b200 as clb

kind = sys.argv[1]
args = json.loads(sys.argv[2])
t0 = time.time()
if kind == "gemm":
    m, n, k, prec = args["m"], args["n"], args["k"], args.get("prec", "fp32")
    a = O.fill(m * k, 1).reshape(m, k)
    b = O.fill(k * n, 2).reshape(k, n)
    c = clb.gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), prec).cpu().numpy()
    ref = (a.astype(np.float64) @ b.astype(np.float64)).astype(np.float32)
    res = O.parity_metrics(c, ref)
else:
    N, C, H, W, M, k = (args[x] for x in ("N", "C", "H", "W", "M", "k"))
    method, prec = args["method"], args.get("prec", "fp32")
    x, w = O.make_problem(N, C, H, W, M, k, args.get("seed", 0))
    y = clb.run_method(method, torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), prec)
    y = y.cpu().numpy()
    ref = O.conv_batch(x, w)
    res = O.parity_metrics(y, ref)
res.update(kind=kind, args=args, secs=round(time.time() - t0, 2))
print("RESULT " + json.dumps(res))
