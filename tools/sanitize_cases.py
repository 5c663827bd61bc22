"""Small cases over every kernel path, for compute-sanitizer memcheck (one tool per run)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1704_04428_b200 as clb
from paper_1704_04428_b200 import rng

cases = [("kn2row-gpu", (2, 16, 13, 13, 32, 3)), ("kn2row-gpu", (4, 64, 28, 28, 256, 3)),   # CG1 / CG2 + stream-K
         ("kn2row-explicit-gpu", (2, 8, 9, 9, 16, 3)), ("kn2col-gpu", (2, 8, 9, 9, 16, 5)),
         ("kn2row-acc-gpu", (2, 8, 9, 9, 16, 3)), ("im2col-gpu", (2, 3, 12, 12, 16, 3)),
         ("direct-gpu", (2, 3, 20, 20, 16, 3)), ("conv1x1-gpu", (2, 24, 7, 7, 40, 1)),
         ("kn2row-gpu", (3, 32, 19, 21, 48, 5)), ("kn2row-gpu", (2, 64, 30, 30, 64, 3))]   # tap-stacked k = 5 / 3 (CLB_STACKED)
for method, (N, C, H, W, M, k) in cases:
    for prec in ("fp32", "bf16"):
        if method == "direct-gpu" and prec == "bf16":
            continue
        x, w = rng.make_problem(N, C, H, W, M, k)
        y = clb.run_method(method, x, w, prec)
        torch.cuda.synchronize()
        print(method, prec, tuple(y.shape), flush=True)
a = torch.rand(70, 33, device="cuda"); b = torch.rand(33, 50, device="cuda")
clb.gemm(a, b); torch.cuda.synchronize(); print("gemm ok")
