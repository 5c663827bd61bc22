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
# round-2 paths: padded rows + two sub-tiles (small N), tensor-core direct (auto, C = 3, 16-byte
# aligned), channels-last, the host-buffer pipeline, the chained step.  Run once more under
# CLB_SPLIT=3xf16 for the fp16 split with its speculative prepass / fixup kernels.
for (N, C, H, W, M, k) in [(2, 64, 20, 20, 64, 3), (2, 3, 16, 16, 64, 3), (2, 32, 14, 14, 128, 3)]:
    x, w = rng.make_problem(N, C, H, W, M, k)
    layer = clb.LayerConfig("san", C, H, W, M, k, batch=N)
    with clb.ConvPlan(layer, "auto", "fp32") as plan:
        plan.set_weights(w)
        y = plan.forward(x)
        y = plan.forward(x * 1024.0)            # fp16 split: an exponent miss -> the fixup kernel
        if plan.method != "direct-gpu":
            plan.forward(x.permute(0, 2, 3, 1).contiguous(), layout="nhwc")
        hx, hy = x.cpu().pin_memory(), torch.empty(plan.output_shape()).pin_memory()
        st = torch.cuda.Stream()
        plan.forward_host_async(hx, hy, st)
        st.synchronize()
        torch.cuda.synchronize()
        print("plan", plan.method, (N, C, H, W, M, k), flush=True)
xa, wa = rng.make_problem(2, 32, 14, 14, 64, 3)
xb, wb = rng.make_problem(2, 64, 14, 14, 32, 3)
with clb.ConvPlan(clb.LayerConfig("a", 32, 14, 14, 64, 3, batch=2), "kn2row-gpu", "fp32") as pa, \
        clb.ConvPlan(clb.LayerConfig("b", 64, 14, 14, 32, 3, batch=2), "kn2row-gpu", "fp32") as pb:
    pa.set_weights(wa); pb.set_weights(wb)
    ya, yb = torch.empty(pa.output_shape(), device="cuda"), torch.empty(pb.output_shape(), device="cuda")
    import os
    clb.forward_chain([pa, pb], [xa, xb], [ya, yb])
    torch.cuda.synchronize(); print("chain ok", flush=True)
a = torch.rand(70, 33, device="cuda"); b = torch.rand(33, 50, device="cuda")
clb.gemm(a, b); torch.cuda.synchronize(); print("gemm ok")
