"""tensor-core direct kernel: parity of a few shapes vs the oracle, and its time on VGG conv1_1 b32
against the CUDA-core kernel (run once with CLB_DIRECT_TC=0 for the latter)."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from oracle import oracle as O
import paper_1704_04428_b200 as clb
from paper_1704_04428_b200 import _lib, rng
for (N, C, H, W, M, k) in [(2, 3, 16, 16, 64, 3), (3, 3, 16, 16, 16, 3), (1, 1, 32, 32, 32, 5), (2, 2, 8, 16, 48, 3),
                           (2, 3, 224, 224, 64, 3)]:
    x, w = O.make_problem(N, C, H, W, M, k, 7 + C)
    with clb.ConvPlan(clb.LayerConfig("d", C, H, W, M, k, batch=N), "direct-gpu", "fp32") as plan:
        plan.set_weights(torch.from_numpy(w).cuda())
        y = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy()
        sp = plan.split
    m = O.parity_metrics(y, O.conv_batch(x, w))
    print((N, C, H, W, M, k), sp, "rel_l2 %.2e max_rel %.2e finite %s" % (m["rel_l2"], m["max_rel"], m["finite"]), flush=True)
layer = clb.LayerConfig("vgg16/conv1_1", 3, 224, 224, 64, 3, batch=32)
x, w = rng.make_problem(32, 3, 224, 224, 64, 3)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
with clb.ConvPlan(layer, "direct-gpu", "fp32") as plan:
    plan.set_weights(w)
    y = plan.forward(x)
    torch.cuda.synchronize()
    ts = []
    for _ in range(9):
        flush.zero_()
        kb, ke = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kb.record(); ke.record(); torch.cuda.synchronize()
        _lib.lib().cl_conv_set_profile_events(plan._h, kb.cuda_event, ke.cuda_event)
        plan.forward(x, y)
        torch.cuda.synchronize()
        ts.append(kb.elapsed_time(ke))
    _lib.lib().cl_conv_set_profile_events(plan._h, None, None)
    print("conv1_1 b32", plan.split, "kernel ms (median of 9):", sorted(ts)[4], flush=True)
