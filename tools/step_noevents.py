"""Diagnostic: the AlexNet bench step timed with and without the per-layer kernel events the
bench contract records around each contraction (those events sit between the prepass and the
contraction and break their programmatic-dependent-launch overlap).  Same plans, same L2 flush."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1704_04428_b200 as clb
from paper_1704_04428_b200 import _lib, rng, workloads

layers = workloads.workload("alexnet")
plans, xs, ys = [], [], []
for l in layers:
    x, w = rng.make_problem(l.batch, l.channels, l.height, l.width, l.kernel_count, l.kernel_size)
    p = clb.ConvPlan(l, "auto", "fp32")
    p.set_weights(w)
    plans.append(p)
    xs.append(x)
    ys.append(p.forward(x))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flops = workloads.total_flops(layers)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
kev = [(ev(), ev()) for _ in plans]
for b, e in kev:
    b.record(); e.record()
torch.cuda.synchronize()


def run(with_events, steps=30):
    tot = 0.0
    for _ in range(steps):
        flush.zero_()
        b, e = ev(), ev()
        b.record()
        for li, p in enumerate(plans):
            if with_events:
                _lib.lib().cl_conv_set_profile_events(p._h, kev[li][0].cuda_event, kev[li][1].cuda_event)
            p.forward(xs[li], ys[li])
            if with_events:
                _lib.lib().cl_conv_set_profile_events(p._h, None, None)
        e.record()
        torch.cuda.synchronize()
        tot += b.elapsed_time(e)
    return tot / steps


for _ in range(5):
    run(True, 3)
for rep in range(3):
    for we in (True, False):
        ms = run(we)
        print(f"kernel events {'on ' if we else 'off'}  {ms:.4f} ms/step  {flops / ms / 1e9:.1f} TFLOP/s", flush=True)
