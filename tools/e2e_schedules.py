"""Host<->device pipeline schedules for the AlexNet e2e step, prototyped with torch streams
around the library's device-buffer forward (cl_conv_forward via plan.forward on sub-batch
views is not available, so each chunk is its own plan call on a chunk-sized plan).

Per step: 4 layers, pinned host input -> device -> conv -> device -> pinned host output.
Schedules (chunks of 16 images per layer):
  per_layer   : each layer its own H2D / D2H stream, all H2D enqueued first (library default)
  shared      : one H2D and one D2H stream in call order
  d2h_prio    : shared, with the D2H stream at high priority and compute at low
  interleave  : H2D chunks of the next layer enqueued only after the current layer's compute
                of the same chunk index (keeps H2D from running far ahead of compute)
Prints ms per step and the e2e TFLOP/s for each schedule."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1704_04428_b200 as clb
from paper_1704_04428_b200 import rng, workloads

CH = 8
layers = workloads.workload("alexnet")
dev = torch.device("cuda")
plans, hx, hy, dx, dy = [], [], [], [], []
for l in layers:
    x, w = rng.make_problem(l.batch, l.channels, l.height, l.width, l.kernel_count, l.kernel_size)
    sub = clb.LayerConfig(l.name, l.channels, l.height, l.width, l.kernel_count, l.kernel_size, batch=l.batch // CH)
    p = clb.ConvPlan(sub, "auto", "fp32")
    p.set_weights(w)
    plans.append(p)
    hx.append(x.cpu().pin_memory())
    yshape = (l.batch,) + tuple(p.output_shape()[1:])
    hy.append(torch.empty(yshape).pin_memory())
    dx.append(torch.empty_like(x))
    dy.append(torch.empty(yshape, device=dev))
flops = workloads.total_flops(layers)


def chunks(t):
    return t.chunk(CH, 0)


def run(schedule, steps=6):
    comp = torch.cuda.Stream(priority=0)
    if schedule == "per_layer":
        s_in = [torch.cuda.Stream() for _ in layers]
        s_out = [torch.cuda.Stream() for _ in layers]
    else:
        hi = -1 if schedule == "d2h_prio" else 0
        a, b = torch.cuda.Stream(), torch.cuda.Stream(priority=hi)
        s_in, s_out = [a] * len(layers), [b] * len(layers)
    times = []
    for it in range(steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev_in = [[torch.cuda.Event() for _ in range(CH)] for _ in layers]
        ev_c = [[torch.cuda.Event() for _ in range(CH)] for _ in layers]
        if schedule != "interleave":
            for li in range(len(layers)):
                with torch.cuda.stream(s_in[li]):
                    for c, (h, d) in enumerate(zip(chunks(hx[li]), chunks(dx[li]))):
                        d.copy_(h, non_blocking=True)
                        ev_in[li][c].record(s_in[li])
        for li, p in enumerate(plans):
            if schedule == "interleave":
                with torch.cuda.stream(s_in[li]):
                    for c, (h, d) in enumerate(zip(chunks(hx[li]), chunks(dx[li]))):
                        d.copy_(h, non_blocking=True)
                        ev_in[li][c].record(s_in[li])
            for c, (xc, yc) in enumerate(zip(chunks(dx[li]), chunks(dy[li]))):
                comp.wait_event(ev_in[li][c])
                with torch.cuda.stream(comp):
                    p.forward(xc, yc)
                ev_c[li][c].record(comp)
                s_out[li].wait_event(ev_c[li][c])
                with torch.cuda.stream(s_out[li]):
                    hy[li].chunk(CH, 0)[c].copy_(yc, non_blocking=True)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    ms = sorted(times[1:])[len(times[1:]) // 2] * 1e3
    print(f"{schedule:12s} {ms:7.3f} ms/step  e2e {flops / ms / 1e9:6.2f} TFLOP/s", flush=True)


for rep in range(2):
    for s in ("per_layer", "shared", "d2h_prio", "interleave"):
        run(s)
