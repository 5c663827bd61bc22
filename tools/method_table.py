"""Every GPU method on every BASELINE layer: the evidence behind the `auto` selector (the
reference times every method per layer too: bench.cpp:87-151, convlab_main.cpp:72-101; its
premise is that no method wins everywhere).

Per (layer, method): plan, pack weights, capture one forward (prepass + contraction + any
shift-add) into a CUDA graph and time R replays with CUDA events, L2 flushed before each (a
256 MiB write outside the events); median.  The direct loop nest is skipped where it would take
seconds (large C), methods whose workspace exceeds --max-ws-gb are skipped.

    python tools/method_table.py [--workloads ...] [--reps 5] > profiles/r02_method_table.json
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

import paper_1704_04428_b200 as clb
from paper_1704_04428_b200 import rng, workloads

ap = argparse.ArgumentParser()
ap.add_argument("--workloads", default="c1,alexnet-b1,alexnet,vgg16,googlenet,sweep,scale")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--max-ws-gb", type=float, default=24.0)
ap.add_argument("--precision", default="fp32")
args = ap.parse_args()

METHODS = ["kn2row-gpu", "kn2row-explicit-gpu", "kn2col-gpu", "kn2row-acc-gpu", "im2col-gpu", "direct-gpu"]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rows = []


def time_plan(plan, x, y, ws):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        plan.forward(x, y, ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.forward(x, y, ws)
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.reps + 1):
        flush.zero_()
        b, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        ts.append(b.elapsed_time(e))
    return statistics.median(ts[1:])


for wl in args.workloads.split(","):
    for li, layer in enumerate(workloads.workload(wl)):
        x, w = rng.make_problem(layer.batch, layer.channels, layer.height, layer.width, layer.kernel_count,
                                layer.kernel_size, seed=li)
        y = torch.empty((layer.batch, layer.kernel_count, layer.out_height, layer.out_width), device="cuda")
        with clb.ConvPlan(layer, "auto", args.precision) as p:
            auto = p.method
        res = {"workload": wl, "layer": layer.name, "batch": layer.batch, "gflop": layer.flops() / 1e9, "auto": auto,
               "ms": {}}
        for m in METHODS + (["conv1x1-gpu"] if layer.kernel_size == 1 else []):
            if m == "direct-gpu" and layer.channels > 16 and layer.flops() > 20e9:
                res["ms"][m] = None          # the generic loop nest: seconds at this size
                continue
            try:
                with clb.ConvPlan(layer, m, args.precision) as plan:
                    if plan.workspace_bytes() > args.max_ws_gb * 2 ** 30:
                        res["ms"][m] = None
                        continue
                    if plan.method != m:     # k == 1 routing (explicit / kn2col -> conv1x1)
                        res["ms"][m] = f"routed to {plan.method}"
                        continue
                    plan.set_weights(w)
                    ws = torch.empty(max(plan.workspace_bytes(), 4), dtype=torch.uint8, device="cuda")
                    res["ms"][m] = round(time_plan(plan, x, y, ws), 4)
                    del ws
            except Exception as e:   # unsupported shape for this method
                res["ms"][m] = f"error: {e}"[:120]
            torch.cuda.empty_cache()
        timed = {k: v for k, v in res["ms"].items() if isinstance(v, float)}
        res["best"] = min(timed, key=timed.get)
        res["auto_ms"] = timed.get(auto)
        res["best_over_auto"] = round(timed[res["best"]] / timed[auto], 3) if auto in timed else None
        rows.append(res)
        print(json.dumps(res), file=sys.stderr, flush=True)
        del x, w, y
        torch.cuda.empty_cache()

print(json.dumps({"precision": args.precision, "reps": args.reps,
                  "timing": "CUDA-graph replay of one whole forward, L2 flushed before each, median",
                  "rows": rows}, indent=1))
