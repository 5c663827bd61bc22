"""Per-layer report over all BASELINE configs.

GPU: every layer of every workload through ConvPlan("auto", fp32), dominant-kernel time from
the library's profile events (median of R runs, L2 flushed before each), plus the full
forward time (prepass included).  Parity: image 0 (and N-1) checked against the oracle.
CPU: the reference's own kn2row and im2col (oracle/_ref, convlab::run_method with
GemmBackend::parallel(T), T = host threads) on one image, batch-N time = N x per-image time.

    python tools/report.py [--workloads c1,alexnet,...] [--no-cpu] > profiles/rNN_report.json
"""
import argparse
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import paper_1704_04428_b200 as clb
from paper_1704_04428_b200 import _lib, rng, workloads
from oracle import oracle as O

import os
# fp32-faithful peak of each plan's operand format: measured bf16 burst / 3 for the fp16 split
# (3 f16 MMAs per product), / 4 for the mixed split (4 tf32-MMA slots per 16 K-elements), / 6 for
# CLB_SPLIT=3xtf32; the direct kernel (CUDA cores) is reported against the mixed figure
_pk = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())
SPLIT_PEAK = {"3xf16": float(_pk["bf16_tflops"]) / 3, "mixed": float(_pk["bf16_tflops"]) / 4,
              "3xtf32": float(_pk["bf16_tflops"]) / 6, "fp32-fma": float(_pk["bf16_tflops"]) / 4}
HBM = float(_pk["hbm_gbs"])   # GB/s measured

ap = argparse.ArgumentParser()
ap.add_argument("--workloads", default="c1,alexnet-b1,alexnet,vgg16,googlenet,sweep,scale")
ap.add_argument("--reps", type=int, default=7)
ap.add_argument("--no-cpu", action="store_true")
ap.add_argument("--cpu-runs", type=int, default=2)
args = ap.parse_args()

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
threads = O.host_threads()
rows = []
for wl in args.workloads.split(","):
    for li, layer in enumerate(workloads.workload(wl)):
        x, w = rng.make_problem(layer.batch, layer.channels, layer.height, layer.width, layer.kernel_count,
                                layer.kernel_size, seed=li)
        with clb.ConvPlan(layer, "auto", "fp32") as plan:
            plan.set_weights(w)
            ws = torch.empty(max(plan.workspace_bytes(), 4), dtype=torch.uint8, device="cuda")
            y = plan.forward(x, None, ws)
            torch.cuda.synchronize()
            kt, ft = [], []
            for _ in range(args.reps):
                flush.zero_()
                kb, ke = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                fb, fe = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                kb.record(); ke.record(); torch.cuda.synchronize()
                _lib.lib().cl_conv_set_profile_events(plan._h, kb.cuda_event, ke.cuda_event)
                fb.record()
                plan.forward(x, y, ws)
                fe.record()
                torch.cuda.synchronize()
                kt.append(kb.elapsed_time(ke))
                ft.append(fb.elapsed_time(fe))
            _lib.lib().cl_conv_set_profile_events(plan._h, None, None)
            method = plan.method
            split = plan.split
            # back-to-back forwards replayed from a CUDA graph: no host launch latency in the
            # measurement (what a serving loop / captured network sees); L2 stays warm
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                plan.forward(x, y, ws)        # warm the stream-local state before capture
                torch.cuda.synchronize()
                with torch.cuda.graph(g, stream=s):
                    plan.forward(x, y, ws)
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            gb, ge = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps_g = 20
            gb.record()
            for _ in range(reps_g):
                g.replay()
            ge.record()
            torch.cuda.synchronize()
            graph_ms = gb.elapsed_time(ge) / reps_g
        picks = sorted({0, layer.batch - 1})
        ref = O.conv_batch(x[picks].cpu().numpy(), w.cpu().numpy())
        par = O.parity_metrics(y[picks].cpu().numpy(), ref)
        k_ms, f_ms = statistics.median(kt), statistics.median(ft)
        fl = layer.flops()
        ai = fl / layer.algorithmic_bytes()
        PEAK_3X = SPLIT_PEAK[split]
        bound = min(PEAK_3X, ai * HBM / 1000.0)
        row = {"workload": wl, "layer": layer.name, "N": layer.batch, "C": layer.channels, "HW": layer.height,
               "M": layer.kernel_count, "k": layer.kernel_size, "method": method, "split": split, "peak_tflops": PEAK_3X, "gflop": fl / 1e9,
               "kernel_ms": k_ms, "forward_ms": f_ms, "kernel_tflops": fl / k_ms / 1e9,
               "forward_tflops": fl / f_ms / 1e9, "graph_forward_ms": graph_ms,
               "graph_forward_tflops": fl / graph_ms / 1e9, "frac_of_fp32_peak": fl / k_ms / 1e9 / PEAK_3X,
               "roofline_tflops": bound, "frac_of_layer_roofline": fl / k_ms / 1e9 / bound,
               "rel_l2": par["rel_l2"], "max_rel": par["max_rel"], "allclose": par["allclose"]}
        if not args.no_cpu and O.ref_available():
            xi = np.ascontiguousarray(x[0].cpu().numpy())
            wi = w.cpu().numpy()
            for m in ("kn2row", "im2col"):
                O.ref_run_method(m, xi, wi, threads)   # warm-up
                t = []
                for _ in range(args.cpu_runs):
                    t0 = time.perf_counter()
                    O.ref_run_method(m, xi, wi, threads)
                    t.append(time.perf_counter() - t0)
                per_img = min(t)
                row[f"cpu_{m}_s_per_image"] = per_img
                row[f"cpu_{m}_tflops"] = fl / layer.batch / per_img / 1e12
            # the reference's single-core backend (GemmBackend::blocked), for the thread scaling
            # SURVEY 8(d) asks to report beside parallel(T)
            t0 = time.perf_counter()
            O.ref_run_method("kn2row", xi, wi, 0)
            one = time.perf_counter() - t0
            row["cpu_kn2row_1core_s_per_image"] = one
            row["cpu_kn2row_1core_tflops"] = fl / layer.batch / one / 1e12
            row["cpu_kn2row_thread_scaling"] = one / row["cpu_kn2row_s_per_image"]
            row["cpu_threads"] = threads
        rows.append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
        del x, w, y, ws
        torch.cuda.empty_cache()
print(json.dumps({"peak_fp32_faithful_tflops": SPLIT_PEAK, "fp32_split": os.environ.get("CLB_SPLIT", "auto"),
                  "hbm_gbs": HBM, "rows": rows}, indent=1))
