#!/usr/bin/env python3
"""Benchmark of the B200 kn2row hot path -- one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload alexnet] [--method auto] [--precision fp32]

Metric (BASELINE.json): per-layer effective TFLOP/s = 2 N M C k^2 P Q / time, here summed
over the workload's layers: one STEP is one forward pass of every layer of the workload
(default: configs[1], the AlexNet stride-1 conv stack at batch 128 per GPU) on synthetic
uniform[-1,1) data from the reference generator (tensor.cpp:104-134), weights pre-packed
once outside the timed region (the reference re-packs per call; the north star treats
weights as static -- stated in DESIGN.md).

Timing: W untimed warm-up steps, then exactly K steps between a barrier +
cuda.synchronize on both sides; every step is bracketed by CUDA events on the launching
stream and L2 is flushed (256 MiB write, untimed) before each step.  Under torchrun each
rank runs its own batch (weak scaling, no data-path collective) and the job time is the
MAX over ranks.  `e2e` repeats the workload through the host-buffer C-ABI call
(cl_conv_forward_host: pinned H2D + forward + D2H).

--impl reference times the reference's own CPU kn2row (oracle/_ref = the unmodified
reference core compiled from /root/reference) with all host threads, on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
TRAFFIC_FILE = ROOT / "profiles" / "ncu_traffic.json"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="alexnet")
    ap.add_argument("--batch", type=int, default=None, help="override the per-GPU batch")
    ap.add_argument("--method", default="auto")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "tf32", "bf16"],
                    help="fp32 = fp32-faithful (rel-L2 <= 1e-5; operand split per CLB_SPLIT: mixed "
                         "(default) or 3xtf32); tf32 / bf16 = the 1e-2 fast modes")
    ap.add_argument("--layout", default="nchw", choices=["nchw", "nhwc"],
                    help="device tensors NCHW (the reference interface, default) or channels-last "
                         "(cl_conv_forward_nhwc; the e2e leg stays NCHW)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="target CPU-baseline work")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--e2e-sync", action="store_true",
                    help="e2e through the synchronous cl_conv_forward_host (one layer at a time)")
    ap.add_argument("--per-layer", action="store_true", help="add a per-layer table to the JSON line")
    return ap.parse_args()


NOMINAL_BF16 = 2250.0   # dense bf16 TFLOP/s, B200 nominal (B200_PROFILING.md, context only)


def fp32_split():
    """The fp32-faithful operand split the library uses (same switch as api.cu planes_for):
    'mixed' = hi*Hi in two tf32 MMAs + the two cross terms in one bf16 K=16 MMA each (4
    tf32-MMA slots per 16 K-elements); '3xtf32' = the classic split (6 slots)."""
    return "3xtf32" if os.environ.get("CLB_SPLIT") == "3xtf32" else "mixed"


def tensor_factor(precision):
    """Effective-TFLOP/s per tf32 TFLOP/s of the tensor pipe for each precision mode."""
    if precision == "fp32":
        return 1.0 / 3.0 if fp32_split() == "3xtf32" else 0.5
    return {"tf32": 1.0, "bf16": 2.0}[precision]


def mma_peak_for(precision):
    """Our own kind::tf32 MMA peak (tools/mma_probe.cu, committed under profiles/), in the
    precision's effective units (tensor_factor)."""
    f = Path(__file__).resolve().parent / "profiles" / "tf32_mma_peak.json"
    if not f.exists():
        return None
    return json.loads(f.read_text())["tf32_mma_peak_tflops"] * tensor_factor(precision)


def peaks():
    try:
        p = json.loads(PEAKS_FILE.read_text())
        return {"bf16": float(p["bf16_tflops"]), "bf16_sustained": float(p["bf16_tflops_sustained"]),
                "hbm": float(p["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"bf16": 1590.0, "bf16_sustained": 1400.0, "hbm": 6650.0, "source": "fallback (B200_PROFILING.md)"}


# ------------------------------------------------------------------------- clocks ----
class ClockSampler:
    """SM clock / power / throttle reasons sampled DURING the timed region (B200_PROFILING.md
    clocks line): NVML polled every 5 ms from a thread (nvidia-smi -lms as fallback)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples = []          # (t, sm_mhz, max_mhz, power_w, reasons_bitmask)
        self.stop_flag = False
        self.thread = None
        self.proc = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def poll():
                while not self.stop_flag:
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((time.time(), sm, mx, pw, rs))
                    except Exception:
                        pass
                    time.sleep(0.005)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            pass
        try:   # fallback: nvidia-smi
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read_smi, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read_smi(self):
        for line in self.proc.stdout:
            p = [x.strip() for x in line.split(",")]
            try:
                self.samples.append((time.time(), float(p[0]), float(p[1]), float(p[2]), int(p[3], 16)))
            except (ValueError, IndexError):
                pass

    def stop(self):
        self.stop_flag = True
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self, t0: float, t1: float):
        win = [s for s in self.samples if t0 <= s[0] <= t1]
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({name for s in win for name, bit in self.REASONS.items() if s[4] & bit})
        return {"sm_mhz": statistics.median(s[1] for s in win), "sm_max_mhz": win[0][2],
                "power_w_max": max(s[3] for s in win), "reasons": reasons, "samples": len(win)}


# ------------------------------------------------------------------- CPU baseline ----
def cpu_reference_sample(layers, seconds: float, threads: int, seed: int = 0):
    """Times the reference's CPU kn2row (oracle/_ref, convlab::run_method with
    GemmBackend::parallel(threads)) on ONE image of each layer, repeating the whole sample
    until ~`seconds` of CPU work.  Returns (TFLOP/s, detail)."""
    import numpy as np
    from oracle import oracle as O

    if not O.ref_available():
        raise RuntimeError("oracle/_ref (compiled reference) is not available")
    data = []
    for li, l in enumerate(layers):
        x, w = O.make_problem(1, l.channels, l.height, l.width, l.kernel_count, l.kernel_size, seed + li)
        data.append((l, np.ascontiguousarray(x[0]), w))
    one_image_flops = sum(l.flops() // l.batch for l in layers)
    for l, x, w in data:  # warm-up (the reference benchmark()'s untimed run, bench.cpp:115-118)
        O.ref_run_method("kn2row", x, w, threads)
    reps, spent = 0, 0.0
    while reps < 2 or (spent < seconds and reps < 1000):
        t0 = time.perf_counter()
        for l, x, w in data:
            O.ref_run_method("kn2row", x, w, threads)
        spent += time.perf_counter() - t0
        reps += 1
    per_pass = spent / reps
    return one_image_flops / per_pass / 1e12, {
        "passes": reps, "seconds": round(spent, 3), "per_image_pass_s": per_pass,
        "one_image_gflop": one_image_flops / 1e9}


def run_reference_arm(args, info, layers, total_flops_per_step):
    if info.rank != 0:
        return 0
    from oracle import oracle as O
    threads = O.host_threads()
    cfg = {"workload": args.workload, "layers": [l.name for l in layers], "per_gpu_batch": layers[0].batch,
           "method": "kn2row (reference CPU)", "backend": f"parallel({threads})"}
    try:
        # each step: one image through every layer (bounded sample of the workload)
        import numpy as np
        data = []
        for li, l in enumerate(layers):
            x, w = O.make_problem(1, l.channels, l.height, l.width, l.kernel_count, l.kernel_size, li)
            data.append((np.ascontiguousarray(x[0]), w))
        sample_flops = sum(l.flops() // l.batch for l in layers)
        for _ in range(args.warmup):
            for x, w in data:
                O.ref_run_method("kn2row", x, w, threads)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            for x, w in data:
                O.ref_run_method("kn2row", x, w, threads)
        dt = time.perf_counter() - t0
    except Exception as e:  # pragma: no cover
        print(json.dumps({"impl": "reference", "unavailable": f"reference CPU path failed: {e}"}))
        return 0
    value = sample_flops * args.steps / dt / 1e12
    sample = (f"1 image of each of the {len(layers)} {args.workload} layers per step "
              f"(reference convlab::run_method(Kn2row), GemmBackend::parallel({threads})); "
              f"the reference has no batch dim, batch-N time = N x per-image time")
    print(json.dumps({
        "impl": "reference", "metric": "effective TFLOP/s (2*N*M*C*k^2*P*Q / time), summed over the workload layers",
        "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (reference generator, uniform[-1,1))", "config": cfg,
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))
    return 0


# ------------------------------------------------------------------------- our arm ----
def main():
    args = parse_args()
    from paper_1704_04428_b200 import dist, workloads

    info = dist.from_env()
    layers = workloads.workload(args.workload, args.batch)
    if args.impl == "reference":
        return run_reference_arm(args, info, layers, workloads.total_flops(layers))

    import torch

    import paper_1704_04428_b200 as clb
    from paper_1704_04428_b200 import _lib, rng

    info = dist.init("nccl")
    dev = info.local_rank
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    pk = peaks()

    # ---- setup (untimed): plans, packed weights, resident inputs/outputs/workspaces ----
    plans, xs, ys, wss, evs = [], [], [], [], []
    for li, l in enumerate(layers):
        plan = clb.ConvPlan(l, args.method, args.precision, dev)
        if args.layout == "nhwc" and plan.method not in ("kn2row-gpu", "conv1x1-gpu", "kn2row-acc-gpu"):
            # channels-last is served by the implicit kernel only: plan that one explicitly
            plan.close()
            plan = clb.ConvPlan(l, "kn2row-gpu" if l.kernel_size > 1 else "conv1x1-gpu", args.precision, dev)
        x = torch.empty((l.batch, l.channels, l.height, l.width), device=dev, dtype=torch.float32)
        w = torch.empty((l.kernel_count, l.kernel_size, l.kernel_size, l.channels), device=dev, dtype=torch.float32)
        img = l.channels * l.height * l.width
        rng.fill_uniform(x, rng.split(li, 0), dist.image_offset(info.rank, l.batch, img))
        rng.fill_uniform(w, rng.split(li, 1))
        plan.set_weights(w)
        ws = torch.empty(max(plan.workspace_bytes(), 4), device=dev, dtype=torch.uint8)
        y = torch.empty(plan.output_shape(), device=dev, dtype=torch.float32)
        if args.layout == "nhwc":   # same values, channels-last storage
            x = x.permute(0, 2, 3, 1).contiguous()
            y = y.permute(0, 2, 3, 1).contiguous()
        plans.append(plan)
        xs.append(x)
        ys.append(y)
        wss.append(ws)
    # L2 flush between timed steps: a write larger than the 126 MB L2 (MiB, CLB_FLUSH_MB to vary)
    flush_mb = int(os.environ.get("CLB_FLUSH_MB", "256"))
    flush = torch.empty(flush_mb * 1024 * 1024, device=dev, dtype=torch.uint8)
    flops_step = workloads.total_flops(layers)

    def step(record_kernel=None):
        for li, plan in enumerate(plans):
            if record_kernel is not None:
                b, e = record_kernel[li]
                _lib.lib().cl_conv_set_profile_events(plan._h, b.cuda_event, e.cuda_event)
            plan.forward(xs[li], ys[li], wss[li], layout=args.layout)
            if record_kernel is not None:
                _lib.lib().cl_conv_set_profile_events(plan._h, None, None)

    sampler = ClockSampler(int(os.environ.get("CLB_SMI_INDEX", dev)))
    sampler.start()
    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    launches_per_step = sum(p.launch_count() for p in plans)

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    st_b = [ev() for _ in range(args.steps)]
    st_e = [ev() for _ in range(args.steps)]
    k_ev = [[(ev(), ev()) for _ in plans] for _ in range(args.steps)]
    for pair in (p for row in k_ev for p in row):   # torch creates CUDA events lazily:
        pair[0].record(stream)                       # record once so .cuda_event is a live
        pair[1].record(stream)                       # handle the library can record into
    torch.cuda.synchronize()

    dist.barrier(info)
    torch.cuda.synchronize()
    t_wall0 = time.time()
    for i in range(args.steps):
        flush.zero_()                       # L2 flush, outside the step events
        st_b[i].record(stream)
        step(k_ev[i])
        st_e[i].record(stream)
    torch.cuda.synchronize()
    dist.barrier(info)
    t_wall1 = time.time()
    sampler.stop()

    step_ms = [st_b[i].elapsed_time(st_e[i]) for i in range(args.steps)]
    if os.environ.get("CLB_BENCH_STEP_MS"):        # diagnostics: per-step device times
        print(json.dumps({"step_ms": [round(v, 4) for v in step_ms]}), file=sys.stderr)
    local_ms = sum(step_ms)
    kern_ms = [sum(k_ev[i][li][0].elapsed_time(k_ev[i][li][1]) for i in range(args.steps)) / args.steps
               for li in range(len(plans))]
    job_ms = dist.max_over_ranks(local_ms, info, device=dev)
    total_flops = flops_step * args.steps * info.world
    value = total_flops / (job_ms * 1e-3) / 1e12

    # ---- e2e through the host-buffer C-ABI call ----------------------------------------
    hx = [x.cpu().pin_memory() for x in xs]
    hy = [torch.empty(y.shape, dtype=torch.float32).pin_memory() for y in ys]
    for li, p in enumerate(plans):
        p.forward_host(hx[li], hy[li])
    e2e_steps = max(1, min(args.e2e_steps, args.steps))
    dist.barrier(info)
    torch.cuda.synchronize()
    eb, ee = ev(), ev()
    eb.record(stream)
    for _ in range(e2e_steps):
        if args.e2e_sync:
            for li, p in enumerate(plans):
                p.forward_host(hx[li], hy[li])
        else:
            # the layers are independent: enqueue all four host-buffer calls, then wait for the
            # step's outputs (every H2D / D2H byte of the step is inside the timed region)
            for li, p in enumerate(plans):
                p.forward_host_async(hx[li], hy[li], stream)
            stream.synchronize()
    ee.record(stream)
    torch.cuda.synchronize()
    e2e_ms = dist.max_over_ranks(eb.elapsed_time(ee), info, device=dev)
    e2e_value = flops_step * e2e_steps * info.world / (e2e_ms * 1e-3) / 1e12
    h2d = sum(x.numel() * 4 for x in xs)
    d2h = sum(y.numel() * 4 for y in ys)

    # ---- roofline of the dominant kernel (tc_conv_kernel: the tcgen05 contraction) ------
    kernel_ms_step = sum(kern_ms)
    tf32_peak = pk["bf16"] / 2.0
    mode_peak = tf32_peak * tensor_factor(args.precision)
    nominal_peak = NOMINAL_BF16 / 2.0 * tensor_factor(args.precision)
    achieved = flops_step / (kernel_ms_step * 1e-3) / 1e12
    traffic = None
    try:
        tr = json.loads(TRAFFIC_FILE.read_text())
        if tr.get("workload") == args.workload and tr.get("precision", "fp32") == args.precision:
            traffic = tr.get("dram_bytes_per_step")
    except Exception:
        pass

    if info.rank != 0:
        return 0

    cpu = None
    if not args.no_cpu_baseline and info.world == 1:
        try:
            from oracle import oracle as O
            threads = O.host_threads()
            v, det = cpu_reference_sample(layers, args.cpu_seconds, threads)
            cpu = {"value": v, "unit": "TFLOP/s", "cores": threads, "kind": "reference",
                   "sample": (f"1 image of each of the {len(layers)} {args.workload} layers, reference kn2row "
                              f"(oracle/_ref convlab::run_method, GemmBackend::parallel({threads})), "
                              f"{det['passes']} passes in {det['seconds']} s; batch-N time = N x per-image time")}
        except Exception as e:
            cpu = {"value": None, "unit": "TFLOP/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    clocks = sampler.summary(t_wall0, t_wall1)
    out = {
        "metric": "effective TFLOP/s (2*N*M*C*k^2*P*Q / time), summed over the workload layers",
        "value": value, "unit": "TFLOP/s", "n_gpus": info.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": job_ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": {"fp32": "f32", "tf32": "tf32", "bf16": "bf16"}[args.precision],
        "data": "synthetic: reference generator uniform[-1,1) (tensor.cpp:104-134) on device, random-init weights",
        "config": {
            "workload": args.workload, "layers": [l.name for l in layers], "per_gpu_batch": layers[0].batch,
            "layout": args.layout,
            "global_batch": layers[0].batch * info.world, "method": args.method,
            "resolved_methods": sorted({p.method for p in plans}),
            "precision": {"fp32": ("fp32-faithful (rel-L2 <= 1e-5): hi*Hi tf32 x2 + cross terms bf16 x2"
                                   if fp32_split() == "mixed" else "fp32-faithful 3xTF32"),
                          "tf32": "tf32 (fast mode)",
                          "bf16": "bf16 operands, fp32 accumulate (fast mode)"}[args.precision],
            "parallelism": f"dp{info.world} (batch-sharded, no data-path collective)",
            "l2": "flushed (256 MiB write) before every timed step", "weights": "pre-packed once, untimed",
        },
        "e2e": {"value": e2e_value, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "steps": e2e_steps,
                "api": ("cl_conv_forward_host, synchronous per layer" if args.e2e_sync else
                        "cl_conv_forward_host_async for the 4 layers of a step, then a stream sync per step") +
                       " (pinned host buffers)"},
        "gpu_launches": launches_per_step * args.steps,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": mode_peak, "unit": "TFLOP/s",
                     "frac": achieved / mode_peak, "traffic": traffic,
                     "kernel": {"fp32": ("tc_conv_kernel (tcgen05: hi*Hi kind::tf32 x2 + cross terms kind::f16 x2)"
                                         if fp32_split() == "mixed" else "tc_conv_kernel (tcgen05 kind::tf32 x3)"),
                                "tf32": "tc_conv_kernel (tcgen05 kind::tf32)",
                                "bf16": "tc_conv_kernel (tcgen05 kind::f16, bf16)"}[args.precision],
                     "kernel_ms_per_step": kernel_ms_step,
                     "peak_note": (f"peak = measured bf16 burst {pk['bf16']} / 2 (tf32 rate) x "
                                   f"{tensor_factor(args.precision):.3g} (effective flops per tf32 MMA flop: "
                                   "fp32 split 'mixed' 1/2, '3xtf32' 1/3; tf32 1; bf16 2); "
                                   f"{pk['source']}.  The bf16 figure is cuBLAS under its own power/clock "
                                   "limits, so a tcgen05 kernel can exceed it; measured_mma_peak is our own "
                                   "kind::tf32 ceiling (tools/mma_probe.cu), nominal_peak the dense 2250 TF "
                                   "bf16 datasheet figure, both scaled the same way"),
                     "fp32_split": fp32_split() if args.precision == "fp32" else None,
                     "measured_mma_peak": mma_peak_for(args.precision),
                     "frac_of_measured_mma_peak": (achieved / mma_peak_for(args.precision)
                                                   if mma_peak_for(args.precision) else None),
                     "nominal_peak": nominal_peak,
                     "frac_of_nominal": achieved / nominal_peak},
        "cpu_baseline": cpu,
        "clocks": clocks,
    }
    if args.per_layer:
        out["layers"] = [{"name": l.name, "method": p.method, "gflop": l.flops() / 1e9, "kernel_ms": km,
                          "kernel_tflops": l.flops() / (km * 1e-3) / 1e12,
                          "frac_of_peak": l.flops() / (km * 1e-3) / 1e12 / mode_peak}
                         for l, p, km in zip(layers, plans, kern_ms)]
        out["step_ms_median"] = statistics.median(step_ms)
    print(json.dumps(out))
    for p in plans:
        p.close()
    if info.distributed:
        import torch.distributed as tdist
        tdist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
