#!/usr/bin/env python3
"""Benchmark of the B200 kn2row hot path -- one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload vgg16] [--method auto] [--precision fp32] [--scaling auto]

Metric (BASELINE.json): per-layer effective TFLOP/s = 2 N M C k^2 P Q / time; the headline
`value` sums the FLOPs of every layer of the workload over the step time.  One STEP is one
forward pass of every layer of the workload (default: configs[2], the VGG-16 13-layer stack
at batch 32 per GPU -- the north-star config and the largest single-GPU one) on synthetic
uniform[-1,1) data from the reference generator (tensor.cpp:104-134), weights pre-packed
once outside the timed region (the reference re-packs per call; the north star treats
weights as static -- stated in DESIGN.md).  The per-layer table (`layers`) carries each
layer's dominant-kernel time, its TFLOP/s and its fraction of the tensor-core and layer
rooflines.

Timing: W untimed warm-up steps, then exactly K steps between a barrier +
cuda.synchronize on both sides; every step is bracketed by CUDA events on the launching
stream and L2 is flushed (256 MiB write, untimed) before each step; the job time is the
MAX over ranks.  `value` = FLOPs of all K steps / that time; `value_median` uses the median
step.  `e2e` repeats the workload through the host-buffer C-ABI call
(cl_conv_forward_host_async, pinned host buffers: H2D + forward + D2H inside the timed region).

Multi-GPU: one process per GPU.  `--gpus N` without a torchrun environment re-launches this
script under `python -m torch.distributed.run --nproc-per-node N` (127.0.0.1).  Images are
independent, so ranks share nothing on the data path: weak scaling gives every rank the
per-GPU batch; strong scaling (default for `--workload scale`: global batch 256) splits the
global batch across ranks.  `--dry-run` goes through the launch and sharding (gloo, no GPU)
and prints the configuration line without timing anything.

--impl reference times the reference's own CPU kn2row (oracle/_ref = the unmodified
reference core compiled from /root/reference) with all host threads, on rank 0 only, on a
bounded sample of the same workload (one image of each layer per step).  That arm never
imports this repo's package.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from dataclasses import dataclass, replace
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
CONFIG_FILE = ROOT / "configs" / "baseline.net"
GROUPS = ("c1", "alexnet", "vgg16", "googlenet", "sweep", "scale")
METRIC = "effective TFLOP/s (2*N*M*C*k^2*P*Q / time), summed over the workload layers"
NOMINAL_BF16 = 2250.0   # dense bf16 TFLOP/s, B200 nominal (B200_PROFILING.md, context only)


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="vgg16", help=f"one of {GROUPS} (suffix -bN overrides the batch)")
    ap.add_argument("--batch", type=int, default=None, help="override the batch (per GPU, or global when strong)")
    ap.add_argument("--scaling", choices=["auto", "weak", "strong"], default="auto",
                    help="weak: the batch is per GPU; strong: the batch is global and split across ranks "
                         "(auto: strong for the C5 'scale' workload, weak otherwise)")
    ap.add_argument("--method", default="auto")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "tf32", "bf16"],
                    help="fp32 = fp32-faithful (rel-L2 <= 1e-5; operand split per layer: the fp16 split of "
                         "power-of-2 scaled operands by default, CLB_SPLIT=3xf16|mixed|3xtf32 forces one); "
                         "tf32 / bf16 = the 1e-2 fast modes")
    ap.add_argument("--layout", default="nchw", choices=["nchw", "nhwc"],
                    help="device tensors NCHW (the reference interface, default) or channels-last "
                         "(cl_conv_forward_nhwc; the e2e leg stays NCHW)")
    ap.add_argument("--shard", choices=["batch", "channels", "channels-fused"], default="batch",
                    help="batch: images split across ranks (no data-path collective); channels: every rank "
                         "convolves all images with its slice of the kernels and an NCCL all-gather assembles "
                         "the output (dist.MShardPlan; for batch-1 layers); channels-fused: the same with the "
                         "gather fused into the epilogue (P2P stores into every rank's output over CUDA IPC)")
    ap.add_argument("--chain", action="store_true",
                    help="one cl_conv_forward_chain call per step: each layer's prepass rides on the previous "
                         "layer's contraction (its converter warps), a tail launch finishes it")
    ap.add_argument("--concurrent", action="store_true",
                    help="run the step's independent layers on concurrent streams (grid-capped launches)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="budget of the CPU-baseline sample")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--dry-run", action="store_true", help="launch + sharding only (gloo, no GPU, no timing)")
    return ap.parse_args(argv)


# ------------------------------------------------------------------- workloads ----
# configs/baseline.net in the reference's network grammar (layers.cpp:31-79) plus `pad=` / `n=`
# columns.  Parsed here without importing the package, so the reference arm never loads it.
@dataclass(frozen=True)
class Layer:
    name: str
    channels: int
    height: int
    width: int
    kernel_count: int
    kernel_size: int
    stride: int = 1
    pad: int = -1
    batch: int = 1

    @property
    def p(self):
        pad = self.kernel_size // 2 if self.pad < 0 else self.pad
        return (self.height + 2 * pad - self.kernel_size) // self.stride + 1

    @property
    def q(self):
        pad = self.kernel_size // 2 if self.pad < 0 else self.pad
        return (self.width + 2 * pad - self.kernel_size) // self.stride + 1

    def flops(self, batch=None):
        n = self.batch if batch is None else batch
        return 2 * n * self.kernel_count * self.channels * self.kernel_size ** 2 * self.p * self.q

    def bytes(self, batch=None):
        """Compulsory fp32 HBM bytes 4 (N C H W + M C k^2 + N M P Q)."""
        n = self.batch if batch is None else batch
        return 4 * (n * self.channels * self.height * self.width
                    + self.kernel_count * self.channels * self.kernel_size ** 2 + n * self.kernel_count * self.p * self.q)


def load_layers(name: str, batch=None):
    group, _, suffix = name.partition("-")
    if group not in GROUPS:
        raise SystemExit(f"unknown workload '{name}' (choose from {GROUPS})")
    out = []
    for raw in CONFIG_FILE.read_text().splitlines():
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        toks = line.split()
        kv = {}
        while toks and "=" in toks[-1]:
            k, _, v = toks.pop().partition("=")
            kv[k] = int(v)
        nm = toks[0]
        if nm != group and not nm.startswith(group + "/"):
            continue
        nums = [int(t) for t in toks[1:]]
        out.append(Layer(nm, nums[0], nums[1], nums[2], nums[3], nums[4], nums[5] if len(nums) == 6 else 1,
                         kv.get("pad", -1), kv.get("n", 1)))
    if suffix:
        batch = int(suffix[1:])
    if batch is not None:
        out = [replace(l, batch=batch) for l in out]
    return out


def shard_range(total: int, world: int, rank: int):
    base, extra = divmod(total, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


@dataclass
class Run:
    rank: int
    world: int
    local_rank: int
    scaling: str
    layers: list            # the workload as configured (batch = per GPU (weak) or global (strong))
    rank_batch: int         # images this rank convolves per layer
    image0: int             # first global image index of this rank

    @property
    def distributed(self):
        return self.world > 1


def setup_run(args) -> Run:
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launch has WORLD_SIZE={world}")
    layers = load_layers(args.workload, args.batch)
    scaling = args.scaling
    if scaling == "auto":
        scaling = "strong" if args.workload.partition("-")[0] == "scale" or args.shard.startswith("channels") else "weak"
    b = layers[0].batch
    if any(l.batch != b for l in layers):
        raise SystemExit("bench.py: a workload's layers share one batch")
    if args.shard.startswith("channels"):
        if scaling != "strong":
            raise SystemExit("bench.py: channel sharding is strong scaling (every rank holds the whole batch)")
        i0, i1 = 0, b
    elif scaling == "strong":
        if b < world:
            raise SystemExit(f"bench.py: strong scaling needs batch {b} >= {world} ranks")
        i0, i1 = shard_range(b, world, rank)
    else:
        i0, i1 = rank * b, (rank + 1) * b
    return Run(rank, world, local, scaling, layers, i1 - i0, i0)


def config_of(args, run: Run) -> dict:
    """The `config` object, identical in both arms (the driver compares them)."""
    layers = run.layers
    per_gpu = layers[0].batch if run.scaling == "weak" else None
    glob = layers[0].batch * run.world if run.scaling == "weak" else layers[0].batch
    return {
        "workload": args.workload, "layers": [l.name for l in layers],
        "global_batch": glob, "per_gpu_batch": per_gpu if per_gpu is not None else -(-glob // run.world),
        "scaling": run.scaling, "layout": args.layout, "method": args.method,
        "schedule": "concurrent" if args.concurrent else ("chain" if args.chain else "sequential"),
        "precision": {"fp32": "fp32-faithful (rel-L2 <= 1e-5): " + SPLIT_TEXT[split_mode()],
                      "tf32": "tf32 (fast mode)", "bf16": "bf16 operands, fp32 accumulate (fast mode)"}[args.precision],
        "parallelism": (f"dp{run.world} (batch-sharded, no data-path collective)" if args.shard == "batch" else
                        f"mp{run.world} (output channels sharded, NCCL all-gather of the output slices)"
                        if args.shard == "channels" else
                        f"mp{run.world} (output channels sharded, all-gather fused into the epilogue: P2P stores)"),
        "l2": "flushed (256 MiB write) before every timed step", "weights": "pre-packed once, untimed",
    }


def relaunch_under_torchrun(args) -> int:
    """`--gpus N` without a torchrun environment: one process per GPU via torch.distributed.run."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


# ----------------------------------------------------------------- precision ----
SPLIT_TEXT = {
    "auto": "fp16 split of power-of-2 scaled operands (lo*Hi + hi*Lo + hi*Hi, kind::f16) for the implicit "
            "kn2row layers of >= 1.2 GFLOP (C not 8 / 16 / 48) and the tensor-core direct kernel, mixed split "
            "(hi*Hi tf32 x2 + cross terms bf16 x2) elsewhere",
    "3xf16": "fp16 split of power-of-2 scaled operands (kind::f16 x3) where the method supports it",
    "mixed": "hi*Hi tf32 x2 + cross terms bf16 x2", "3xtf32": "classic 3xTF32"}


def split_mode():
    """The fp32-faithful split selection in force (api.cu conv_planes_for; CLB_SPLIT forces one)."""
    e = os.environ.get("CLB_SPLIT")
    return e if e in ("3xf16", "mixed", "3xtf32") else "auto"


def split_factor(split):
    """Effective TFLOP/s per tf32 TFLOP/s of the tensor pipe for an operand format (a plan's
    `split`): 3xf16 issues 3 f16 MMAs (each half a tf32 MMA's time per K) per product -> 2/3;
    mixed 4 tf32-MMA slots per 16 K -> 1/2; 3xtf32 6 slots -> 1/3; tf32 1; bf16 2."""
    return {"3xf16": 2.0 / 3.0, "mixed": 0.5, "3xtf32": 1.0 / 3.0, "tf32": 1.0, "bf16": 2.0}[split]


def mma_peak_tf32():
    """Our own kind::tf32 MMA peak (tools/mma_probe.cu, profiles/tf32_mma_peak.json)."""
    f = ROOT / "profiles" / "tf32_mma_peak.json"
    if not f.exists():
        return None
    return json.loads(f.read_text())["tf32_mma_peak_tflops"]


def peaks():
    try:
        p = json.loads(PEAKS_FILE.read_text())
        return {"bf16": float(p["bf16_tflops"]), "bf16_sustained": float(p["bf16_tflops_sustained"]),
                "hbm": float(p["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"bf16": 1590.0, "bf16_sustained": 1400.0, "hbm": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def traffic_for(workload, precision, method):
    """DRAM bytes per step of the contraction kernels from the committed ncu capture of this
    workload (profiles/ncu_traffic_<workload>.json, tools/make_traffic.py), or None."""
    for f in (ROOT / "profiles" / f"ncu_traffic_{workload}.json", ROOT / "profiles" / "ncu_traffic.json"):
        try:
            tr = json.loads(f.read_text())
        except Exception:
            continue
        if (tr.get("workload") == workload and tr.get("precision", "fp32") == precision and method == "auto"
                and tr.get("split", "mixed") == (split_mode() if precision == "fp32" else tr.get("split", "mixed"))):
            return tr.get("dram_bytes_per_step"), str(f.relative_to(ROOT))
    return None, None


# ------------------------------------------------------------------------- clocks ----
class ClockSampler:
    """SM clock / power / throttle reasons sampled DURING the timed region (B200_PROFILING.md
    clocks line): NVML polled every 5 ms from a thread (nvidia-smi -lms as fallback)."""

    REASONS = {"gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
               "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100}

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
        note = None
        if not win and self.samples:
            # a timed region shorter than the sampling period: the samples nearest to it
            win = sorted(self.samples, key=lambda s: min(abs(s[0] - t0), abs(s[0] - t1)))[:2]
            note = "timed region shorter than the 5 ms sampling period: nearest samples"
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({name for s in win for name, bit in self.REASONS.items() if s[4] & bit})
        out = {"sm_mhz": statistics.median(s[1] for s in win), "sm_max_mhz": win[0][2],
               "power_w_max": max(s[3] for s in win), "reasons": reasons, "samples": len(win)}
        if note:
            out["note"] = note
        return out


# ------------------------------------------------------------------- CPU baseline ----
def cpu_baseline(layers, threads: int, budget_s: float) -> dict:
    """The reference's own CPU paths through its public benchmark API (oracle/_ref:
    convlab::benchmark(layer, method, runs, backend, seed), bench.cpp:87-151 -- 1 untimed
    warm-up, then timed runs, input generation excluded) on ONE image of every layer of the
    workload (the reference has no batch dimension: batch-N time = N x per-image time):
    kn2row and im2col at GemmBackend::parallel(T), kn2row at blocked (1 core), and kn2row's
    thread scaling 1 -> T over the whole sample.  Returns the cpu_baseline object; `value` is
    kn2row at parallel(T) (the paper's method, the reference arm's path)."""
    from oracle import oracle as O

    if not O.ref_available():
        raise RuntimeError("oracle/_ref (compiled reference) is not available")
    img_flops = sum(l.flops(1) for l in layers)
    t_start = time.perf_counter()

    def run(method, thr):
        per = []
        for li, l in enumerate(layers):
            r = O.ref_benchmark(method, l.channels, l.height, l.width, l.kernel_count, l.kernel_size, 1, thr, li)
            per.append(r["min_s"])
        return per

    per_kn = run("kn2row", threads)
    per_im = run("im2col", threads)
    per_1c = run("kn2row", 0)             # GemmBackend::blocked(): one core
    scaling = {"1": img_flops / sum(per_1c) / 1e9}
    t = 2
    while t < threads and time.perf_counter() - t_start < budget_s:
        scaling[str(t)] = img_flops / sum(run("kn2row", t)) / 1e9
        t *= 2
    scaling[str(threads)] = img_flops / sum(per_kn) / 1e9
    spent = time.perf_counter() - t_start
    return {
        "value": img_flops / sum(per_kn) / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": "reference",
        "sample": (f"1 image of each of the {len(layers)} layers ({img_flops / 1e9:.1f} GFLOP), reference "
                   f"convlab::benchmark (oracle/_ref, the unmodified reference core), 1 warm-up + 1 timed run per "
                   f"layer and backend; kn2row/im2col at GemmBackend::parallel({threads}), kn2row at blocked (1 core) "
                   f"and at 2..{threads} threads; {spent:.1f} s of CPU work; batch-N time = N x per-image time"),
        "kn2row_parallel_tflops": img_flops / sum(per_kn) / 1e12,
        "im2col_parallel_tflops": img_flops / sum(per_im) / 1e12,
        "kn2row_1core_tflops": img_flops / sum(per_1c) / 1e12,
        "kn2row_thread_scaling_gflops": scaling,
        "kn2row_speedup_1_to_T": sum(per_1c) / sum(per_kn),
        "per_layer_s": [{"name": l.name, "kn2row_T": a, "im2col_T": b, "kn2row_1core": c}
                        for l, a, b, c in zip(layers, per_kn, per_im, per_1c)],
    }


def run_reference_arm(args, run: Run) -> int:
    if run.rank != 0:
        return 0
    from oracle import oracle as O   # the CPU checker / reference binding -- not this package
    threads = O.host_threads()
    layers = run.layers
    try:
        # each step: one image through every layer (bounded sample of the workload)
        data = []
        for li, l in enumerate(layers):
            x, w = O.make_problem(1, l.channels, l.height, l.width, l.kernel_count, l.kernel_size, li)
            data.append((x[0].copy(), w))
        sample_flops = sum(l.flops(1) for l in layers)
        for _ in range(args.warmup):
            for x, w in data:
                O.ref_run_method("kn2row", x, w, threads)
        step_s = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            for x, w in data:
                O.ref_run_method("kn2row", x, w, threads)
            step_s.append(time.perf_counter() - t0)
        dt = sum(step_s)
    except Exception as e:  # pragma: no cover
        print(json.dumps({"impl": "reference", "unavailable": f"reference CPU path failed: {e}"}))
        return 0
    value = sample_flops * args.steps / dt / 1e12
    sample = (f"1 image of each of the {len(layers)} {args.workload} layers per step "
              f"(reference convlab::run_method(Kn2row), GemmBackend::parallel({threads})); "
              f"the reference has no batch dim, batch-N time = N x per-image time")
    print(json.dumps({
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": "TFLOP/s", "n_gpus": run.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "step_ms_median": statistics.median(step_s) * 1e3,
        "higher_is_better": True, "scaling": run.scaling, "vs_baseline": None,
        "dtype": "f32", "data": "synthetic: reference generator uniform[-1,1) (tensor.cpp:104-134)",
        "config": config_of(args, run),
        "device": f"host CPU only ({threads} threads on rank 0; no GPU used by this arm)",
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))
    return 0


def dry_run(args, run: Run) -> int:
    import torch.distributed as dist
    if run.distributed:
        dist.init_process_group("gloo")
    batches = [run.rank_batch]
    if run.distributed:
        out = [None] * run.world
        dist.all_gather_object(out, (run.rank, run.image0, run.rank_batch))
        batches = [b for _, _, b in sorted(out)]
        dist.barrier()
        dist.destroy_process_group()
    if run.rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "value": None, "unit": "TFLOP/s", "n_gpus": run.world,
                          "scaling": run.scaling, "rank_batches": batches, "config": config_of(args, run)}))
    return 0


# ------------------------------------------------------------------------- our arm ----
def run_ours(args, run: Run) -> int:
    import torch

    import paper_1704_04428_b200 as clb
    from paper_1704_04428_b200 import _lib, dist, rng

    info = dist.RankInfo(run.rank, run.world, run.local_rank)
    if run.distributed:
        os.environ.setdefault("NCCL_DEBUG", "INFO")            # NCCL init log (transport, NVLS) to a file
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", f"/tmp/clb_nccl.{run.rank}.log")
    dist.init("nccl")
    dev = run.local_rank
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    pk = peaks()
    rank_layers = [replace(l, batch=run.rank_batch) for l in run.layers]

    # ---- setup (untimed): plans, packed weights, resident inputs/outputs/workspaces ----
    plans, xs, ys, wss = [], [], [], []
    for li, l in enumerate(rank_layers):
        lc = clb.LayerConfig(l.name, l.channels, l.height, l.width, l.kernel_count, l.kernel_size, l.stride,
                             None if l.pad < 0 else l.pad, l.batch)
        if args.shard.startswith("channels"):
            plan = dist.MShardPlan(lc, info, args.method, args.precision, dev, fused=args.shard == "channels-fused")
        else:
            plan = clb.ConvPlan(lc, args.method, args.precision, dev)
        if args.layout == "nhwc" and plan.method not in ("kn2row-gpu", "conv1x1-gpu", "kn2row-acc-gpu"):
            plan.close()   # channels-last is served by the implicit kernel only
            plan = clb.ConvPlan(lc, "kn2row-gpu" if l.kernel_size > 1 else "conv1x1-gpu", args.precision, dev)
        x = torch.empty((l.batch, l.channels, l.height, l.width), device=dev, dtype=torch.float32)
        w = torch.empty((l.kernel_count, l.kernel_size, l.kernel_size, l.channels), device=dev, dtype=torch.float32)
        img = l.channels * l.height * l.width
        # one global reference stream per layer: this rank's images are images [image0, image0 + batch)
        rng.fill_uniform(x, rng.split(li, 0), run.image0 * img)
        rng.fill_uniform(w, rng.split(li, 1))
        if plan.method == "direct-gpu" and not args.shard.startswith("channels"):
            # host upload: the direct kernel's constant-bank weight path is used for weights that
            # come from the host (a device upload never blocks on a D2H copy; DESIGN 4.1c)
            plan.set_weights_host(w.cpu())
        else:
            plan.set_weights(w)
        base = plan.plan if args.shard.startswith("channels") else plan
        ws = torch.empty(max(base.workspace_bytes(), 4), device=dev, dtype=torch.uint8)
        y = torch.empty(plan.output_shape(), device=dev, dtype=torch.float32)
        if args.layout == "nhwc":   # same values, channels-last storage
            x = x.permute(0, 2, 3, 1).contiguous()
            y = y.permute(0, 2, 3, 1).contiguous()
        plans.append(plan)
        xs.append(x)
        ys.append(y)
        wss.append(ws)
    flush_mb = int(os.environ.get("CLB_FLUSH_MB", "256"))   # L2 flush: a write larger than the 126 MB L2
    flush = torch.empty(flush_mb * 1024 * 1024, device=dev, dtype=torch.uint8)
    flops_job = sum(l.flops() for l in run.layers) * (run.world if run.scaling == "weak" else 1)
    bases = [p.plan if args.shard.startswith("channels") else p for p in plans]   # the ConvPlans this rank runs
    # FLOPs of this rank's launches (its kernel slice when sharding channels)
    rank_flops = [l.flops() * ((p.m1 - p.m0) / l.kernel_count if args.shard.startswith("channels") else 1)
                  for l, p in zip(rank_layers, plans)]

    # concurrent layers (--concurrent): each layer on its own stream with an SM share proportional
    # to its standalone time, forked from / joined into the step stream, captured as one CUDA graph
    if args.chain and (args.layout != "nchw" or args.shard != "batch"):
        raise SystemExit("bench.py: --chain runs NCHW batch-sharded plans")
    conc = None
    if args.concurrent:
        if args.shard != "batch" or args.chain:
            raise SystemExit("bench.py: --concurrent runs batch-sharded plans, one per stream (no --chain)")
        from paper_1704_04428_b200 import concurrency
        n_sms = torch.cuda.get_device_properties(dev).multi_processor_count
        conc = concurrency.build(plans, xs, ys, wss, stream, n_sms, args.layout)

    def step(record_kernel=None):
        if conc is not None:
            conc.replay()                      # the whole fan-out: one graph launch
            return
        if args.chain:
            if record_kernel is not None:
                for li, plan in enumerate(bases):
                    b, e = record_kernel[li]
                    _lib.lib().cl_conv_set_profile_events(plan._h, b.cuda_event, e.cuda_event)
            clb.forward_chain(plans, xs, ys, wss, stream)
            if record_kernel is not None:
                for plan in bases:
                    _lib.lib().cl_conv_set_profile_events(plan._h, None, None)
            return
        for li, plan in enumerate(plans):
            if record_kernel is not None:
                b, e = record_kernel[li]
                _lib.lib().cl_conv_set_profile_events(bases[li]._h, b.cuda_event, e.cuda_event)
            if args.shard.startswith("channels"):
                ys[li] = plan.forward(xs[li])          # this rank's slice + the NCCL all-gather
            else:
                plan.forward(xs[li], ys[li], wss[li], layout=args.layout)
            if record_kernel is not None:
                _lib.lib().cl_conv_set_profile_events(bases[li]._h, None, None)

    sampler = ClockSampler(int(os.environ.get("CLB_SMI_INDEX", dev)))
    sampler.start()
    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    launches_per_step = sum(p.launch_count() for p in bases)

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    st_b = [ev() for _ in range(args.steps)]
    st_e = [ev() for _ in range(args.steps)]
    k_ev = [[(ev(), ev()) for _ in plans] for _ in range(args.steps)] if conc is None else None
    for pair in (p for row in (k_ev or []) for p in row):   # torch creates CUDA events lazily:
        pair[0].record(stream)                       # record once so .cuda_event is a live
        pair[1].record(stream)                       # handle the library can record into
    torch.cuda.synchronize()

    dist.barrier(info)
    torch.cuda.synchronize()
    t_wall0 = time.time()
    for i in range(args.steps):
        flush.zero_()                       # L2 flush, outside the step events
        st_b[i].record(stream)
        step()
        st_e[i].record(stream)
    torch.cuda.synchronize()
    dist.barrier(info)
    t_wall1 = time.time()
    sampler.stop()
    # the per-layer kernel times come from as many further steps with the library's profile events
    # around each layer's dominant kernel (an event between a prepass and its contraction breaks
    # their programmatic-dependent-launch overlap, so these steps are not the ones timed above)
    if k_ev:
        for i in range(args.steps):
            flush.zero_()
            step(k_ev[i])
        torch.cuda.synchronize()

    step_ms = [st_b[i].elapsed_time(st_e[i]) for i in range(args.steps)]
    local_ms = sum(step_ms)
    if conc is None:
        kern_ms = [statistics.median(k_ev[i][li][0].elapsed_time(k_ev[i][li][1]) for i in range(args.steps))
                   for li in range(len(plans))]
    else:   # overlapping layers have no per-layer kernel time: their standalone forwards instead
        kern_ms = list(conc.standalone_ms)
    job_ms = dist.max_over_ranks(local_ms, info, device=dev)
    med_ms = dist.max_over_ranks(statistics.median(step_ms), info, device=dev)
    value = flops_job * args.steps / (job_ms * 1e-3) / 1e12
    value_median = flops_job / (med_ms * 1e-3) / 1e12

    # ---- e2e through the host-buffer C-ABI call (pinned host in / out, every byte timed) ----
    hx = [x.cpu().pin_memory() for x in xs] if args.layout == "nchw" else \
         [x.permute(0, 3, 1, 2).contiguous().cpu().pin_memory() for x in xs]   # the host call takes NCHW
    hy = [torch.empty(p.output_shape(), dtype=torch.float32).pin_memory() for p in plans]
    # the layers are independent: each is issued on its own stream (the async call orders its
    # copy-in after prior work on its stream), so their transfers overlap on both copy engines
    e2e_streams = [torch.cuda.Stream() for _ in plans]

    def e2e_step():
        if args.shard.startswith("channels"):
            # H2D of the input, the sharded forward (slice + NCCL all-gather), D2H of the output
            for li, p in enumerate(plans):
                xs[li].copy_(hx[li], non_blocking=True)
                hy[li].copy_(p.forward(xs[li]), non_blocking=True)
            stream.synchronize()
            return
        for li, p in enumerate(plans):
            p.forward_host_async(hx[li], hy[li], e2e_streams[li])
        for s in e2e_streams:
            s.synchronize()

    e2e_step()
    e2e_steps = max(1, min(args.e2e_steps, args.steps))
    dist.barrier(info)
    torch.cuda.synchronize()
    eb, ee = ev(), ev()
    eb.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    ee.record(stream)
    torch.cuda.synchronize()
    e2e_ms = dist.max_over_ranks(eb.elapsed_time(ee), info, device=dev)
    e2e_value = flops_job * e2e_steps / (e2e_ms * 1e-3) / 1e12
    h2d = sum(x.numel() * 4 for x in hx)
    d2h = sum(y.numel() * 4 for y in hy)

    # ---- roofline of the dominant kernel (tc_conv_kernel: the tcgen05 contraction) ------
    # each layer against the peak of its own operand format (plan.split); the step's tcgen05
    # layers against the FLOP-weighted combination (sum of the layers' times at their peaks)
    tf32_peak = pk["bf16"] / 2.0
    hbm = pk["hbm"]
    tc_idx = [i for i, p in enumerate(plans) if p.method != "direct-gpu"]
    tc_flops = sum(rank_flops[i] for i in tc_idx)
    tc_ms = sum(kern_ms[i] for i in tc_idx)
    splits = sorted({plans[i].split for i in tc_idx})

    def combined(peak_tf32):
        if not tc_idx or not peak_tf32:
            return None
        return tc_flops / sum(rank_flops[i] / (peak_tf32 * split_factor(plans[i].split)) for i in tc_idx)

    mode_peak = combined(tf32_peak)
    nominal_peak = combined(NOMINAL_BF16 / 2.0)
    mma_peak = combined(mma_peak_tf32())
    if conc is not None:     # concurrent step: the whole step (prepasses and all) is the measure
        tc_ms = med_ms
    achieved = tc_flops / (tc_ms * 1e-3) / 1e12 if tc_ms > 0 else None
    traffic, traffic_src = traffic_for(args.workload, args.precision, args.method)
    if run.world > 1 or args.batch is not None:
        traffic, traffic_src = None, None       # the capture is of the 1-GPU default batch
    layer_rows = []
    for l, p, km, fl in zip(rank_layers, plans, kern_ms, rank_flops):
        ai = l.flops() / l.bytes()
        lpeak = tf32_peak * split_factor(p.split if p.split in ("3xf16", "mixed", "3xtf32", "tf32", "bf16")
                                         else {"fp32": "mixed", "tf32": "tf32", "bf16": "bf16"}[args.precision])
        bound = min(lpeak, ai * hbm / 1e3)
        tf = fl / (km * 1e-3) / 1e12
        layer_rows.append({"name": l.name, "method": p.method, "split": p.split, "batch": l.batch,
                           "gflop": round(fl / 1e9, 3), "kernel_ms": round(km, 4), "kernel_tflops": round(tf, 1),
                           "peak_tflops": round(lpeak, 1), "frac_of_peak": round(tf / lpeak, 3),
                           "layer_roofline_tflops": round(bound, 1), "frac_of_layer_roofline": round(tf / bound, 3),
                           "bound": "tensor" if bound >= lpeak else "hbm",
                           "share_of_step": round(km / statistics.median(step_ms), 3)})

    if run.rank != 0:
        for p in plans:
            p.close()
        return 0

    cpu = None
    if not args.no_cpu_baseline and run.world == 1:
        try:
            from oracle import oracle as O
            cpu = cpu_baseline(run.layers, O.host_threads(), args.cpu_seconds)
        except Exception as e:
            cpu = {"value": None, "unit": "TFLOP/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    clocks = sampler.summary(t_wall0, t_wall1)
    out = {
        "metric": METRIC,
        "value": value, "unit": "TFLOP/s", "n_gpus": run.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": job_ms / args.steps, "step_ms_median": med_ms, "value_median": value_median,
        "step_ms": [round(t, 4) for t in step_ms],
        "higher_is_better": True, "scaling": run.scaling, "vs_baseline": None,
        "dtype": {"fp32": "f32", "tf32": "tf32", "bf16": "bf16"}[args.precision],
        "data": "synthetic: reference generator uniform[-1,1) (tensor.cpp:104-134) on device, random-init weights",
        "config": config_of(args, run),
        "rank_batch": run.rank_batch,
        "resolved_methods": sorted({p.method for p in plans}),
        "e2e": {"value": e2e_value, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "steps": e2e_steps,
                "api": "cl_conv_forward_host_async per layer, each layer on its own stream, all streams synchronised "
                       "per step (pinned host buffers)"},
        "gpu_launches": launches_per_step * args.steps,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": mode_peak, "unit": "TFLOP/s",
                     "frac": achieved / mode_peak if achieved and mode_peak else None, "traffic": traffic,
                     "traffic_source": traffic_src,
                     "algorithmic_bytes_per_step": sum(rank_layers[i].bytes() for i in tc_idx),
                     "kernel": "tc_conv_kernel (tcgen05; operand formats " + ", ".join(splits) + ": " + "; ".join(
                         {"3xf16": "3xf16 = lo*Hi + hi*Lo + hi*Hi kind::f16 fp16",
                          "mixed": "mixed = hi*Hi kind::tf32 x2 + cross terms kind::f16 bf16 x2",
                          "3xtf32": "3xtf32 = kind::tf32 x3", "tf32": "tf32 = kind::tf32",
                          "bf16": "bf16 = kind::f16 bf16"}[s_] for s_ in splits) + ")",
                     "kernel_ms_per_step": tc_ms, "kernel_layers": len(tc_idx),
                     # the kernels are timed inside steps K+1..2K of one continuous run, where the board's
                     # power cap can engage (sw_power_cap, `step_ms` shows when): MEASURED_PEAKS.json's
                     # sustained cuBLAS figure is the like-for-like denominator there; `peak` / `frac`
                     # stay on the (higher) burst figure
                     "peak_sustained": (mode_peak * pk["bf16_sustained"] / pk["bf16"]
                                        if mode_peak and pk.get("bf16_sustained") else None),
                     "frac_of_sustained_peak": (achieved / (mode_peak * pk["bf16_sustained"] / pk["bf16"])
                                                if achieved and mode_peak and pk.get("bf16_sustained") else None),
                     "peak_note": (f"peak = measured bf16 burst {pk['bf16']} / 2 (tf32 rate) x the operand format's "
                                   "effective flops per tf32 MMA flop (3xf16 2/3 = bf16 / 3, mixed 1/2, 3xtf32 1/3, "
                                   "tf32 1, bf16 2), FLOP-weighted over the layers (sum of the layers' times at "
                                   f"their peaks); {pk['source']}.  achieved = FLOPs of the tcgen05 layers / the median "
                                   "per-step sum of their CUDA-event-timed contraction launches; the direct-gpu layer "
                                   "(VGG conv1_1, CUDA cores, HBM-bound) is in `layers` against its own roofline"),
                     "fp32_split": split_mode() if args.precision == "fp32" else None,
                     "operand_splits": splits,
                     "measured_mma_peak": mma_peak,
                     "frac_of_measured_mma_peak": achieved / mma_peak if achieved and mma_peak else None,
                     "nominal_peak": nominal_peak,
                     "frac_of_nominal": achieved / nominal_peak if achieved and nominal_peak else None},
        "layers": layer_rows,
        "concurrent": (None if conc is None else
                       {"sm_caps": conc.caps, "standalone_forward_ms": [round(t, 4) for t in conc.standalone_ms],
                        "standalone_sum_ms": round(sum(conc.standalone_ms), 4),
                        "note": "layers on concurrent streams with SM caps proportional to their standalone forward "
                                "time, captured as one CUDA graph; per-layer rows carry the standalone forward time "
                                "(prepass + contraction) and roofline.achieved uses the median whole step"}),
        "cpu_baseline": cpu,
        "clocks": clocks,
    }
    print(json.dumps(out))
    for p in plans:
        p.close()
    if run.distributed:
        import torch.distributed as tdist
        tdist.destroy_process_group()
    return 0


def main(argv=None):
    args = parse_args(argv)
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args)
    run = setup_run(args)
    if args.dry_run:
        return dry_run(args, run)
    if args.impl == "reference":
        return run_reference_arm(args, run)
    return run_ours(args, run)


if __name__ == "__main__":
    sys.exit(main())
