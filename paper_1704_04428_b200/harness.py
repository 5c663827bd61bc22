"""Harness mirror for the GPU methods (reference bench.hpp/bench.cpp).

benchmark(layer, method, runs, seed)  <- convlab::benchmark (bench.cpp:87-151):
    1 untimed warm-up, `runs` timed end-to-end executions of the method (here: the device
    forward incl. its prepass, CUDA events on the launching stream; input generation and the
    one-time weight pre-pack excluded -- the north star treats weights as static), mean / min /
    population stddev, fnv1a checksum of the output (bench.cpp:25-36) and the reference's
    nondeterminism check on the first timed run (bench.cpp:126-128).
emit_csv / parse_csv  <- bench.cpp:211-294: the reference's 10 columns first, byte-exact
    header, shortest round-trip floats; GPU columns appended (batch, pad, precision, gpus,
    eff_tflops, pct_peak).
Inputs come from the reference generator on the device (rng.fill_uniform), seeded like
benchmark(): input split(seed, 0), kernels split(seed, 1) (bench.cpp:109-112).
"""
from __future__ import annotations

import io
import math
import struct
from dataclasses import dataclass, field
from typing import Iterable, List

from .methods import ConvPlan, LayerConfig, footprint

CSV_HEADER = ("layer,method,runs,mean_s,min_s,stddev_s,input_bytes,kernel_bytes,intermediate_bytes,"
              "output_bytes")
GPU_COLUMNS = "batch,pad,precision,gpus,eff_tflops,pct_peak"
# tensor-core peak of each operand format (pct_peak column): bf16 burst (MEASURED_PEAKS.json
# figure) / 3 for the fp16 split (3 f16 MMAs per product), / 4 for the mixed split (4 tf32-MMA
# slots per 16 K-elements), / 6 for the classic 3xTF32 split; x 1/2 tf32, x 1 bf16 fast modes
_BF16_PEAK = 1667.0
SPLIT_PEAK_TFLOPS = {"3xf16": _BF16_PEAK / 3, "mixed": _BF16_PEAK / 4, "3xtf32": _BF16_PEAK / 6,
                     "tf32": _BF16_PEAK / 2, "bf16": _BF16_PEAK, "fp32-fma": _BF16_PEAK / 4}


@dataclass
class BenchResult:
    layer: str
    method: str
    runs: int
    mean_s: float
    min_s: float
    stddev_s: float
    input_bytes: int
    kernel_bytes: int
    intermediate_bytes: int
    output_bytes: int
    batch: int = 1
    pad: int = 0
    precision: str = "fp32"
    gpus: int = 1
    eff_tflops: float = 0.0
    pct_peak: float = 0.0
    samples: List[float] = field(default_factory=list, compare=False)
    output_checksum: int = field(default=0, compare=False)

    def csv_equal(self, other: "BenchResult") -> bool:
        keys = ("layer", "method", "runs", "mean_s", "min_s", "stddev_s", "input_bytes", "kernel_bytes",
                "intermediate_bytes", "output_bytes")
        return all(getattr(self, k) == getattr(other, k) for k in keys)


def fnv1a(t) -> int:
    """bench.cpp:25-36 over the fp32 bit patterns, bytes low..high (a CUDA or CPU tensor);
    computed by cl_checksum_fnv1a on a host copy."""
    import ctypes

    from . import _lib
    a = t.detach().float().contiguous().cpu()
    return int(_lib.lib().cl_checksum_fnv1a(ctypes.c_void_p(a.data_ptr()), a.numel()))


def benchmark(layer: LayerConfig, method: str = "auto", runs: int = 5, seed: int = 0, precision: str = "fp32",
              checksum: bool = True, device: int = 0) -> BenchResult:
    import torch

    from . import rng
    if runs < 1:
        raise ValueError("benchmark: runs must be >= 1")
    require_device(device)
    if layer.stride != 1 and method not in ("im2col-gpu", "im2row-gpu", "direct-gpu"):
        raise ValueError(f"benchmark: strided layer '{layer.name}' is not supported")
    with ConvPlan(layer, method, precision, device) as plan:
        x = torch.empty((layer.batch, layer.channels, layer.height, layer.width), device=f"cuda:{device}")
        w = torch.empty((layer.kernel_count, layer.kernel_size, layer.kernel_size, layer.channels),
                        device=f"cuda:{device}")
        rng.fill_uniform(x, rng.split(seed, 0))
        rng.fill_uniform(w, rng.split(seed, 1))
        plan.set_weights(w)
        ws = torch.empty(max(plan.workspace_bytes(), 4), dtype=torch.uint8, device=x.device)
        y = plan.forward(x, None, ws)                         # warm-up (bench.cpp:115-118)
        torch.cuda.synchronize()
        first = fnv1a(y) if checksum else 0
        samples = []
        for r in range(runs):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            plan.forward(x, y, ws)
            e1.record()
            torch.cuda.synchronize()
            samples.append(e0.elapsed_time(e1) * 1e-3)
            if r == 0 and checksum and fnv1a(y) != first:      # bench.cpp:126-128
                raise RuntimeError(f"benchmark: nondeterministic output for layer '{layer.name}', method {method}")
        resolved = plan.method
        split = plan.split
    mean = sum(samples) / runs
    std = math.sqrt(sum((s - mean) ** 2 for s in samples) / runs)   # population stddev
    fp = footprint(layer, resolved)
    tf = layer.flops() / min(samples) / 1e12
    return BenchResult(layer.name, resolved, runs, mean, min(samples), std, fp["input_bytes"], fp["kernel_bytes"],
                       fp["intermediate_bytes"], fp["output_bytes"], layer.batch, layer.pad, precision, 1, tf,
                       100.0 * tf / SPLIT_PEAK_TFLOPS.get(split, _BF16_PEAK / 4), samples, first)


def _fmt(v: float) -> str:
    """Shortest round-trip form (the reference uses std::to_chars, bench.cpp:38-42)."""
    return repr(float(v))


def emit_csv(results: Iterable[BenchResult], out=None, gpu_columns: bool = True) -> str:
    buf = io.StringIO()
    buf.write(CSV_HEADER + ("," + GPU_COLUMNS if gpu_columns else "") + "\n")
    for r in results:
        row = [r.layer, r.method, str(r.runs), _fmt(r.mean_s), _fmt(r.min_s), _fmt(r.stddev_s), str(r.input_bytes),
               str(r.kernel_bytes), str(r.intermediate_bytes), str(r.output_bytes)]
        if gpu_columns:
            row += [str(r.batch), str(r.pad), r.precision, str(r.gpus), _fmt(r.eff_tflops), _fmt(r.pct_peak)]
        buf.write(",".join(row) + "\n")
    text = buf.getvalue()
    if out is not None:
        out.write(text)
    return text


def parse_csv(text: str) -> List[BenchResult]:
    """bench.cpp:258-288: header check, 10 (or 16 with GPU columns) fields, numeric errors name
    the line."""
    lines = text.splitlines()
    if not lines:
        raise RuntimeError("csv: empty input")
    header = lines[0].rstrip("\r")
    gpu = header == CSV_HEADER + "," + GPU_COLUMNS
    if header != CSV_HEADER and not gpu:
        raise RuntimeError("csv: unexpected header: " + header)
    want = 16 if gpu else 10
    out = []
    for no, line in enumerate(lines[1:], 2):
        line = line.rstrip("\r")
        if not line:
            continue
        f = line.split(",")
        if len(f) != want:
            raise RuntimeError(f"csv line {no}: expected {want} fields, got {len(f)}")
        try:
            r = BenchResult(f[0], f[1], int(f[2]), float(f[3]), float(f[4]), float(f[5]), int(f[6]), int(f[7]),
                            int(f[8]), int(f[9]))
            if gpu:
                r.batch, r.pad, r.precision, r.gpus = int(f[10]), int(f[11]), f[12], int(f[13])
                r.eff_tflops, r.pct_peak = float(f[14]), float(f[15])
        except ValueError:
            raise RuntimeError(f"csv line {no}: bad numeric field") from None
        out.append(r)
    return out


# ---------------------------------------------------------------------------------------
# verify  <- convlab::verify (bench.cpp:158-209; bench.hpp:69-101)
# ---------------------------------------------------------------------------------------
VERIFY_DEFAULT_METHODS = ["kn2row-gpu", "kn2row-explicit-gpu", "kn2col-gpu", "kn2row-acc-gpu", "im2col-gpu", "im2row-gpu",
                          "conv1x1-gpu"]


@dataclass
class VerifyEntry:
    layer: str
    method: str
    passed: bool = False
    max_abs_err: float = 0.0
    rel_l2: float = 0.0
    max_rel: float = 0.0


@dataclass
class VerifyReport:
    entries: List[VerifyEntry] = field(default_factory=list)
    skipped: List[str] = field(default_factory=list)

    def all_pass(self) -> bool:
        return all(e.passed for e in self.entries)


def require_device(device: int = 0) -> None:
    """The GPU harness entry points fail loudly without a B200 (no CPU fallback)."""
    from . import _lib
    if device >= int(_lib.lib().cl_device_count()):
        raise _lib.ClError(_lib.CL_ENODEVICE, f"no CUDA device {device} visible (the B200 path has no CPU fallback)")


def verify(layers: Iterable[LayerConfig], methods: Iterable[str] = None, seed: int = 0, max_hw: int = 0,
           precision: str = "fp32", rel: float = 1e-5, abs_tol: float = 1e-6, perturb=None,
           device: int = 0, comparator=None) -> VerifyReport:
    """Deterministic data per layer (input stream split(seed, 2 idx), kernels split(seed, 2 idx + 1),
    bench.cpp:174-177; a batch continues the input stream, so image 0 is the reference's),
    the library's own direct method as the comparator (the reference uses conv_mcmk_sum,
    bench.cpp:187 -- here direct-gpu, an fp32 FMA restatement of the same loop nest), and one
    entry per (layer, method).  fp32 is held to the reference law allclose(rel, abs + rel
    max|ref|) (bench.cpp:188-192); the TF32/BF16 fast modes to the north star's rel-L2 <= 1e-2.
    Strided layers and conv1x1 on k != 1 are skipped, not failed (bench.cpp:164-167, 194-198).

    `comparator(x, w) -> y` (torch tensors, NCHW / MKKC / NCHW) replaces the direct-gpu
    comparator: the tests pass the CPU oracle conv_mcmk_sum here (the reference's own comparator,
    bench.cpp:186), which the package itself never imports (oracle/ is test infrastructure)."""
    import torch

    from . import rng
    from .methods import method_requires_1x1
    methods = list(methods) if methods is not None else list(VERIFY_DEFAULT_METHODS)
    require_device(device)
    report = VerifyReport()
    dev = f"cuda:{device}"
    for idx, layer in enumerate(layers):
        if layer.stride != 1:
            report.skipped.append(f"{layer.name}: stride {layer.stride} (strided convolution is out of scope)")
            continue
        h = min(layer.height, max_hw) if max_hw > 0 else layer.height
        w = min(layer.width, max_hw) if max_hw > 0 else layer.width
        if layer.kernel_size > min(h, w) + layer.kernel_size // 2:   # ConvProblem (conv_direct.cpp:15-20)
            report.skipped.append(f"{layer.name}: kernel {layer.kernel_size} too large for {h}x{w}")
            continue
        lay = LayerConfig(layer.name, layer.channels, h, w, layer.kernel_count, layer.kernel_size, 1, layer.pad,
                          layer.batch)
        x = torch.empty((lay.batch, lay.channels, h, w), device=dev)
        wt = torch.empty((lay.kernel_count, lay.kernel_size, lay.kernel_size, lay.channels), device=dev)
        rng.fill_uniform(x, rng.split(seed, 2 * idx))
        rng.fill_uniform(wt, rng.split(seed, 2 * idx + 1))
        if comparator is not None:
            ref = comparator(x, wt).to(dev)
        else:
            with ConvPlan(lay, "direct-gpu", "fp32", device) as plan:
                plan.set_weights(wt)
                ref = plan.forward(x)
        ref64 = ref.double()
        ref_max = ref64.abs().max().item()
        tol_abs = abs_tol + rel * ref_max                                # scaled_tolerance (tensor.cpp:211-213)
        for method in methods:
            if method_requires_1x1(method) and lay.kernel_size != 1:
                report.skipped.append(f"{lay.name}: conv1x1 needs k == 1, layer has k = {lay.kernel_size}")
                continue
            with ConvPlan(lay, method, precision, device) as plan:
                plan.set_weights(wt)
                out = plan.forward(x)
            torch.cuda.synchronize(device)
            if perturb is not None:
                perturb(out)
            d = out.double() - ref64
            e = VerifyEntry(lay.name, method)
            e.max_abs_err = d.abs().max().item()
            e.rel_l2 = (d.norm() / ref64.norm().clamp_min(1e-300)).item()
            e.max_rel = e.max_abs_err / max(ref_max, 1e-300)
            finite = bool(torch.isfinite(out).all().item())
            if precision == "fp32":
                e.passed = finite and bool((d.abs() <= tol_abs + rel * ref64.abs()).all().item())
            else:
                e.passed = finite and e.rel_l2 <= 1e-2
            report.entries.append(e)
    return report
