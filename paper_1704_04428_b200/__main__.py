"""Command line mirror of the reference CLI (tools/convlab_main.cpp:47-197) for the GPU methods:

    python -m paper_1704_04428_b200 verify    --net FILE [--methods CSV] [--seed S] [--max-hw N] [--corrupt]
    python -m paper_1704_04428_b200 bench     --net FILE [--methods CSV] [--runs R] [--out CSV] [--seed S]
    python -m paper_1704_04428_b200 footprint --net FILE [--methods CSV] [--out CSV]

plus the GPU dimensions the reference lacks: --batch N (overrides the file's n=), --precision
{fp32,tf32,bf16}, --device D.  Output lines and exit codes (0 ok, 1 verify failure, 2 usage)
follow the reference.  .net files use the reference grammar with optional pad=/n= keys.
"""
import argparse
import sys
from pathlib import Path

from . import harness
from ._lib import ClError
from .methods import ALL_METHODS, GPU_METHODS, LayerConfig, footprint, method_requires_1x1, parse_method_list, \
    parse_network_text

EXIT_OK, EXIT_VERIFY_FAILURE, EXIT_USAGE = 0, 1, 2


def _layers(args):
    layers = parse_network_text(Path(args.net).read_text(), args.net)
    if args.batch:
        layers = [LayerConfig(l.name, l.channels, l.height, l.width, l.kernel_count, l.kernel_size, l.stride, l.pad,
                              args.batch) for l in layers]
    return layers


def _methods(csv, default, allowed=None):
    allowed = allowed or GPU_METHODS + ["auto"]
    if not csv:
        return list(default)
    methods = parse_method_list(csv)
    bad = [m for m in methods if m not in allowed]
    if bad:
        raise ValueError(f"not a runnable method here: {', '.join(bad)} (choose from {', '.join(allowed)})")
    return methods


def run_verify(args) -> int:
    perturb = (lambda t: t.view(-1)[:1].add_(1.0)) if args.corrupt else None   # convlab_main.cpp:53-55
    report = harness.verify(_layers(args), _methods(args.methods, harness.VERIFY_DEFAULT_METHODS), args.seed,
                            args.max_hw, args.precision, perturb=perturb, device=args.device)
    for note in report.skipped:
        print(f"skip: {note}", file=sys.stderr)
    failures = 0
    for e in report.entries:
        failures += 0 if e.passed else 1
        print(f"{'pass' if e.passed else 'FAIL'}  {e.layer}  {e.method}  max|err| = {e.max_abs_err:.6g}  "
              f"rel-L2 = {e.rel_l2:.3g}")
    print(f"{len(report.entries)} checks, {failures} failures, {len(report.skipped)} skipped")
    return EXIT_OK if report.all_pass() else EXIT_VERIFY_FAILURE


def run_bench(args) -> int:
    results = []
    for layer in _layers(args):
        if layer.stride != 1:
            print(f"skip: {layer.name}: stride {layer.stride} (strided convolution is out of scope)", file=sys.stderr)
            continue
        for method in _methods(args.methods, ["auto"]):
            if method_requires_1x1(method) and layer.kernel_size != 1:
                print(f"skip: {layer.name}: conv1x1 needs k == 1", file=sys.stderr)
                continue
            r = harness.benchmark(layer, method, args.runs, args.seed, args.precision, device=args.device)
            print(f"{r.layer}  {r.method}  mean {r.mean_s:.6g} s  min {r.min_s:.6g} s  stddev {r.stddev_s:.6g} s  "
                  f"{r.eff_tflops:.1f} TFLOP/s")
            results.append(r)
    if args.out:
        with open(args.out, "w") as f:
            harness.emit_csv(results, f)
        print(f"wrote {len(results)} rows to {args.out}")
    return EXIT_OK


def run_footprint(args) -> int:
    rows = []
    for layer in _layers(args):
        if layer.stride != 1:
            print(f"skip: {layer.name}: stride {layer.stride} (strided convolution is out of scope)", file=sys.stderr)
            continue
        for method in _methods(args.methods, GPU_METHODS, [m for m in ALL_METHODS if m != "auto"]):
            if method_requires_1x1(method) and layer.kernel_size != 1:
                continue
            fp = footprint(layer, method)
            print(f"{layer.name}  {method}  input {fp['input_bytes']}  kernels {fp['kernel_bytes']}  intermediate "
                  f"{fp['intermediate_bytes']}  output {fp['output_bytes']} bytes")
            rows.append(harness.BenchResult(layer.name, method, 0, 0.0, 0.0, 0.0, fp["input_bytes"],
                                            fp["kernel_bytes"], fp["intermediate_bytes"], fp["output_bytes"]))
    if args.out:
        with open(args.out, "w") as f:
            harness.emit_csv(rows, f, gpu_columns=False)
        print(f"wrote {len(rows)} rows to {args.out}")
    return EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1704_04428_b200",
                                 description="B200 convolution-as-GEMM methods (reference CLI mirror)")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(p):
        p.add_argument("--net", required=True, help="network description file")
        p.add_argument("--methods", default="", help="comma-separated method list")
        p.add_argument("--seed", type=int, default=0, help="data generation seed")
        p.add_argument("--batch", type=int, default=0, help="images per layer (overrides the file's n=)")
        p.add_argument("--precision", default="fp32", choices=["fp32", "tf32", "bf16"])
        p.add_argument("--device", type=int, default=0)

    v = sub.add_parser("verify", help="check every method against the direct comparator")
    common(v)
    v.add_argument("--max-hw", type=int, default=0, help="cap layer H and W at this value")
    v.add_argument("--corrupt", action="store_true", help="perturb outputs (negative-control hook)")
    b = sub.add_parser("bench", help="time methods on each layer")
    common(b)
    b.add_argument("--runs", type=int, default=5, help="timed runs per (layer, method)")
    b.add_argument("--out", default="", help="write results CSV here")
    f = sub.add_parser("footprint", help="closed-form memory accounting")
    common(f)
    f.add_argument("--out", default="", help="write footprint CSV here")
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return EXIT_USAGE if e.code else EXIT_OK
    try:
        return {"verify": run_verify, "bench": run_bench, "footprint": run_footprint}[args.cmd](args)
    except (ValueError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except ClError as e:   # device / library failure (e.g. no B200 visible): no CPU fallback
        print(f"error: {e}", file=sys.stderr)
        return EXIT_VERIFY_FAILURE


if __name__ == "__main__":
    sys.exit(main())
