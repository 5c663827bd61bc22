"""CPU-side tests: the C-ABI library loads and exports every symbol include/*.h declares,
host logic mirrors the reference interface, contract violations surface before any device
work, and the multi-rank sharding/timing logic (gloo, world size 2)."""
import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _declared_symbols():
    syms = set()
    for h in (ROOT / "include").glob("*.h"):
        syms |= set(re.findall(r"CL_API\s+[\w\s\*]+?\b(cl_\w+)\s*\(", h.read_text()))
    return syms


def test_library_exports_every_declared_symbol():
    import ctypes
    lib = ctypes.CDLL(str(ROOT / "paper_1704_04428_b200" / "libconvlab_b200.so"))
    syms = _declared_symbols()
    assert len(syms) >= 19
    for s in sorted(syms):
        assert hasattr(lib, s), s
    from paper_1704_04428_b200 import _lib
    assert set(_lib.EXPORTS) == syms


def test_package_import_fails_loudly_without_library(tmp_path):
    """No silent fallback: importing the package without the .so raises."""
    pkg = tmp_path / "paper_1704_04428_b200"
    pkg.mkdir()
    for f in (ROOT / "paper_1704_04428_b200").glob("*.py"):
        (pkg / f.name).write_text(f.read_text())
    r = subprocess.run([sys.executable, "-c", "import paper_1704_04428_b200"], cwd=tmp_path,
                       capture_output=True, text=True)
    assert r.returncode != 0 and "no CPU fallback" in r.stderr


def test_abi_basics_and_errors_without_gpu():
    import ctypes
    import paper_1704_04428_b200 as clb
    from paper_1704_04428_b200 import _lib
    L = clb.lib
    assert L.cl_abi_version() == 1
    for name, v in _lib.METHODS.items():
        assert L.cl_method_name(v).decode() == name
        out = ctypes.c_int()
        assert L.cl_method_from_name(name.encode(), ctypes.byref(out)) == 1 and out.value == v
    assert _lib.METHODS["im2row-gpu"] == 8 and L.cl_method_name(9) == b"unknown"
    # contract violations are CL_EINVAL (the reference's std::invalid_argument) even without a GPU
    cases = [
        dict(n=1, c=3, h=8, w=8, m=4, k=2, pad=-1, stride=1),   # even k  (tensor.cpp:64)
        dict(n=1, c=3, h=2, w=2, m=4, k=7, pad=-1, stride=1),   # k > min(H,W)+k/2 (conv_direct.cpp:15-20)
        dict(n=0, c=3, h=8, w=8, m=4, k=3, pad=-1, stride=1),   # zero dim
    ]
    for c in cases:
        d = _lib.ConvDesc(**c)
        h = ctypes.c_void_p()
        assert L.cl_conv_plan(ctypes.byref(d), 1, 0, 0, ctypes.byref(h)) == _lib.CL_EINVAL, c
        assert L.cl_last_error()
    # more than 2^31 pixel rows in one plan (32-bit engine coordinates): refused before device work
    d = _lib.ConvDesc(n=50000, c=3, h=224, w=224, m=4, k=3, pad=1, stride=1)
    h = ctypes.c_void_p()
    assert L.cl_conv_plan(ctypes.byref(d), 1, 0, 0, ctypes.byref(h)) == _lib.CL_EUNSUPPORTED
    assert b"split the batch" in L.cl_last_error()
    d = _lib.ConvDesc(n=1, c=3, h=8, w=8, m=4, k=3, pad=1, stride=1)
    assert L.cl_conv_plan(ctypes.byref(d), 6, 0, 0, ctypes.byref(h)) == _lib.CL_EINVAL   # conv1x1 with k=3
    assert L.cl_conv_plan(ctypes.byref(d), 42, 0, 0, ctypes.byref(h)) == _lib.CL_EINVAL  # unknown method value
    assert b"unknown method" in L.cl_last_error()
    if L.cl_device_count() == 0:
        assert L.cl_conv_plan(ctypes.byref(d), 1, 0, 0, ctypes.byref(h)) == _lib.CL_ENODEVICE
        assert b"no CPU fallback" in L.cl_last_error() or b"device" in L.cl_last_error()


def test_method_names_and_lists():
    import paper_1704_04428_b200 as clb
    assert clb.parse_method_list("kn2row-gpu,,im2col") == ["kn2row-gpu", "im2col"]
    with pytest.raises(ValueError, match="unknown method 'x'"):
        clb.parse_method_list("kn2row,x")
    with pytest.raises(ValueError, match="empty method list"):
        clb.parse_method_list(",")
    assert clb.method_requires_1x1("conv1x1-gpu") and not clb.method_requires_1x1("kn2row-gpu")
    for m in clb.REFERENCE_METHODS:
        assert clb.method_from_name(m) == m


def test_footprint_matches_reference_closed_forms(oracle):
    """bench.cpp:58-85 (and the pinned3 golden numbers, tests/data/golden_bench_columns.csv)."""
    import ctypes
    import paper_1704_04428_b200 as clb
    pinned = {("l1", "kn2row"): (768, 432, 9216, 1024), ("l1", "im2col"): (768, 432, 6912, 1024),
              ("l2", "kn2row"): (1152, 64, 288, 288), ("l3", "im2col"): (280, 600, 7000, 420),
              ("l3", "kn2col"): (280, 600, 10500, 420), ("l1", "direct-sum"): (768, 432, 0, 1024)}
    shapes = {"l1": (3, 8, 8, 4, 3), "l2": (8, 6, 6, 2, 1), "l3": (2, 5, 7, 3, 5)}
    for (ln, m), want in pinned.items():
        fp = clb.footprint(clb.LayerConfig(ln, *shapes[ln]), m)
        assert (fp["input_bytes"], fp["kernel_bytes"], fp["intermediate_bytes"], fp["output_bytes"]) == want
    if oracle.ref_available():
        R = oracle.ref()
        out = (ctypes.c_uint64 * 4)()
        for m in ("kn2row", "kn2col", "im2col", "im2row", "direct-sum", "conv1x1"):
            for sh in shapes.values():
                assert R.ref_footprint(m.encode(), *sh, out) == 0
                fp = clb.footprint(clb.LayerConfig("x", *sh), m)
                assert list(out) == [fp["input_bytes"], fp["kernel_bytes"], fp["intermediate_bytes"],
                                     fp["output_bytes"]], (m, sh)


def test_network_grammar_and_workloads():
    import paper_1704_04428_b200 as clb
    from paper_1704_04428_b200 import workloads
    ls = clb.parse_network_text("# c\nconv1 3 227 227 96 11 4\nconv2 96 27 27 256 5  # x\nc3 8 5 5 4 3 pad=0 n=7\n")
    assert [l.name for l in ls] == ["conv1", "conv2", "c3"] and ls[0].stride == 4 and ls[2].pad == 0
    assert ls[2].batch == 7 and ls[2].out_height == 3
    for bad in ("a 1 2 3 4", "a 1 2 3 4 2", "a 1 2 0 4 3", "a 1 2 x 4 3", "a 1 1 1 1 1\na 1 1 1 1 1"):
        with pytest.raises(RuntimeError, match=r"<text>:\d"):
            clb.parse_network_text(bad)
    # BASELINE totals
    assert round(workloads.total_flops(workloads.workload("vgg16")) / 1e9, 3) == 982.184
    assert round(workloads.total_flops(workloads.workload("c1")) / 1e9, 3) == 0.231
    assert round(workloads.total_flops(workloads.workload("scale")) / 1e9, 3) == 947.040
    assert len(workloads.workload("googlenet")) == 9 and len(workloads.workload("alexnet")) == 4
    assert all(l.batch == 1 for l in workloads.workload("alexnet-b1"))


def test_rng_split_matches_reference(oracle):
    from paper_1704_04428_b200 import rng
    for s, lane in ((0, 0), (0, 1), (12345, 7), (2 ** 63 + 5, 3)):
        assert rng.split(s, lane) == oracle.split(s, lane)


def test_cpp_facade_host_logic():
    exe = ROOT / "tests" / "cpp" / "facade_test"
    if not exe.exists():
        subprocess.run(["make", "-s", "-C", str(exe.parent)], check=True)
    r = subprocess.run([str(exe), "cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "PASSED" in r.stdout, r.stdout + r.stderr


def test_shard_range_properties():
    from paper_1704_04428_b200 import dist
    for total in (1, 7, 256, 1000):
        for world in (1, 2, 3, 8):
            rs = [dist.shard_range(total, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [e - b for b, e in rs]
            assert max(sizes) - min(sizes) <= 1


_WORKER = r'''
import os, sys, json
sys.path.insert(0, sys.argv[1])
import numpy as np, torch, torch.distributed as dist_
from paper_1704_04428_b200 import dist
from oracle import oracle as O
info = dist.init("gloo")
B, C, H, W, M, k = 2, 3, 6, 6, 4, 3
img = C * H * W
# rank r's images = images [rB, (r+1)B) of one global reference stream
x = O.fill(B * img, O.split(0, 0), dist.image_offset(info.rank, B, img)).reshape(B, C, H, W)
w = O.fill(M * k * k * C, O.split(0, 1)).reshape(M, k, k, C)
y = O.conv_batch(x, w)
gathered = [torch.zeros(B, M, H, W) for _ in range(info.world)]
dist_.all_gather(gathered, torch.from_numpy(y))
t = dist.max_over_ranks(1.0 + info.rank, info)
s = dist.sum_over_ranks(10.0, info)
if info.rank == 0:
    xg = O.fill(info.world * B * img, O.split(0, 0)).reshape(-1, C, H, W)
    ok = np.array_equal(torch.cat(gathered).numpy(), O.conv_batch(xg, w))
    print(json.dumps({"ok": bool(ok), "max": t, "sum": s}))
dist_.destroy_process_group()
'''


_MSHARD_WORKER = r'''
import sys, json
sys.path.insert(0, sys.argv[1])
import numpy as np, torch, torch.distributed as dist_
from paper_1704_04428_b200 import dist
from oracle import oracle as O
info = dist.init("gloo")
x, w = O.make_problem(2, 3, 6, 5, 7, 3, 4)      # M = 7 over 2 ranks: uneven slices (4 + 3)
conv = lambda xx, ww: torch.from_numpy(O.conv_batch(xx.numpy(), ww.numpy()))
y = dist.mshard_conv(torch.from_numpy(x), torch.from_numpy(w), info, conv)
if info.rank == 0:
    print(json.dumps({"ok": bool(np.array_equal(y.numpy(), O.conv_batch(x, w))), "shape": list(y.shape)}))
dist_.destroy_process_group()
'''


def test_two_rank_gloo_channel_sharding(tmp_path):
    """SURVEY 8(e) output-channel sharding: slices + all-gather + permute == full conv."""
    import json
    script = tmp_path / "mshard.py"
    script.write_text(_MSHARD_WORKER)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29519", str(script), str(ROOT)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=dict(os.environ, OMP_NUM_THREADS="1"))
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert res == {"ok": True, "shape": [2, 7, 6, 5]}
    from paper_1704_04428_b200 import dist
    assert [dist.channel_slice(7, 2, r) for r in (0, 1)] == [(0, 4), (4, 7)]


def test_two_rank_gloo_sharding(tmp_path):
    """The N>1 path on CPU: per-rank generation offsets reproduce the global batch,
    MAX/SUM reductions behave, results gather to the single-process answer."""
    script = tmp_path / "worker.py"
    script.write_text(_WORKER)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29517", str(script), str(ROOT)]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][0]
    import json
    res = json.loads(line)
    assert res == {"ok": True, "max": 2.0, "sum": 20.0}


def test_harness_csv_roundtrip_and_header():
    """bench.cpp:211-294: byte-exact reference header, 10 reference columns first, GPU columns
    appended; parse(emit(x)) == x; malformed input errors name the line."""
    from paper_1704_04428_b200 import harness
    assert harness.CSV_HEADER == ("layer,method,runs,mean_s,min_s,stddev_s,input_bytes,kernel_bytes,"
                                  "intermediate_bytes,output_bytes")
    rs = [harness.BenchResult("l1", "kn2row-gpu", 2, 1.25e-05, 1.1e-05, 1.5e-06, 768, 432, 0, 1024, 8, 1, "fp32", 1,
                              12.5, 4.5),
          harness.BenchResult("l3", "im2col-gpu", 3, 0.1, 0.09999999999999999, 0.0, 280, 600, 7000, 420)]
    for gpu in (True, False):
        text = harness.emit_csv(rs, gpu_columns=gpu)
        back = harness.parse_csv(text)
        assert all(a.csv_equal(b) for a, b in zip(rs, back))
        assert text.splitlines()[0].startswith(harness.CSV_HEADER)
    assert harness.parse_csv(harness.emit_csv(rs))[0] == rs[0]
    with pytest.raises(RuntimeError, match="csv line 2"):
        harness.parse_csv(harness.CSV_HEADER + "\nl1,x,2,1,1,1,1,1,1\n")
    with pytest.raises(RuntimeError, match="unexpected header"):
        harness.parse_csv("layer,method\n")


def test_fnv1a_matches_reference_checksum(oracle):
    import numpy as np
    import torch
    from paper_1704_04428_b200 import harness
    a = oracle.fill(1000, 3)
    assert harness.fnv1a(torch.from_numpy(a)) == oracle.fnv1a(a)


def _cli(*args):
    import subprocess
    import sys
    return subprocess.run([sys.executable, "-m", "paper_1704_04428_b200", *args], capture_output=True, text=True,
                          cwd=str(Path(__file__).resolve().parents[1]), timeout=300)


def test_cli_footprint_matches_reference_columns(tmp_path):
    """convlab_main.cpp run_footprint: one line per (layer, method), CSV with the reference's
    byte-exact header and runs = 0 rows; reference method names are accepted (closed form)."""
    net = tmp_path / "p.net"
    net.write_text("l1 3 16 16 4 3\nl2 8 10 10 6 5  # comment\n")
    out = tmp_path / "fp.csv"
    r = _cli("footprint", "--net", str(net), "--methods", "kn2row,im2col-gpu,conv1x1", "--out", str(out))
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("l")]
    assert lines[0] == "l1  kn2row  input 3072  kernels 432  intermediate 36864  output 4096 bytes"
    assert len(lines) == 4                               # conv1x1 skipped on k != 1 layers
    from paper_1704_04428_b200 import harness
    rows = harness.parse_csv(out.read_text())
    assert out.read_text().splitlines()[0] == harness.CSV_HEADER
    assert [(x.layer, x.method, x.runs) for x in rows][:2] == [("l1", "kn2row", 0), ("l1", "im2col-gpu", 0)]


def test_cli_usage_and_device_errors(tmp_path):
    net = tmp_path / "p.net"
    net.write_text("l1 3 16 16 4 3\n")
    assert _cli("nonsense").returncode == 2                                  # kExitUsage
    r = _cli("bench", "--net", str(net), "--methods", "kn2row")              # a CPU method: not runnable here
    assert r.returncode == 2 and "not a runnable method" in r.stderr
    assert _cli("footprint", "--net", str(tmp_path / "missing.net")).returncode == 2
    import torch
    if not torch.cuda.is_available():
        r = _cli("verify", "--net", str(net))
        assert r.returncode == 1 and "no CPU fallback" in r.stderr          # fails loudly, no fallback


def test_bench_reference_arm_json_contract():
    """bench.py --impl reference (CPU only, so it runs here): one JSON line with the driver's
    keys, the reference arm's own cpu_baseline and an e2e block with zero transfer bytes."""
    import json
    import subprocess
    import sys
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    root = str(Path(__file__).resolve().parents[1])
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1",
                        "--workload", "c1"], cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["cores"] >= 1


def test_bench_reference_arm_never_loads_the_package():
    """The reference arm times the reference alone: bench.py must not import (and so must not
    load the .so of) this repo's package on that path."""
    import json
    import subprocess
    import sys
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    root = str(Path(__file__).resolve().parents[1])
    code = ("import sys, bench; rc = bench.main(['--impl', 'reference', '--steps', '1', '--warmup', '0', "
            "'--workload', 'c1']); "
            "print('LOADED' if any(m.startswith('paper_1704_04428_b200') for m in sys.modules) else 'CLEAN'); "
            "sys.exit(rc)")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().splitlines()[-1] == "CLEAN", r.stdout
    ref = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    # same config object as our arm's (the driver compares the two lines)
    d = subprocess.run([sys.executable, "bench.py", "--dry-run", "--workload", "c1"], cwd=root, capture_output=True,
                       text=True, timeout=600)
    assert d.returncode == 0, d.stderr[-2000:]
    ours = json.loads([l for l in d.stdout.splitlines() if l.startswith("{")][0])
    assert ref["config"] == ours["config"]


@pytest.mark.parametrize("workload,scaling,batches", [("scale", "strong", [128, 128]), ("c1", "weak", [1, 1])])
def test_bench_gpus_flag_launches_ranks(workload, scaling, batches):
    """`bench.py --gpus 2` without torchrun re-launches itself under torch.distributed.run (one
    process per GPU); --dry-run exercises that launch and the batch sharding on gloo/CPU:
    strong scaling splits the C5 global batch 256 into 128 per rank, weak keeps the per-GPU
    batch."""
    import json
    import subprocess
    import sys
    root = str(Path(__file__).resolve().parents[1])
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--workload", workload, "--dry-run"], cwd=root,
                       capture_output=True, text=True, timeout=600, env=dict(env, OMP_NUM_THREADS="1"))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == scaling and d["rank_batches"] == batches
    assert d["config"]["per_gpu_batch"] == batches[0]
    assert d["config"]["global_batch"] == sum(batches)


def test_concurrency_sm_shares():
    """concurrency.sm_shares: caps proportional to the weights, even (CTA pairs), >= 2 each,
    never above the SM count (every launch's CTAs must stay co-resident), remainder to the
    heaviest layers."""
    from paper_1704_04428_b200 import concurrency
    for weights in ([1.0], [1, 1], [5, 1, 1, 1], [0.05, 0.06, 0.04, 0.04, 0.03, 0.02, 0.03, 0.035, 0.025],
                    [1e-3] * 40):
        caps = concurrency.sm_shares(weights, 148)
        assert len(caps) == len(weights)
        assert sum(caps) <= 148 and all(c >= 2 and c % 2 == 0 for c in caps), (weights, caps)
        heavy = max(range(len(weights)), key=lambda i: weights[i])
        assert caps[heavy] == max(caps)
    assert concurrency.sm_shares([1.0], 148) == [148]
    assert sum(concurrency.sm_shares([3, 1], 148)) == 148
    with pytest.raises(ValueError):
        concurrency.sm_shares([1.0] * 80, 148)      # 80 layers x 2 SMs do not fit


def test_bench_roofline_peaks_per_operand_split():
    """bench.py's per-layer peaks follow each plan's operand format (fp16 split = bf16 / 3, mixed =
    bf16 / 4, 3xTF32 = bf16 / 6, fast modes tf32 / bf16), and the split text covers every
    CLB_SPLIT selection; no GPU involved."""
    import bench
    bf16 = 1653.6
    tf32 = bf16 / 2
    assert abs(tf32 * bench.split_factor("3xf16") - bf16 / 3) < 1e-9
    assert abs(tf32 * bench.split_factor("mixed") - bf16 / 4) < 1e-9
    assert abs(tf32 * bench.split_factor("3xtf32") - bf16 / 6) < 1e-9
    assert bench.split_factor("tf32") == 1.0 and bench.split_factor("bf16") == 2.0
    assert set(bench.SPLIT_TEXT) == {"auto", "3xf16", "mixed", "3xtf32"}
    assert bench.split_mode() in bench.SPLIT_TEXT
