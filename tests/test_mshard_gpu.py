"""Output-channel sharding (SURVEY.md 8(e) alternative, dist.MShardPlan) on real B200 plans.

  ws2 / gloo : two ranks (both on cuda:0 -- their kernels never wait on each other), each plans
               its kernel slice and runs the plan's HOST path; gloo gathers the slices on the host
  ws1 / nccl : the device path through NCCL's all_gather_into_tensor (world size 1 on this
               one-GPU box; the same call spans 8 GPUs over NVLink / NVSwitch)
  *-fused    : the gather fused into the epilogue (cl_conv_set_peer_outputs): each rank's
               contraction stores its channel slice into every rank's full output through
               CUDA-IPC-mapped pointers (ws2: both ranks on cuda:0, the peer buffer mapped from the
               other process; the kernels never wait on each other -- a barrier after both finish)
Both against the single-process oracle on the same seeded inputs.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent

_WORKER = r'''
import json, sys
sys.path.insert(0, sys.argv[1])
backend = sys.argv[2]
import numpy as np, torch, torch.distributed as tdist
import paper_1704_04428_b200 as clb
from paper_1704_04428_b200 import dist
from oracle import oracle as O
info = dist.from_env()
torch.cuda.set_device(0)
fused = backend.endswith("-fused")
backend = backend.replace("-fused", "")
if backend == "nccl":
    tdist.init_process_group("nccl", device_id=torch.device("cuda:0"))
else:
    tdist.init_process_group("gloo")
out = []
for (N, C, H, W, M, k) in [(1, 64, 56, 56, 64, 3), (2, 96, 27, 27, 250, 5), (1, 256, 28, 28, 256, 1), (3, 16, 13, 13, 7, 3)]:
    x, w = O.make_problem(N, C, H, W, M, k, N + M)
    layer = clb.LayerConfig("ms", C, H, W, M, k, batch=N)
    mp = dist.MShardPlan(layer, info, device=0, fused=fused)
    if backend == "nccl" or fused:
        mp.set_weights(torch.from_numpy(w).cuda())
        y = mp.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    else:
        mp.set_weights_host(torch.from_numpy(w))
        y = mp.forward_host(torch.from_numpy(x)).numpy()
    slice_ = (mp.m0, mp.m1)
    mp.close()
    if info.rank == 0:
        m = O.parity_metrics(y, O.conv_batch(x, w))
        out.append({"shape": [N, C, H, W, M, k], "slice": slice_, "rel_l2": m["rel_l2"], "max_rel": m["max_rel"],
                    "out_shape": list(y.shape)})
if info.rank == 0:
    print(json.dumps(out))
tdist.destroy_process_group()
'''


def _launch(tmp_path, nproc, backend, port):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    script = tmp_path / "ms.py"
    script.write_text(_WORKER)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(script), str(ROOT), backend]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=dict(os.environ, OMP_NUM_THREADS="4"))
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads([l for l in r.stdout.splitlines() if l.startswith("[")][-1])


@pytest.mark.parametrize("nproc,backend,port", [(2, "gloo", 29531), (1, "nccl", 29533), (2, "gloo-fused", 29535),
                                               (1, "nccl-fused", 29537)])
def test_mshard_plan(tmp_path, nproc, backend, port):
    res = _launch(tmp_path, nproc, backend, port)
    assert len(res) == 4
    for r in res:
        N, C, H, W, M, k = r["shape"]
        assert r["out_shape"] == [N, M, H, W]
        assert r["rel_l2"] <= 1e-5 and r["max_rel"] <= 1e-4, r
    if nproc == 2:
        assert res[3]["slice"] == [0, 4]        # M = 7 over 2 ranks: 4 + 3 (uneven, padded gather)


@pytest.mark.parametrize("flags", [["--shard", "channels"], ["--shard", "channels-fused"], ["--concurrent"],
                                   ["--chain"], ["--layout", "nhwc"], ["--precision", "bf16"]],
                         ids=lambda f: "".join(f).replace("--", "-").lstrip("-"))
def test_bench_modes_print_one_line(flags):
    """Every bench.py mode on the smallest workload (C1): exits 0 and prints the driver's JSON
    line with a roofline, an e2e and a launch count (a per-plan attribute missing on MShardPlan
    once broke `--shard channels` without any test noticing)."""
    r = subprocess.run([sys.executable, "bench.py", "--workload", "c1", "--steps", "3", "--warmup", "3",
                        "--e2e-steps", "2", "--no-cpu-baseline", *flags], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["value"] > 0 and line["gpu_launches"] > 0 and line["n_gpus"] == 1
    assert line["roofline"]["achieved"] and line["e2e"]["value"] > 0
    assert len(line["step_ms"]) == 3
