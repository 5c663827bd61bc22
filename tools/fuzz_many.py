"""Wider one-off run of the seeded random-shape GPU sweeps in tests/test_fuzz_gpu.py
(more seeds than the committed tests): prints one line per seed and the failure count."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1704_04428_b200 as clb  # noqa: E402
import tests.test_fuzz_gpu as F  # noqa: E402
from oracle import oracle as O  # noqa: E402

gpu = (torch, clb)
bad = 0
for seed in range(100, 116):
    try:
        F.test_random_shapes_all_methods(O, gpu, seed)
        print("small seed", seed, "ok", flush=True)
    except AssertionError as e:
        bad += 1
        print("small seed", seed, "FAIL", str(e)[:600], flush=True)
for seed in range(200, 208):
    try:
        F.test_random_large_shapes_implicit(O, gpu, seed)
        print("large seed", seed, "ok", flush=True)
    except AssertionError as e:
        bad += 1
        print("large seed", seed, "FAIL", str(e)[:600], flush=True)
print("failures", bad)
