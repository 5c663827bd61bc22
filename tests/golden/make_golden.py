"""Generates tests/golden/ref_outputs.npz from the UNMODIFIED reference library.

Run in the build container (needs /root/reference to build oracle/_ref):
    python tests/golden/make_golden.py
Each case: (name, C, H, W, M, k, seed).  Inputs are regenerated from the seed by the
reference generator (split(seed,0) for the CHW input, split(seed,1) for MKKC kernels --
bench.cpp:109-112), so only the reference outputs are stored:
  <name>/direct_sum : convlab::run_method(DirectSum)  (the oracle, conv_direct.cpp:93-102)
  <name>/kn2row     : convlab::run_method(Kn2row, blocked)  (conv_kn2.cpp:145-162)
  <name>/im2col     : convlab::run_method(Im2col, blocked)  (conv_im2.cpp:108-132)
  <name>/fnv1a      : bench.cpp:25-36 checksum of direct_sum
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402

CASES = [
    # border-dominated shapes (acceptance_main.cpp:182-199; conv_kn2_test.cpp:221-231)
    ("b_2x2_k3", 2, 2, 2, 2, 3, 148),
    ("b_2x6_k3", 3, 2, 6, 4, 3, 11),
    ("b_6x2_k3", 3, 6, 2, 4, 3, 12),
    ("b_3x3_k5", 2, 3, 3, 3, 5, 13),
    ("b_3x8_k5", 2, 3, 8, 3, 5, 14),
    ("b_4x4_k7", 2, 4, 4, 2, 7, 15),
    ("b_1x2_k1", 3, 1, 2, 2, 1, 16),
    # grid / oracle cases (conv_kn2_test.cpp:154-160, 178-185, 242-263)
    ("g_c3_6x5_k3", 3, 6, 5, 4, 3, 141),
    ("g_c3_6x5_k5", 3, 6, 5, 4, 5, 143),
    ("g_c16_13_k3", 16, 13, 13, 8, 3, 142),
    ("g_c16_13_k1", 16, 13, 13, 4, 1, 61),
    ("g_c1_13_k5", 1, 13, 13, 4, 5, 99),
    # small versions of the BASELINE shapes (tap counts 1..11, odd widths)
    ("s_c32_7_k3", 32, 7, 7, 40, 3, 1),
    ("s_c48_7_k5", 48, 7, 7, 24, 5, 2),
    ("s_c40_9_k7", 40, 9, 9, 16, 7, 3),
    ("s_c8_12_k11", 8, 12, 12, 8, 11, 4),
    ("s_c64_14_k3", 64, 14, 14, 64, 3, 5),
]


def main():
    out = {}
    for name, C, H, W, M, k, seed in CASES:
        x, w = O.make_problem(1, C, H, W, M, k, seed)
        ds = O.ref_run_method("direct-sum", x[0], w)
        out[f"{name}/direct_sum"] = ds
        out[f"{name}/kn2row"] = O.ref_run_method("kn2row", x[0], w)
        out[f"{name}/im2col"] = O.ref_run_method("im2col", x[0], w)
        out[f"{name}/fnv1a"] = np.array([O.fnv1a(ds)], dtype=np.uint64)
    np.savez_compressed(Path(__file__).with_name("ref_outputs.npz"), **out)
    print(f"wrote {len(CASES)} cases")


if __name__ == "__main__":
    main()
