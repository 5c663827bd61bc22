"""Pins the CPU oracle (oracle/oracle.c) before it is trusted as the parity checker.

Two anchors: the reference's own golden vectors / known answers (restated from its unit
tests, cited per case), and the reference library itself (oracle/_ref, compiled from
/root/reference) through the committed fixtures tests/golden/ref_outputs.npz.
"""
from pathlib import Path

import numpy as np
import pytest

from tests.golden.make_golden import CASES

GOLDEN = Path(__file__).parent / "golden" / "ref_outputs.npz"


def test_seed0_bits_pinned(oracle):
    # tensor_test.cpp:131-139
    bits = oracle.fill(4, 0).view(np.uint32).tolist()
    assert bits == [0x3F444150, 0xBE0C3B10, 0xBF727746, 0x3F711770]


def test_generator_range_and_determinism(oracle):
    # tensor_test.cpp: values in [-1, 1), same seed same bits, different seeds differ
    a = oracle.fill(4 * 9 * 11, 5)
    assert (a >= -1).all() and (a < 1).all()
    assert np.array_equal(a.view(np.uint32), oracle.fill(4 * 9 * 11, 5).view(np.uint32))
    assert not np.array_equal(oracle.fill(64, 1), oracle.fill(64, 2))
    # slice fills equal a whole fill (batch buffers are filled as one stream)
    whole = oracle.fill(1000, 77)
    assert np.array_equal(whole[300:], oracle.fill(700, 77, first_index=300))


def test_scsk_known_answer(oracle):
    # conv_direct_test.cpp:42-49: all-ones 3x3 on the 1..9 grid, zero padding
    img = np.arange(1, 10, dtype=np.float32).reshape(3, 3)
    out = oracle.conv2d_scsk(img, np.ones((3, 3), np.float32))
    assert out.ravel().tolist() == [12, 21, 16, 27, 45, 33, 24, 39, 28]


def test_shift_add_known_answers(oracle):
    # conv_kn2_test.cpp:126-132: all-ones 3x3 blocks count in-bounds taps
    out = oracle.shift_add_row(np.ones((9, 9), np.float32), 3, 1, 3, 3)
    assert out.ravel().tolist() == [4, 6, 4, 6, 9, 6, 4, 6, 4]
    # conv_kn2_test.cpp:106-111: k=1 is the identity, bitwise
    blk = oracle.fill(60, 132).reshape(3, 20)
    assert np.array_equal(oracle.shift_add_row(blk, 1, 3, 4, 5), blk)
    # conv_kn2_test.cpp:113-124: only the centre block survives
    k, cnt, h, w = 3, 2, 4, 4
    inter = np.zeros((k * k * cnt, h * w), np.float32)
    centre = oracle.fill(cnt * h * w, 133).reshape(cnt, h * w)
    inter[4 * cnt:5 * cnt] = centre
    assert np.array_equal(oracle.shift_add_row(inter, k, cnt, h, w), centre)
    # col orientation is the transpose law (conv_kn2.cpp:120-142)
    r = oracle.fill(9 * 2 * 20, 9).reshape(18, 20)
    assert np.array_equal(oracle.shift_add_col(np.ascontiguousarray(r.T), 3, 2, 4, 5),
                          oracle.shift_add_row(r, 3, 2, 4, 5).T)


def test_im2col_known_answers(oracle):
    # conv_im2_test.cpp:41-47: centre column enumerates the patch in tap order
    x = np.arange(1, 10, dtype=np.float32).reshape(1, 3, 3)
    pm = oracle.im2col_patch(x, 3)
    assert pm[:, 4].tolist() == [float(r + 1) for r in range(9)]
    # conv_im2_test.cpp:31-39: corner column of a 2x2 image has exactly 4 in-bounds taps
    x2 = oracle.fill(4, 81).reshape(1, 2, 2)
    assert int((oracle.im2col_patch(x2, 3)[:, 0] != 0).sum()) == 4


def test_reorder_offset_law(oracle):
    # conv_kn2_test.cpp:46-56
    w = oracle.fill(2 * 3 * 3 * 2, 122).reshape(2, 3, 3, 2)
    r = oracle.kn2row_reorder(w)
    for m in range(2):
        for i in range(3):
            for j in range(3):
                for c in range(2):
                    assert r[(i * 3 + j) * 2 + m, c] == w[m, i, j, c]


def test_delta_kernels_reproduce_input(oracle):
    # conv_kn2_test.cpp:148-152
    x = oracle.fill(3 * 5 * 5, 137).reshape(3, 5, 5)
    w = np.zeros((3, 3, 3, 3), np.float32)
    for m in range(3):
        w[m, 1, 1, m % 3] = 1.0
    assert np.array_equal(oracle.conv_kn2row(x, w), x)
    assert np.array_equal(oracle.conv_mcmk_sum(x, w), x)


def test_per_tap_decomposition_bitwise(oracle):
    # conv_kn2_test.cpp:195-219: intermediate tap block == 1x1 conv with that tap's slice
    k, M, C, H, W = 3, 2, 3, 5, 5
    x = oracle.fill(C * H * W, 146).reshape(C, H, W)
    w = oracle.fill(M * k * k * C, 147).reshape(M, k, k, C)
    inter = oracle.gemm_ref(oracle.kn2row_reorder(w), x.reshape(C, H * W))
    for i in range(k):
        for j in range(k):
            one = oracle.conv_kn2row(x, np.ascontiguousarray(w[:, i:i + 1, j:j + 1, :]))
            t = i * k + j
            assert np.array_equal(inter[t * M:(t + 1) * M], one.reshape(M, H * W))


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_oracle_matches_reference_fixtures(oracle, case):
    """Bitwise: the restated oracle == the reference library's own outputs."""
    name, C, H, W, M, k, seed = case
    g = np.load(GOLDEN)
    x, w = oracle.make_problem(1, C, H, W, M, k, seed)
    ds = oracle.conv_mcmk_sum(x[0], w)
    assert np.array_equal(ds.view(np.uint32), g[f"{name}/direct_sum"].view(np.uint32))
    assert oracle.fnv1a(ds) == int(g[f"{name}/fnv1a"][0])
    assert np.array_equal(oracle.conv_kn2row(x[0], w), g[f"{name}/kn2row"])
    assert np.array_equal(oracle.conv_im2col(x[0], w), g[f"{name}/im2col"])
    # the generalised loop nest at pad = k/2, stride 1 is the same function
    ln = oracle.conv_loopnest(x, w, k // 2, 1)[0]
    assert oracle.ref_allclose(ln, ds)


def test_oracle_bitwise_vs_live_reference(oracle):
    """Live check against oracle/_ref (skipped where the reference was not compiled)."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    x, w = oracle.make_problem(1, 64, 28, 28, 32, 3, 0)
    for method, fn in (("direct-sum", oracle.conv_mcmk_sum), ("kn2row", oracle.conv_kn2row),
                       ("im2col", oracle.conv_im2col)):
        assert np.array_equal(fn(x[0], w), oracle.ref_run_method(method, x[0], w)), method
    # the batch convention: image 0 of a batch stream is the reference benchmark() input
    xb, _ = oracle.make_problem(3, 4, 5, 5, 2, 3, 0)
    x0, _ = oracle.make_problem(1, 4, 5, 5, 2, 3, 0)
    assert np.array_equal(xb[0], x0[0])


def test_loopnest_pad_stride_generalisation(oracle):
    """pad/stride beyond the reference (SURVEY 8c gap): check against a float64 numpy
    restatement of the same loop nest."""
    x, w = oracle.make_problem(2, 3, 9, 7, 4, 3, 21)
    for pad, stride in ((0, 1), (1, 2), (2, 1), (0, 2)):
        y = oracle.conv_loopnest(x, w, pad, stride)
        N, C, H, W = x.shape
        M, k = w.shape[:2]
        xp = np.zeros((N, C, H + 2 * pad, W + 2 * pad))
        xp[:, :, pad:pad + H, pad:pad + W] = x
        P, Q = y.shape[2:]
        ref = np.zeros((N, M, P, Q))
        for a in range(k):
            for b in range(k):
                patch = xp[:, :, a:a + stride * (P - 1) + 1:stride, b:b + stride * (Q - 1) + 1:stride]
                ref += np.einsum("nchw,mc->nmhw", patch, w[:, a, b, :].astype(np.float64))
        assert np.allclose(y, ref, rtol=1e-5, atol=1e-5)


def test_tolerance_law(oracle):
    # tensor_test.cpp allclose formula + verify's scaled tolerance (bench.cpp:191)
    a = oracle.fill(16, 9)
    assert oracle.ref_allclose(a, a)
    assert not oracle.ref_allclose(a + 1.0, a)
    m = oracle.parity_metrics(a * (1 + 1e-7), a)
    assert m["rel_l2"] < 2e-7 and m["allclose"]
