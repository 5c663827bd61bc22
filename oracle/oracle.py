"""TEST INFRASTRUCTURE ONLY -- numpy/ctypes front-end of the CPU oracle.

Loads ``oracle/liboracle.so`` (the C restatement in ``oracle.c``) and, when present,
``oracle/_ref/libconvlab_ref.so`` (the unmodified reference core compiled from
``/root/reference/proj/core`` by ``oracle/Makefile``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / reference arm may import
this module; the product package never does.

Every function cites the reference routine it restates (see oracle.c for line numbers).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"
REF_PATH = HERE / "_ref" / "libconvlab_ref.so"

_f32p = ctypes.POINTER(ctypes.c_float)
_u64 = ctypes.c_uint64
_i = ctypes.c_int


def build(force: bool = False) -> None:
    """Builds liboracle.so and (when /root/reference exists) _ref/libconvlab_ref.so."""
    if force or not LIB_PATH.exists() or (not REF_PATH.exists() and Path("/root/reference").exists()):
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def _load(path: Path) -> ctypes.CDLL:
    if not path.exists():
        build()
    return ctypes.CDLL(str(path))


_lib = None
_ref = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        L = _load(LIB_PATH)
        L.orc_mix64.restype = _u64
        L.orc_mix64.argtypes = [_u64]
        L.orc_unit_value.restype = ctypes.c_float
        L.orc_unit_value.argtypes = [_u64, _u64]
        L.orc_split.restype = _u64
        L.orc_split.argtypes = [_u64, _u64]
        L.orc_fill.argtypes = [_f32p, _u64, _u64, _u64]
        L.orc_fnv1a.restype = _u64
        L.orc_fnv1a.argtypes = [_f32p, _u64]
        L.orc_conv2d_scsk.argtypes = [_f32p, _i, _i, _f32p, _i, _f32p]
        L.orc_conv_mcmk_sum.argtypes = [_f32p, _f32p, _f32p] + [_i] * 5
        L.orc_conv_loopnest.argtypes = [_f32p, _f32p, _f32p] + [_i] * 8
        L.orc_gemm_ref.argtypes = [_f32p, _f32p, _f32p, _i, _i, _i]
        L.orc_kn2row_reorder.argtypes = [_f32p, _f32p, _i, _i, _i]
        L.orc_shift_add_row.argtypes = [_f32p, _f32p, _i, _i, _i, _i]
        L.orc_shift_add_col.argtypes = [_f32p, _f32p, _i, _i, _i, _i]
        L.orc_conv_kn2row.argtypes = [_f32p, _f32p, _f32p] + [_i] * 5
        L.orc_im2col_patch.argtypes = [_f32p, _f32p, _i, _i, _i, _i]
        L.orc_conv_im2col.argtypes = [_f32p, _f32p, _f32p] + [_i] * 5
        L.orc_max_abs.restype = ctypes.c_float
        L.orc_max_abs.argtypes = [_f32p, _u64]
        L.orc_allclose_scaled.restype = _i
        L.orc_allclose_scaled.argtypes = [_f32p, _f32p, _u64, ctypes.c_float, ctypes.c_float]
        _lib = L
    return _lib


def ref_available() -> bool:
    if not REF_PATH.exists() and Path("/root/reference").exists():
        build()
    return REF_PATH.exists()


def ref() -> ctypes.CDLL:
    """The unmodified reference library (oracle/_ref)."""
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError(f"reference library not built: {REF_PATH}")
        R = ctypes.CDLL(str(REF_PATH))
        R.ref_last_error.restype = ctypes.c_char_p
        R.ref_unit_value.restype = ctypes.c_float
        R.ref_unit_value.argtypes = [_u64, _u64]
        R.ref_split.restype = _u64
        R.ref_split.argtypes = [_u64, _u64]
        R.ref_run_method.argtypes = [ctypes.c_char_p, _i, _f32p, _f32p, _f32p] + [_i] * 5
        R.ref_shift_add_row.argtypes = [_f32p, _f32p, _i, _i, _i, _i]
        R.ref_footprint.argtypes = [ctypes.c_char_p] + [_i] * 5 + [ctypes.POINTER(_u64)]
        R.ref_benchmark.argtypes = ([ctypes.c_char_p] + [_i] * 7 + [_u64, ctypes.POINTER(ctypes.c_double),
                                                                    ctypes.POINTER(_u64)])
        R.ref_hardware_threads.restype = _i
        _ref = R
    return _ref


def _p(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags["C_CONTIGUOUS"], (a.dtype, a.flags)
    return a.ctypes.data_as(_f32p)


# ---- generator (tensor.cpp:104-134) ------------------------------------------------

def split(seed: int, lane: int) -> int:
    return int(lib().orc_split(seed, lane))


def fill(n: int, seed: int, first_index: int = 0) -> np.ndarray:
    out = np.empty(n, dtype=np.float32)
    lib().orc_fill(_p(out), n, seed, first_index)
    return out


def make_problem(N: int, C: int, H: int, W: int, M: int, k: int, seed: int = 0):
    """Seeded NCHW input and MKKC weights, SURVEY.md 8(d) convention: input = one stream
    split(seed, 0) over all N*C*H*W values (image 0 == reference benchmark() input,
    bench.cpp:109-112), weights = split(seed, 1)."""
    x = fill(N * C * H * W, split(seed, 0)).reshape(N, C, H, W)
    w = fill(M * k * k * C, split(seed, 1)).reshape(M, k, k, C)
    return x, w


def fnv1a(a: np.ndarray) -> int:
    a = np.ascontiguousarray(a, dtype=np.float32)
    return int(lib().orc_fnv1a(_p(a), a.size))


# ---- conv methods --------------------------------------------------------------------

def conv_mcmk_sum(x_chw: np.ndarray, w_mkkc: np.ndarray) -> np.ndarray:
    """THE ORACLE: conv_mcmk_sum (conv_direct.cpp:93-102), one CHW image."""
    C, H, W = x_chw.shape
    M, k, _, C2 = w_mkkc.shape
    assert C == C2
    y = np.empty((M, H, W), dtype=np.float32)
    lib().orc_conv_mcmk_sum(_p(np.ascontiguousarray(x_chw)), _p(np.ascontiguousarray(w_mkkc)), _p(y),
                            C, H, W, M, k)
    return y


def conv_batch(x_nchw: np.ndarray, w_mkkc: np.ndarray, images=None) -> np.ndarray:
    """conv_mcmk_sum per image (the reference has no batch dim; images are independent).
    ``images`` restricts to a sample of image indices (returns only those)."""
    N = x_nchw.shape[0]
    idx = range(N) if images is None else images
    return np.stack([conv_mcmk_sum(x_nchw[n], w_mkkc) for n in idx])


def conv_loopnest(x_nchw: np.ndarray, w_mkkc: np.ndarray, pad: int, stride: int = 1) -> np.ndarray:
    """conv_mcmk_loopnest (conv_direct.cpp:104-143) generalised to (pad, stride), batched."""
    N, C, H, W = x_nchw.shape
    M, k, _, _ = w_mkkc.shape
    P = (H + 2 * pad - k) // stride + 1
    Q = (W + 2 * pad - k) // stride + 1
    y = np.empty((N, M, P, Q), dtype=np.float32)
    lib().orc_conv_loopnest(_p(np.ascontiguousarray(x_nchw)), _p(np.ascontiguousarray(w_mkkc)), _p(y),
                            N, C, H, W, M, k, pad, stride)
    return y


def conv2d_scsk(img: np.ndarray, ker: np.ndarray) -> np.ndarray:
    H, W = img.shape
    k = ker.shape[0]
    out = np.empty((H, W), dtype=np.float32)
    lib().orc_conv2d_scsk(_p(np.ascontiguousarray(img, np.float32)), H, W,
                          _p(np.ascontiguousarray(ker, np.float32)), k, _p(out))
    return out


def kn2row_reorder(w_mkkc: np.ndarray) -> np.ndarray:
    M, k, _, C = w_mkkc.shape
    r = np.empty((k * k * M, C), dtype=np.float32)
    lib().orc_kn2row_reorder(_p(np.ascontiguousarray(w_mkkc)), _p(r), M, k, C)
    return r


def gemm_ref(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    m, p = a.shape
    p2, n = b.shape
    assert p == p2
    c = np.empty((m, n), dtype=np.float32)
    lib().orc_gemm_ref(_p(np.ascontiguousarray(a)), _p(np.ascontiguousarray(b)), _p(c), m, p, n)
    return c


def shift_add_row(inter: np.ndarray, k: int, M: int, H: int, W: int) -> np.ndarray:
    out = np.empty((M, H * W), dtype=np.float32)
    lib().orc_shift_add_row(_p(np.ascontiguousarray(inter, np.float32)), _p(out), k, M, H, W)
    return out


def shift_add_col(inter: np.ndarray, k: int, M: int, H: int, W: int) -> np.ndarray:
    out = np.empty((H * W, M), dtype=np.float32)
    lib().orc_shift_add_col(_p(np.ascontiguousarray(inter, np.float32)), _p(out), k, M, H, W)
    return out


def conv_kn2row(x_chw: np.ndarray, w_mkkc: np.ndarray) -> np.ndarray:
    C, H, W = x_chw.shape
    M, k, _, _ = w_mkkc.shape
    y = np.empty((M, H, W), dtype=np.float32)
    lib().orc_conv_kn2row(_p(np.ascontiguousarray(x_chw)), _p(np.ascontiguousarray(w_mkkc)), _p(y),
                          C, H, W, M, k)
    return y


def im2col_patch(x_chw: np.ndarray, k: int) -> np.ndarray:
    C, H, W = x_chw.shape
    pm = np.empty((k * k * C, H * W), dtype=np.float32)
    lib().orc_im2col_patch(_p(np.ascontiguousarray(x_chw, np.float32)), _p(pm), C, H, W, k)
    return pm


def conv_im2col(x_chw: np.ndarray, w_mkkc: np.ndarray) -> np.ndarray:
    C, H, W = x_chw.shape
    M, k, _, _ = w_mkkc.shape
    y = np.empty((M, H, W), dtype=np.float32)
    lib().orc_conv_im2col(_p(np.ascontiguousarray(x_chw)), _p(np.ascontiguousarray(w_mkkc)), _p(y),
                          C, H, W, M, k)
    return y


# ---- tolerance laws ------------------------------------------------------------------

def ref_allclose(a: np.ndarray, oracle: np.ndarray, rel: float = 1e-5, abs_: float = 1e-6) -> bool:
    """allclose at scaled_tolerance({rel, abs}, max|oracle|) -- verify(), bench.cpp:191-205."""
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(oracle, np.float32)
    assert a.shape == b.shape
    return bool(lib().orc_allclose_scaled(_p(a), _p(b), a.size, rel, abs_))


def parity_metrics(out: np.ndarray, oracle: np.ndarray) -> dict:
    """North-star parity metrics: rel-L2 and max|d|/max|ref| in fp64,
    plus the reference allclose verdict."""
    o = np.asarray(out, np.float64)
    r = np.asarray(oracle, np.float64)
    diff = o - r
    denom = float(np.linalg.norm(r)) or 1.0
    mx = float(np.max(np.abs(r))) if r.size else 0.0
    return {
        "rel_l2": float(np.linalg.norm(diff)) / denom,
        "max_rel": (float(np.max(np.abs(diff))) / mx) if mx > 0 else float(np.max(np.abs(diff), initial=0.0)),
        "allclose": ref_allclose(out, oracle),
        "finite": bool(np.isfinite(o).all()),
    }


# ---- reference library wrappers (oracle/_ref) ----------------------------------------

def ref_run_method(method: str, x_chw: np.ndarray, w_mkkc: np.ndarray, threads: int = 0) -> np.ndarray:
    C, H, W = x_chw.shape
    M, k, _, _ = w_mkkc.shape
    y = np.empty((M, H, W), dtype=np.float32)
    R = ref()
    rc = R.ref_run_method(method.encode(), threads, _p(np.ascontiguousarray(x_chw)),
                          _p(np.ascontiguousarray(w_mkkc)), _p(y), C, H, W, M, k)
    if rc == 1:
        raise ValueError(R.ref_last_error().decode())
    if rc != 0:
        raise RuntimeError(R.ref_last_error().decode())
    return y


def ref_benchmark(method: str, C: int, H: int, W: int, M: int, k: int, runs: int, threads: int,
                  seed: int = 0) -> dict:
    stats = (ctypes.c_double * 3)()
    chk = _u64()
    R = ref()
    rc = R.ref_benchmark(method.encode(), threads, C, H, W, M, k, runs, seed, stats, ctypes.byref(chk))
    if rc != 0:
        raise RuntimeError(R.ref_last_error().decode())
    return {"mean_s": stats[0], "min_s": stats[1], "stddev_s": stats[2], "checksum": int(chk.value)}


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
