"""The reference's counter-based generator (tensor.cpp:104-134) for device-resident data.

split() is the host-side stream derivation (tensor.cpp:125-127); fill_uniform() runs the
value function unit_value(seed, i) on the GPU (cl_fill_uniform), bit-identical to
fill_deterministic, so synthetic inputs equal what the reference's benchmark()/verify()
would generate (bench.cpp:109-112, 173-176).
"""
from __future__ import annotations

import ctypes

from . import _lib

_M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
SPLIT_GAMMA = 0xD1B54A32D192ED03


def mix64(z: int) -> int:
    z &= _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def split(seed: int, lane: int) -> int:
    return mix64(seed + (lane + 1) * SPLIT_GAMMA)


def fill_uniform(t, seed: int, first_index: int = 0, stream=None):
    """Fills a contiguous CUDA fp32 tensor in place with unit_value(seed, first_index + i)."""
    import torch
    assert t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()
    s = stream if stream is not None else torch.cuda.current_stream()
    _lib.check(_lib.lib().cl_fill_uniform(ctypes.c_void_p(t.data_ptr()), t.numel(), seed & _M64, first_index,
                                          ctypes.c_void_p(s.cuda_stream)))
    return t


def make_problem(N: int, C: int, H: int, W: int, M: int, k: int, seed: int = 0, device: int = 0):
    """Seeded NCHW input (stream split(seed,0)) and MKKC weights (split(seed,1)) on the GPU."""
    import torch
    x = torch.empty((N, C, H, W), device=f"cuda:{device}", dtype=torch.float32)
    w = torch.empty((M, k, k, C), device=f"cuda:{device}", dtype=torch.float32)
    fill_uniform(x, split(seed, 0))
    fill_uniform(w, split(seed, 1))
    return x, w
