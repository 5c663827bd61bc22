"""ctypes binding of the C ABI in include/convlab_b200.h (libconvlab_b200.so).

There is no fallback: if the library is missing or cannot be loaded this module raises,
and every compute entry point returns an error on a host without an sm_100 GPU.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libconvlab_b200.so"

# cl_status
CL_OK, CL_EINVAL, CL_EUNSUPPORTED, CL_ECUDA, CL_ENOMEM, CL_ENODEVICE, CL_EINTERNAL = range(7)
# cl_method
METHODS = {
    "auto": 0,
    "kn2row-gpu": 1,
    "kn2row-explicit-gpu": 2,
    "kn2col-gpu": 3,
    "kn2row-acc-gpu": 4,
    "im2col-gpu": 5,
    "conv1x1-gpu": 6,
    "direct-gpu": 7,
    "im2row-gpu": 8,
}
METHOD_NAMES = {v: k for k, v in METHODS.items()}
# cl_precision
PRECISIONS = {"fp32": 0, "tf32": 1, "bf16": 2}

EXPORTS = [
    "cl_conv_plan", "cl_conv_set_weights", "cl_conv_set_weights_host", "cl_conv_output_dims", "cl_conv_workspace_bytes",
    "cl_conv_resolved_method", "cl_conv_operand_split", "cl_conv_forward", "cl_conv_forward_nhwc", "cl_conv_forward_host", "cl_conv_forward_host_async", "cl_conv_last_launch_count",
    "cl_conv_destroy", "cl_gemm_f32", "cl_gemm_workspace_bytes", "cl_shift_add_row", "cl_last_error",
    "cl_method_name", "cl_method_from_name", "cl_abi_version", "cl_device_count", "cl_fill_uniform",
    "cl_conv_set_profile_events", "cl_conv_set_max_sms", "cl_conv_forward_chain", "cl_conv_set_peer_outputs",
    "cl_ipc_get_mem_handle", "cl_ipc_open_mem_handle", "cl_ipc_close_mem_handle", "cl_checksum_fnv1a",
]


class ConvDesc(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in ("n", "c", "h", "w", "m", "k", "pad", "stride")]


class ClError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[cl_status {status}] {msg}")
        self.status = status


class ClInvalid(ClError, ValueError):
    """CL_EINVAL: the reference's std::invalid_argument."""


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1704_04428_b200.build_ext` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(str(LIB_PATH))
    vp, sz, i32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
    L.cl_conv_plan.argtypes = [ctypes.POINTER(ConvDesc), i32, i32, i32, ctypes.POINTER(vp)]
    L.cl_conv_set_weights.argtypes = [vp, vp, vp]
    L.cl_conv_set_weights_host.argtypes = [vp, vp, vp]
    L.cl_conv_output_dims.argtypes = [vp, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]
    L.cl_conv_workspace_bytes.restype = sz
    L.cl_conv_workspace_bytes.argtypes = [vp]
    L.cl_conv_resolved_method.argtypes = [vp]
    L.cl_conv_operand_split.argtypes = [vp]
    L.cl_conv_operand_split.restype = ctypes.c_char_p
    L.cl_conv_forward.argtypes = [vp, vp, vp, vp, vp]
    L.cl_conv_forward_nhwc.argtypes = [vp, vp, vp, vp, vp]
    L.cl_conv_forward_host.argtypes = [vp, vp, vp, vp]
    L.cl_conv_forward_host_async.argtypes = [vp, vp, vp, vp]
    L.cl_conv_last_launch_count.argtypes = [vp]
    L.cl_conv_destroy.argtypes = [vp]
    L.cl_conv_destroy.restype = None
    L.cl_gemm_f32.argtypes = [i32, i32, i32, vp, vp, vp, i32, vp, sz, vp]
    L.cl_gemm_workspace_bytes.restype = sz
    L.cl_gemm_workspace_bytes.argtypes = [i32, i32, i32, i32]
    L.cl_shift_add_row.argtypes = [vp, vp, i32, i32, i32, i32, i32, i32, vp]
    L.cl_fill_uniform.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, vp]
    L.cl_conv_set_profile_events.argtypes = [vp, vp, vp]
    L.cl_conv_set_max_sms.argtypes = [vp, i32]
    L.cl_conv_set_peer_outputs.argtypes = [vp, ctypes.POINTER(vp), i32, i32, i32]
    L.cl_ipc_get_mem_handle.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_uint64)]
    L.cl_ipc_open_mem_handle.argtypes = [vp, ctypes.POINTER(vp)]
    L.cl_ipc_close_mem_handle.argtypes = [vp]
    L.cl_conv_forward_chain.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp),
                                        i32, vp]
    L.cl_checksum_fnv1a.restype = ctypes.c_uint64
    L.cl_checksum_fnv1a.argtypes = [vp, ctypes.c_uint64]
    L.cl_last_error.restype = ctypes.c_char_p
    L.cl_method_name.restype = ctypes.c_char_p
    L.cl_method_name.argtypes = [i32]
    L.cl_method_from_name.argtypes = [ctypes.c_char_p, ctypes.POINTER(i32)]
    _lib = L
    return L


def check(status: int) -> None:
    if status == CL_OK:
        return
    msg = lib().cl_last_error().decode()
    if status == CL_EINVAL:
        raise ClInvalid(status, msg)
    raise ClError(status, msg)
