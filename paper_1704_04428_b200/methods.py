"""Host-side mirror of the reference operator interface for the conv hot path.

Reference: /root/reference/proj/core/include/convlab/{methods,layers,bench}.hpp
  - ConvMethod names + method_from_name / parse_method_list  (methods.cpp:11-61)
  - LayerConfig{name,C,H,W,M,k,stride}                       (layers.hpp:12-22), + pad, batch
  - run_method(method, problem, backend)                     (methods.cpp:65-88)
  - footprint(layer, method)                                 (bench.cpp:58-85)
  - the k == 1 routing rule: kn2row/kn2col -> conv1x1; conv1x1 with k != 1 raises
    (methods.cpp:75-85)

The GPU methods run only through libconvlab_b200.so (C ABI); torch supplies device memory
and streams.  The reference's CPU methods are listed by name so method lists parse the same,
but this package never executes them (they live in oracle/ as test infrastructure).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from . import _lib

# Reference method names in canonical order (methods.cpp:11-41) -- CPU, reference-only.
REFERENCE_METHODS = ["direct-sum", "direct-loopnest", "im2col", "im2row", "kn2row", "kn2col", "conv1x1"]
# GPU methods of this package (the -gpu suffix of SURVEY.md 8b) plus the selector.
GPU_METHODS = ["kn2row-gpu", "kn2row-explicit-gpu", "kn2col-gpu", "kn2row-acc-gpu", "im2col-gpu", "im2row-gpu",
               "conv1x1-gpu", "direct-gpu"]
ALL_METHODS = REFERENCE_METHODS + GPU_METHODS + ["auto"]
PRECISIONS = ("fp32", "tf32", "bf16")


def method_from_name(name: str) -> Optional[str]:
    return name if name in ALL_METHODS else None


def parse_method_list(csv: str) -> List[str]:
    """methods.cpp:43-61: comma list, empty items skipped, unknown -> ValueError."""
    out = []
    for item in csv.split(","):
        if not item:
            continue
        if method_from_name(item) is None:
            raise ValueError(f"unknown method '{item}'")
        out.append(item)
    if not out:
        raise ValueError("empty method list")
    return out


def method_requires_1x1(method: str) -> bool:
    return method in ("conv1x1", "conv1x1-gpu")


@dataclass
class LayerConfig:
    """layers.hpp:12-22 plus the two fields the GPU path needs: pad (default k/2, the
    reference's implicit padding, conv_direct.hpp:7-10) and batch N."""
    name: str
    channels: int
    height: int
    width: int
    kernel_count: int
    kernel_size: int
    stride: int = 1
    pad: Optional[int] = None
    batch: int = 1

    def __post_init__(self):
        if min(self.channels, self.height, self.width, self.kernel_count, self.kernel_size, self.batch) <= 0:
            raise ValueError(f"layer '{self.name}': zero dimension")
        if self.kernel_size % 2 == 0:
            raise ValueError(f"layer '{self.name}': kernel size must be odd, got {self.kernel_size}")
        if self.pad is None:
            self.pad = self.kernel_size // 2

    @property
    def out_height(self) -> int:
        return (self.height + 2 * self.pad - self.kernel_size) // self.stride + 1

    @property
    def out_width(self) -> int:
        return (self.width + 2 * self.pad - self.kernel_size) // self.stride + 1

    def flops(self) -> int:
        """Effective FLOPs 2 N M C k^2 P Q (padded taps counted)."""
        return (2 * self.batch * self.kernel_count * self.channels * self.kernel_size ** 2
                * self.out_height * self.out_width)

    def algorithmic_bytes(self) -> int:
        """Compulsory fp32 HBM bytes 4 (N C H W + M C k^2 + N M P Q)."""
        return 4 * (self.batch * self.channels * self.height * self.width
                    + self.kernel_count * self.channels * self.kernel_size ** 2
                    + self.batch * self.kernel_count * self.out_height * self.out_width)


def footprint(layer: LayerConfig, method: str) -> dict:
    """bench.cpp:58-85 closed forms (per image, as the reference), keyed like FootprintBytes.
    GPU methods report the intermediate they materialise: the implicit kernels none."""
    c, h, w, m, k = layer.channels, layer.height, layer.width, layer.kernel_count, layer.kernel_size
    fp = {"input_bytes": 4 * c * h * w, "kernel_bytes": 4 * m * k * k * c, "output_bytes": 4 * m * h * w}
    if method in ("im2col", "im2row", "im2col-gpu", "im2row-gpu"):
        inter = 4 * k * k * c * h * w
    elif method in ("kn2row", "kn2col", "kn2row-explicit-gpu", "kn2col-gpu"):
        inter = 4 * k * k * m * h * w
    else:  # direct methods, conv1x1, implicit / accumulating kn2row on the GPU
        inter = 0
    fp["intermediate_bytes"] = inter
    return fp


def parse_network_text(text: str, origin: str = "<text>") -> List[LayerConfig]:
    """layers.cpp:31-79 grammar: `name C H W M k [stride]`, `#` comments; errors name
    origin:line.  Two optional trailing columns extend it for the GPU path: `pad=P`
    and `n=N` (key=value so reference files parse unchanged)."""
    layers, seen = [], set()
    for no, raw in enumerate(text.splitlines(), 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        toks = line.split()
        kv = {}
        while toks and "=" in toks[-1]:
            key, _, val = toks.pop().partition("=")
            kv[key] = val
        if len(toks) not in (6, 7):
            raise RuntimeError(f"{origin}:{no}: expected `name C H W M k [stride]`")
        name = toks[0]
        try:
            nums = [int(t) for t in toks[1:]]
            pad = int(kv["pad"]) if "pad" in kv else None
            batch = int(kv.get("n", 1))
        except ValueError:
            raise RuntimeError(f"{origin}:{no}: non-integer field") from None
        if any(v <= 0 for v in nums):
            raise RuntimeError(f"{origin}:{no}: zero dimension")
        if nums[4] % 2 == 0:
            raise RuntimeError(f"{origin}:{no}: kernel size must be odd")
        if name in seen:
            raise RuntimeError(f"{origin}:{no}: duplicate layer name '{name}'")
        seen.add(name)
        stride = nums[5] if len(nums) == 6 else 1
        layers.append(LayerConfig(name, nums[0], nums[1], nums[2], nums[3], nums[4], stride, pad, batch))
    return layers


class ConvPlan:
    """One planned layer on one GPU (cl_conv_plan / set_weights / forward / destroy).

    Tensors are torch CUDA fp32 tensors: x [N,C,H,W], w [M,k,k,C] (MKKC), y [N,M,P,Q].
    """

    def __init__(self, layer: LayerConfig, method: str = "auto", precision: str = "fp32", device: int = 0):
        if method not in _lib.METHODS:
            raise ValueError(f"not a GPU method: '{method}' (choose from {sorted(_lib.METHODS)})")
        if precision not in _lib.PRECISIONS:
            raise ValueError(f"unknown precision '{precision}'")
        self.layer = layer
        self.precision = precision
        self.device = device
        L = _lib.lib()
        d = _lib.ConvDesc(layer.batch, layer.channels, layer.height, layer.width, layer.kernel_count,
                          layer.kernel_size, layer.pad, layer.stride)
        h = ctypes.c_void_p()
        _lib.check(L.cl_conv_plan(ctypes.byref(d), _lib.METHODS[method], _lib.PRECISIONS[precision], device,
                                  ctypes.byref(h)))
        self._h = h
        p, q = ctypes.c_int32(), ctypes.c_int32()
        _lib.check(L.cl_conv_output_dims(h, ctypes.byref(p), ctypes.byref(q)))
        self.out_hw = (p.value, q.value)
        self.method = _lib.METHOD_NAMES[L.cl_conv_resolved_method(h)]
        # operand format: 3xf16 / mixed / 3xtf32 (fp32-faithful), tf32 / bf16, fp32-fma (direct)
        self.split = L.cl_conv_operand_split(h).decode()

    # -- lifetime ------------------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().cl_conv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- compute -------------------------------------------------------------------------
    @staticmethod
    def _stream(stream):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream()
        return ctypes.c_void_p(s.cuda_stream)

    def workspace_bytes(self) -> int:
        return int(_lib.lib().cl_conv_workspace_bytes(self._h))

    def set_max_sms(self, max_sms: int):
        """Cap the SMs this plan's tcgen05 launches occupy (0 = all; cl_conv_set_max_sms)."""
        _lib.check(_lib.lib().cl_conv_set_max_sms(self._h, int(max_sms)))

    def launch_count(self) -> int:
        return int(_lib.lib().cl_conv_last_launch_count(self._h))

    def set_weights(self, w, stream=None):
        L = self.layer
        self._check_device_tensor(w, (L.kernel_count, L.kernel_size, L.kernel_size, L.channels), "w")
        _lib.check(_lib.lib().cl_conv_set_weights(self._h, ctypes.c_void_p(w.data_ptr()), self._stream(stream)))
        self._w = w  # keep alive until the async pack completes

    def set_weights_host(self, w_host, stream=None):
        """MKKC weights from a host tensor (cl_conv_set_weights_host: synchronous upload)."""
        L = self.layer
        self._check_host_tensor(w_host, L.kernel_count * L.kernel_size * L.kernel_size * L.channels, "w_host")
        _lib.check(_lib.lib().cl_conv_set_weights_host(self._h, ctypes.c_void_p(w_host.data_ptr()),
                                                       self._stream(stream)))

    def output_shape(self):
        return (self.layer.batch, self.layer.kernel_count, *self.out_hw)

    def _check_device_tensor(self, t, shape, what):
        """Every buffer handed to the C ABI: fp32, contiguous, on this plan's device, exactly the
        expected shape (a wrong buffer would make the kernels read or write out of bounds)."""
        import torch
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{what}: expected a torch tensor, got {type(t).__name__}")
        if not t.is_cuda or t.device.index != self.device:
            raise ValueError(f"{what}: must be on cuda:{self.device}, got {t.device}")
        if t.dtype != torch.float32:
            raise ValueError(f"{what}: must be float32, got {t.dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{what}: must be contiguous")
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"{what}: shape {tuple(t.shape)} != expected {tuple(shape)}")

    def _check_host_tensor(self, t, numel, what):
        import torch
        if not isinstance(t, torch.Tensor) or t.is_cuda:
            raise ValueError(f"{what}: expected a host (CPU) torch tensor")
        if t.dtype != torch.float32 or not t.is_contiguous():
            raise ValueError(f"{what}: must be contiguous float32")
        if t.numel() != numel:
            raise ValueError(f"{what}: {t.numel()} elements != expected {numel}")

    def input_shape(self, layout: str = "nchw"):
        L = self.layer
        return ((L.batch, L.channels, L.height, L.width) if layout == "nchw"
                else (L.batch, L.height, L.width, L.channels))

    def forward(self, x, y=None, workspace=None, stream=None, layout: str = "nchw"):
        """layout "nchw" (the reference's CHW images stacked) or "nhwc" (channels last, the
        reference's HWC layout; implicit kn2row / conv1x1 / kn2row-acc plans)."""
        import torch
        L = self.layer
        if layout not in ("nchw", "nhwc"):
            raise ValueError(f"layout must be 'nchw' or 'nhwc', got '{layout}'")
        self._check_device_tensor(x, self.input_shape(layout), "x")
        out_shape = self.output_shape() if layout == "nchw" else (L.batch, *self.out_hw, L.kernel_count)
        if y is None:
            y = torch.empty(out_shape, device=x.device, dtype=torch.float32)
        self._check_device_tensor(y, out_shape, "y")
        if workspace is not None:
            if not workspace.is_cuda or workspace.device.index != self.device or not workspace.is_contiguous():
                raise ValueError(f"workspace: must be a contiguous tensor on cuda:{self.device}")
            have = workspace.numel() * workspace.element_size()
            if have < self.workspace_bytes():
                raise ValueError(f"workspace: {have} bytes < required {self.workspace_bytes()}")
        ws = ctypes.c_void_p(workspace.data_ptr()) if workspace is not None else None
        fn = _lib.lib().cl_conv_forward if layout == "nchw" else _lib.lib().cl_conv_forward_nhwc
        _lib.check(fn(self._h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), ws, self._stream(stream)))
        return y

    def _check_host_io(self, x_host, y_host):
        L = self.layer
        self._check_host_tensor(x_host, L.batch * L.channels * L.height * L.width, "x_host")
        self._check_host_tensor(y_host, L.batch * L.kernel_count * self.out_hw[0] * self.out_hw[1], "y_host")

    def forward_host_async(self, x_host, y_host, stream=None):
        """Host-buffer call that returns after enqueueing (synchronise `stream` before reading
        y_host).  The copy-in is ordered after prior work on `stream` (so a previous layer's
        host output can be this call's input); independent layers overlap their transfers when
        each is issued on its own stream."""
        self._check_host_io(x_host, y_host)
        _lib.check(_lib.lib().cl_conv_forward_host_async(self._h, ctypes.c_void_p(x_host.data_ptr()),
                                                         ctypes.c_void_p(y_host.data_ptr()), self._stream(stream)))
        return y_host

    def forward_host(self, x_host, y_host, stream=None):
        """End-to-end host-buffer call (H2D + forward + D2H, synchronous)."""
        self._check_host_io(x_host, y_host)
        _lib.check(_lib.lib().cl_conv_forward_host(self._h, ctypes.c_void_p(x_host.data_ptr()),
                                                   ctypes.c_void_p(y_host.data_ptr()), self._stream(stream)))
        return y_host


def forward_chain(plans: Sequence["ConvPlan"], xs, ys, workspaces=None, stream=None):
    """One step of independent-or-chained layers on one stream (cl_conv_forward_chain): layer
    i+1's NCHW -> split prepass rides on layer i's contraction (its converter warps), a tail
    launch finishes it.  xs / ys: NCHW CUDA tensors per plan; results equal per-plan forwards."""
    n = len(plans)
    if not (len(xs) == len(ys) == n) or (workspaces is not None and len(workspaces) != n):
        raise ValueError("forward_chain: one x, y (and workspace) per plan")
    for p, x, y, ws in zip(plans, xs, ys, workspaces or [None] * n):
        p._check_device_tensor(x, p.input_shape("nchw"), "x")
        p._check_device_tensor(y, p.output_shape(), "y")
        if ws is not None and ws.numel() * ws.element_size() < p.workspace_bytes():
            raise ValueError(f"workspace: {ws.numel() * ws.element_size()} bytes < required {p.workspace_bytes()}")
    arr = ctypes.c_void_p * n
    ph = arr(*[p._h.value for p in plans])
    xh = arr(*[x.data_ptr() for x in xs])
    yh = arr(*[y.data_ptr() for y in ys])
    wh = arr(*[(w.data_ptr() if w is not None else None) for w in (workspaces or [None] * n)])
    _lib.check(_lib.lib().cl_conv_forward_chain(ph, xh, yh, wh, n, ConvPlan._stream(stream)))
    return ys


def run_method(method: str, x, w, precision: str = "fp32", pad: Optional[int] = None, stride: int = 1):
    """Functional form of methods.cpp:65-88 for GPU methods: x [N,C,H,W] and w [M,k,k,C]
    torch CUDA tensors -> y [N,M,P,Q].  Applies the reference's k == 1 routing."""
    N, C, H, W = x.shape
    M, k, k2, C2 = w.shape
    if C != C2:
        raise ValueError(f"ConvProblem: input has {C} channels, kernels have {C2}")
    if k != k2:
        raise ValueError("kernels must be square")
    layer = LayerConfig("run_method", C, H, W, M, k, stride, pad, N)
    with ConvPlan(layer, method, precision, x.device.index or 0) as plan:
        plan.set_weights(w.contiguous())
        return plan.forward(x.contiguous())


def gemm(a, b, precision: str = "fp32", out=None):
    """C = A.B on the tcgen05 engine (row-major fp32, the reference gemm() contract)."""
    import torch
    m, k = a.shape
    k2, n = b.shape
    if k != k2:
        raise ValueError(f"gemm: inner dimensions differ, a is {m}x{k}, b is {k2}x{n}")
    c = out if out is not None else torch.empty((m, n), device=a.device, dtype=torch.float32)
    s = torch.cuda.current_stream()
    _lib.check(_lib.lib().cl_gemm_f32(m, n, k, ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()),
                                      ctypes.c_void_p(c.data_ptr()), _lib.PRECISIONS[precision], None, 0,
                                      ctypes.c_void_p(s.cuda_stream)))
    return c


def shift_add_row(inter, n: int, m: int, h: int, w: int, k: int, pad: Optional[int] = None):
    """Device shift_add (row orientation) over inter[(k^2 m) x (n h w)] -> y [n, m, P, Q]."""
    import torch
    pad = k // 2 if pad is None else pad
    P, Q = h + 2 * pad - k + 1, w + 2 * pad - k + 1
    y = torch.empty((n, m, P, Q), device=inter.device, dtype=torch.float32)
    s = torch.cuda.current_stream()
    _lib.check(_lib.lib().cl_shift_add_row(ctypes.c_void_p(inter.data_ptr()), ctypes.c_void_p(y.data_ptr()), n, m,
                                           h, w, k, pad, ctypes.c_void_p(s.cuda_stream)))
    return y
