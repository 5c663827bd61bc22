"""Multi-GPU plumbing for the batch-sharded path.

One process per GPU (torchrun), images are independent, so ranks share nothing on the data
path: rank r owns a contiguous image range and generates / convolves it locally.  The only
collectives are control-plane: a barrier around the timed region and a MAX all-reduce of
the per-rank device times (the job time is the slowest rank's).
"""
from __future__ import annotations

import os
from dataclasses import dataclass


@dataclass
class RankInfo:
    rank: int = 0
    world: int = 1
    local_rank: int = 0

    @property
    def distributed(self) -> bool:
        return self.world > 1


def from_env() -> RankInfo:
    return RankInfo(int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
                    int(os.environ.get("LOCAL_RANK", 0)))


def init(backend: str = "nccl") -> RankInfo:
    info = from_env()
    if info.distributed:
        import torch.distributed as dist
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            kw = {}
            if backend == "nccl":
                import torch
                torch.cuda.set_device(info.local_rank)
                kw["device_id"] = torch.device(f"cuda:{info.local_rank}")
            dist.init_process_group(backend, **kw)
    return info


def shard_range(total: int, world: int, rank: int) -> tuple:
    """Contiguous, balanced split of `total` images: the first total % world ranks get one
    extra.  Strong-scaling helper (weak scaling gives every rank the full per-GPU batch)."""
    base, extra = divmod(total, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def image_offset(rank: int, per_rank_batch: int, image_elems: int) -> int:
    """First generator index of rank r's images when all ranks' images form ONE reference
    stream (so rank r's data equals images [r B, (r+1) B) of the global batch)."""
    return rank * per_rank_batch * image_elems


def barrier(info: RankInfo) -> None:
    if info.distributed:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(value: float, info: RankInfo, device=None) -> float:
    if not info.distributed:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, info: RankInfo, device=None) -> float:
    if not info.distributed:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ------------------------------------------------------------ output-channel sharding ----
# SURVEY.md 8(e) alternative for small-batch layers (C1, AlexNet b1) where batch sharding has
# nothing to split: rank g computes kernels [g M/G, (g+1) M/G) for every image (each rank
# reads the whole input, weights are sliced once), then one all-gather (NCCL over NVLink /
# NVSwitch on GPUs) assembles the NCHW output.  The gather lands rank-major
# [G][N][M/G][PQ]; one permute copy restores NCHW.  Optional and off the measured path.

def channel_slice(m: int, world: int, rank: int) -> tuple:
    """Balanced contiguous kernel (output-channel) range of `rank`; requires m >= world."""
    return shard_range(m, world, rank)


def mshard_conv(x, w_mkkc, info: RankInfo, conv_fn, m_total: int = None):
    """y = conv(x, w) with the M dimension sharded over ranks.

    x: [N, C, H, W] (every rank holds all of it), w_mkkc: [M, k, k, C] full weights (or None
    with `m_total` when the callable already holds its slice, as MShardPlan's plan does),
    conv_fn(x, w_slice) -> y_slice [N, M_g, P, Q] runs this rank's share (the B200 plan in
    the product, any callable in tests).  Returns the full y [N, M, P, Q] on every rank.
    """
    import torch
    import torch.distributed as dist

    M = w_mkkc.shape[0] if w_mkkc is not None else m_total
    if M < info.world:
        raise ValueError(f"cannot shard {M} kernels over {info.world} ranks")
    b, e = channel_slice(M, info.world, info.rank)
    y_local = conv_fn(x, w_mkkc[b:e].contiguous() if w_mkkc is not None else None)
    if not (dist.is_available() and dist.is_initialized()):
        return y_local          # single process: the slice is the whole output
    N, _, P, Q = y_local.shape
    # uneven slices: pad every rank's block to the largest slice so one collective suffices
    mg = max(channel_slice(M, info.world, r)[1] - channel_slice(M, info.world, r)[0] for r in range(info.world))
    send = y_local
    if e - b < mg:
        send = torch.zeros((N, mg, P, Q), dtype=y_local.dtype, device=y_local.device)
        send[:, : e - b] = y_local
    gathered = torch.empty((info.world, N, mg, P, Q), dtype=y_local.dtype, device=y_local.device)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(gathered, send.contiguous())   # one NCCL all-gather over NVLink
    else:                                                          # gloo (CPU tests)
        dist.all_gather(list(gathered.unbind(0)), send.contiguous())
    y = torch.empty((N, M, P, Q), dtype=y_local.dtype, device=y_local.device)
    for r in range(info.world):
        rb, re_ = channel_slice(M, info.world, r)
        y[:, rb:re_] = gathered[r, :, : re_ - rb]
    return y


class MShardPlan:
    """Output-channel-sharded layer on a real B200 plan (SURVEY.md 8(e) alternative): rank g
    plans kernels [g M/G, (g+1) M/G) (dist.channel_slice) with its own ConvPlan, convolves the
    whole input, and `mshard_conv`'s all-gather assembles the NCHW output on every rank --
    NCCL (all_gather_into_tensor over NVLink / NVSwitch) for device tensors, gloo for the host
    path.  Weights are sliced and packed once (set_weights).  Optional, off the measured path:
    it serves batch-1 layers (C1, AlexNet b1, the C5 k-sweep) that batch sharding cannot split.
    """

    def __init__(self, layer, info: RankInfo, method: str = "auto", precision: str = "fp32", device: int = None,
                 fused: bool = False):
        import dataclasses
        from .methods import ConvPlan
        if layer.kernel_count < info.world:
            raise ValueError(f"cannot shard {layer.kernel_count} kernels over {info.world} ranks")
        self.layer, self.info = layer, info
        self.m0, self.m1 = channel_slice(layer.kernel_count, info.world, info.rank)
        self.device = info.local_rank if device is None else device
        if fused and method == "auto":
            # the fused gather lives in the implicit / conv1x1 epilogue (not the explicit GEMM +
            # shift-add the timing cache may pick for a small slice)
            method = "conv1x1-gpu" if layer.kernel_size == 1 else "kn2row-gpu"
        self.plan = ConvPlan(dataclasses.replace(layer, kernel_count=self.m1 - self.m0), method, precision,
                             self.device)
        self.fused = fused
        self._opened = []
        if fused:
            self._setup_fused()

    def _setup_fused(self):
        """Fused all-gather: every rank allocates its FULL output, the ranks exchange CUDA IPC handles
        (over the process group), and this rank's plan writes its channel slice into every rank's
        output from its epilogue (cl_conv_set_peer_outputs: P2P stores over NVLink / NVSwitch, the
        gather overlapping the contraction) -- no collective on the data path."""
        import ctypes
        import torch
        import torch.distributed as dist
        from . import _lib
        L = self.layer
        self.y_full = torch.empty((L.batch, L.kernel_count, *self.plan.out_hw), device=f"cuda:{self.device}",
                                  dtype=torch.float32)
        h = (ctypes.c_char * 64)()
        off = ctypes.c_uint64()
        _lib.check(_lib.lib().cl_ipc_get_mem_handle(ctypes.c_void_p(self.y_full.data_ptr()), h, ctypes.byref(off)))
        handles = [(bytes(h), off.value)]
        if dist.is_available() and dist.is_initialized():
            handles = [None] * self.info.world
            dist.all_gather_object(handles, (bytes(h), off.value))
        ptrs = []
        for r, (hb, offset) in enumerate(handles):
            if r == self.info.rank:
                ptrs.append(self.y_full.data_ptr())
                continue
            base = ctypes.c_void_p()
            _lib.check(_lib.lib().cl_ipc_open_mem_handle(ctypes.create_string_buffer(hb, 64), ctypes.byref(base)))
            self._opened.append(base.value)
            ptrs.append(base.value + offset)   # the peer tensor sits `offset` bytes into its allocation
        arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
        _lib.check(_lib.lib().cl_conv_set_peer_outputs(self.plan._h, arr, len(ptrs), self.m0, L.kernel_count))

    @property
    def method(self):
        return self.plan.method

    @property
    def split(self):
        """Operand format of this rank's slice plan (bench.py's per-layer peak follows it)."""
        return self.plan.split

    def set_weights(self, w_full):
        """w_full: the FULL [M, k, k, C] weights (device tensor); this rank keeps its slice."""
        self.plan.set_weights(w_full[self.m0:self.m1].contiguous())

    def set_weights_host(self, w_full):
        self.plan.set_weights_host(w_full[self.m0:self.m1].contiguous())

    def output_shape(self):
        L = self.layer
        return (L.batch, L.kernel_count, *self.plan.out_hw)

    def forward(self, x):
        """x: full [N, C, H, W] device tensor on every rank -> full y (NCCL all-gather, or the
        fused epilogue stores + a stream sync and a barrier)."""
        if self.fused:
            import ctypes
            import torch
            import torch.distributed as dist
            from . import _lib
            self.plan._check_device_tensor(x, self.plan.input_shape("nchw"), "x")
            s = torch.cuda.current_stream()
            # y_full stands in for the slice output (the epilogue writes the peers' full outputs)
            _lib.check(_lib.lib().cl_conv_forward(self.plan._h, ctypes.c_void_p(x.data_ptr()),
                                                  ctypes.c_void_p(self.y_full.data_ptr()), None,
                                                  ctypes.c_void_p(s.cuda_stream)))
            s.synchronize()                  # this rank's stores (to every rank) are complete
            if dist.is_available() and dist.is_initialized():
                dist.barrier()               # ... and every other rank's into this one
            return self.y_full
        return mshard_conv(x, None, self.info, lambda xx, _w: self.plan.forward(xx),
                           m_total=self.layer.kernel_count)

    def forward_host(self, x_host):
        """Host path: H2D + forward + D2H of this rank's slice, gathered on the host (gloo)."""
        import torch

        def conv(xx, _w):
            y = torch.empty((self.layer.batch, self.m1 - self.m0, *self.plan.out_hw), dtype=torch.float32)
            return self.plan.forward_host(xx.contiguous(), y)
        return mshard_conv(x_host, None, self.info, conv, m_total=self.layer.kernel_count)

    def close(self):
        from . import _lib
        for ptr in self._opened:
            _lib.lib().cl_ipc_close_mem_handle(ptr)
        self._opened = []
        self.plan.close()
