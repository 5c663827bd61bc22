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


def mshard_conv(x, w_mkkc, info: RankInfo, conv_fn):
    """y = conv(x, w) with the M dimension sharded over ranks.

    x: [N, C, H, W] (every rank holds all of it), w_mkkc: [M, k, k, C] full weights,
    conv_fn(x, w_slice) -> y_slice [N, M_g, P, Q] runs this rank's share (the B200 plan in
    the product, any callable in tests).  Returns the full y [N, M, P, Q] on every rank.
    """
    import torch
    import torch.distributed as dist

    M = w_mkkc.shape[0]
    if M < info.world:
        raise ValueError(f"cannot shard {M} kernels over {info.world} ranks")
    b, e = channel_slice(M, info.world, info.rank)
    y_local = conv_fn(x, w_mkkc[b:e].contiguous())
    if not info.distributed:
        return y_local
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
