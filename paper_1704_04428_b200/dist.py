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
