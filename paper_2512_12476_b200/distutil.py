"""torch.distributed plumbing for the sharded search (one process per GPU).

The engine's own exchange (per-round arm records, incumbent plan) runs inside
libhpg.so over NCCL; the launcher only has to hand every rank the same
128-byte ncclUniqueId and to reduce timings. Backend-agnostic so the CPU test
suite can exercise it with gloo.
"""
import torch
import torch.distributed as dist


def _dev():
    return torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend() == "nccl" else torch.device("cpu")


def broadcast_bytes(payload, src: int = 0, size: int = 128) -> bytes:
    """rank `src` passes `payload` (len == size); every rank returns it."""
    t = torch.zeros(size, dtype=torch.uint8, device=_dev())
    if dist.get_rank() == src:
        t.copy_(torch.tensor(list(payload), dtype=torch.uint8))
    dist.broadcast(t, src)
    return bytes(t.cpu().tolist())


def max_over_ranks(x: float) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=_dev())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=_dev())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def shard_of(run_index: int, world: int) -> int:
    """owner rank of a lockstep run (mirror of search.cpp's round-robin deal)"""
    return run_index % world
