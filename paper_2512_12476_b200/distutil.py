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


def sweep_range(total: int, rank: int, world: int):
    """contiguous plan-index shard [k0, k0 + n) of a sweep over `total` plans
    (independent units, no data-path collective)"""
    k0 = total * rank // world
    return k0, total * (rank + 1) // world - k0


def merge_argmin(best_cost: float, best_k: int, n_feasible: int):
    """global (min cost, lowest k) over the ranks' shard results: one all-gather
    of the float64 cost and one of the int64 (k, n_feasible) pair per rank, so
    plan indices keep all 64 bits (an empty shard reports inf and k = 2^64-1)."""
    world = dist.get_world_size()
    c = torch.tensor([best_cost], dtype=torch.float64, device=_dev())
    k_signed = best_k - (1 << 64) if best_k >= (1 << 63) else best_k
    i = torch.tensor([k_signed, n_feasible], dtype=torch.int64, device=_dev())
    cs = [torch.empty_like(c) for _ in range(world)]
    ks = [torch.empty_like(i) for _ in range(world)]
    dist.all_gather(cs, c)
    dist.all_gather(ks, i)
    rows = []
    for cc, kk in zip(cs, ks):
        k, nf = (int(x) for x in kk.cpu().tolist())
        rows.append((float(cc.cpu().item()), k + (1 << 64) if k < 0 else k, nf))
    best = min(rows, key=lambda r: (r[0], r[1]))
    return best[0], best[1], sum(r[2] for r in rows)
