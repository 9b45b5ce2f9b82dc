"""Host-side fleet plumbing for the multi-GPU path.

The path partitions by service instance: rank r of G owns a contiguous block of
instances, windows never cross instances, so stats, scores, MD and flags are
local.  The one exchange is the fleet-wide threshold, done inside libenova.so
over NCCL (include/enova.h, enova_fit_threshold with a communicator).  This
module holds the host logic around it, with no method arithmetic:

* ``shard_range``        -- the contiguous instance block of a rank;
* ``broadcast_unique_id`` -- rank 0's 128-byte NCCL id to every rank over a
  torch.distributed group (gloo or nccl);
* ``max_over_ranks``     -- device-timed numbers are reported as the max over
  ranks (bench.py contract);
* ``sum_over_ranks``     -- integer totals (windows processed) across ranks.
"""
from __future__ import annotations

import torch


def shard_range(n_global: int, world: int, rank: int) -> tuple[int, int]:
    """[begin, end) of the instances rank `rank` owns: contiguous blocks, the
    first n_global % world ranks one instance larger (rank order = instance
    order, which is what makes the rank-ordered tail gather canonical)."""
    n_global, world, rank = int(n_global), int(world), int(rank)
    if world <= 0 or not (0 <= rank < world) or n_global < 0:
        raise ValueError("bad shard request")
    base, extra = divmod(n_global, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def _dist():
    import torch.distributed as dist
    return dist


def _comm_device(group=None):
    dist = _dist()
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def broadcast_unique_id(id128: bytes | None, rank: int, world: int, group=None) -> bytes:
    """Return rank 0's 128-byte id on every rank (id128 is only read on rank 0)."""
    if rank == 0:
        if id128 is None or len(id128) != 128:
            raise ValueError("rank 0 must supply the 128-byte unique id")
        t = torch.tensor(list(id128), dtype=torch.uint8)
    else:
        t = torch.zeros(128, dtype=torch.uint8)
    dist = _dist()
    if world > 1 and dist.is_initialized():
        dev = _comm_device(group)
        t = t.to(dev)
        dist.broadcast(t, 0, group=group)
        t = t.cpu()
    return bytes(t.tolist())


def max_over_ranks(x: float, group=None) -> float:
    """Max of a per-rank float over the group (identity without a process group)."""
    dist = _dist()
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_comm_device(group))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(x: int, group=None) -> int:
    """Exact integer sum over the group."""
    dist = _dist()
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return int(x)
    t = torch.tensor([int(x)], dtype=torch.int64, device=_comm_device(group))
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())
