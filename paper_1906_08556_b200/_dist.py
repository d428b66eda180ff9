"""Multi-GPU plumbing: one process per GPU, utterances sharded contiguously, one all-reduce
of the flat E-step accumulator per EM iteration (NCCL over NVLink on the box, gloo in CPU tests).

The frame-posterior path and i-vector extraction shard with no collective; only the EM
sufficient statistics have a real exchange step.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def world():
    """(rank, world_size) of the default process group, or (0, 1) outside torch.distributed."""
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard_range(n_items, rank, world_size):
    """Contiguous [lo, hi) share of ``n_items`` for ``rank`` (balanced to within one item)."""
    base, extra = divmod(n_items, world_size)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def shard(ids, rank=None, world_size=None):
    if rank is None or world_size is None:
        rank, world_size = world()
    lo, hi = shard_range(len(ids), rank, world_size)
    return list(ids[lo:hi])


def allreduce_sum_(flat: torch.Tensor):
    """In-place sum of a flat buffer over all ranks (no-op single process)."""
    _, ws = world()
    if ws > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM)
    return flat


def gather_rows(local: torch.Tensor, counts):
    """Concatenate per-rank row blocks (sizes ``counts``) on every rank (extraction output)."""
    rank, ws = world()
    if ws == 1:
        return local
    width = local.shape[1:]
    maxn = max(counts)
    buf = torch.zeros((maxn,) + tuple(width), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    parts = [torch.empty_like(buf) for _ in range(ws)]
    dist.all_gather(parts, buf)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)
