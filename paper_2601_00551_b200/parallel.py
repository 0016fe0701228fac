"""Detector sharding and the two per-iteration exchanges.

The reference parallelises over sensor blocks of 8 inside one process and
merges block results in fixed order (radiator.py:316-348).  Here the same axis
is promoted to GPUs: rank r owns detectors [J*r/P, J*(r+1)/P); the ball cloud
is replicated; per-ball gradients and the loss are summed with
``torch.distributed.all_reduce`` (NCCL on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Shard:
    rank: int = 0
    world: int = 1

    def range(self, n_total: int) -> tuple[int, int]:
        lo = (n_total * self.rank) // self.world
        hi = (n_total * (self.rank + 1)) // self.world
        return lo, hi


def current_shard() -> Shard:
    if dist.is_available() and dist.is_initialized():
        return Shard(dist.get_rank(), dist.get_world_size())
    return Shard(0, 1)


def allreduce_sum_(t: torch.Tensor) -> torch.Tensor:
    """In-place sum over ranks (no-op without a process group)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t


def allreduce_scalar(x: float, device) -> float:
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        t = torch.tensor([x], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())
    return float(x)


def gather_rows(local: torch.Tensor, n_total: int) -> torch.Tensor:
    """Concatenate every rank's contiguous row block in rank order."""
    world = dist.get_world_size()
    rank = dist.get_rank()
    sizes = [Shard(r, world).range(n_total) for r in range(world)]
    width = local.shape[1]
    maxrows = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((maxrows, width), dtype=local.dtype, device=local.device)
    lo, hi = sizes[rank]
    pad[: hi - lo] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([parts[r][: sizes[r][1] - sizes[r][0]] for r in range(world)], dim=0)


def sharded_backward(compute_local, n_det_total: int, shard: Shard, device):
    """Host-side composition used by the engine and by the gloo tests:
    ``compute_local(lo, hi)`` returns (loss_sum_local, grads tuple of tensors
    already scaled by 2/N_total); the loss sum and every gradient tensor are
    summed over ranks.  Returns (loss_sum_global, grads)."""
    lo, hi = shard.range(n_det_total)
    loss_local, grads = compute_local(lo, hi)
    for g in grads:
        if g is not None:
            allreduce_sum_(g)
    return allreduce_scalar(loss_local, device), grads
