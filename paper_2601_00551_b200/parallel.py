"""Detector sharding and the two per-iteration exchanges.

The reference parallelises over sensor blocks of 8 inside one process and
merges block results in fixed order (radiator.py:316-348).  Here the same axis
is promoted to GPUs: rank r owns detectors [J*r/P, J*(r+1)/P); the ball cloud
is replicated; per-ball gradients, the loss, the error flags and the op
count are summed by ONE ``torch.distributed.all_reduce`` per iteration (NCCL
on GPUs, gloo in the CPU tests).
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


# Pass tail: TAIL doubles appended to the per-ball gradient buffer (written
# on the GPU by pab_pass_tail): loss sum, coincident flag, non-finite flag,
# op count.  Summed by the same all-reduce as the gradients, so one
# collective per iteration carries everything the ranks must agree on, and
# an error seen by one rank's detectors is raised by every rank.
TAIL = 4


def tail_values(loss_sum: float, coincident: bool, nonfinite: bool, ops: int) -> list:
    return [float(loss_sum), 1.0 if coincident else 0.0, 1.0 if nonfinite else 0.0, float(ops)]


def read_tail(tail) -> tuple[float, bool, bool, int]:
    """(loss sum, coincident anywhere, non-finite anywhere, op count) of a
    reduced tail (host sequence of TAIL floats)."""
    return float(tail[0]), bool(tail[1] > 0), bool(tail[2] > 0), int(tail[3])


def sharded_backward(compute_local, n_det_total: int, shard: Shard, device):
    """Host-side composition of the engine's iteration, used by the gloo
    tests: ``compute_local(lo, hi)`` returns (loss_sum_local, grads tuple of
    tensors already scaled by 2/N_total, (coincident, nonfinite, ops)); the
    gradients and the pass tail are packed into one buffer and summed over
    ranks by ONE all-reduce.  Returns (loss_sum_global, grads, (coincident,
    nonfinite, ops) over all ranks)."""
    lo, hi = shard.range(n_det_total)
    loss_local, grads, flags = compute_local(lo, hi)
    coincident, nonfinite, ops = flags
    parts = [g.reshape(-1).to(torch.float64) for g in grads if g is not None]
    tail = torch.tensor(tail_values(loss_local, coincident, nonfinite, ops), dtype=torch.float64)
    flat = torch.cat(parts + [tail]).to(device)
    allreduce_sum_(flat)
    out, k = [], 0
    for g in grads:
        if g is None:
            out.append(None)
            continue
        m = g.numel()
        out.append(flat[k:k + m].view(g.shape).to(g.dtype))
        k += m
    loss_sum, co, nf, n_ops = read_tail(flat[k:k + TAIL].cpu().tolist())
    return loss_sum, tuple(out), (co, nf, n_ops)
