"""Multi-GPU sharding of the BSA hot path (SURVEY.md §8 row "multi-GPU").

The path shards by (batch, head): every (b, h) problem — its selection, forward and backward — is
independent, so ranks need NO collective on the data path. Two launch modes, one process per GPU:

* weak  ("problem"): every rank runs its own full problem (its own batch element / seed); total work
  grows with the number of GPUs.
* strong ("heads"):  the heads of ONE problem are split into contiguous slices, one per rank (the
  Wan-14B 40-head configuration over 1/2/4/8 GPUs).

The only collectives are for measurement: the step time is the max over ranks and the executed FLOPs
are summed (torch.distributed all_reduce on a tiny tensor, nccl on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

import torch


def head_range(num_heads: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [h0, h1) slice of the heads owned by `rank`; sizes differ by at most one."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(num_heads, world)
    h0 = rank * base + min(rank, extra)
    return h0, h0 + base + (1 if rank < extra else 0)


def problem_seed(seed: int, rank: int) -> int:
    """Weak scaling: rank r works on an independent problem drawn with its own seed."""
    return seed + 1000 * rank


def reduce_step_stats(time_ms: float, flops: float, device=None, group=None) -> tuple[float, float]:
    """(max over ranks of the timed region, sum over ranks of the executed FLOPs).

    With world size 1 (or no process group) this is the identity.
    """
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(time_ms), float(flops)
    t = torch.tensor([float(time_ms)], dtype=torch.float64, device=device)
    f = torch.tensor([float(flops)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(f, op=dist.ReduceOp.SUM, group=group)
    return float(t.item()), float(f.item())


def rank_time_spread(time_ms: float, device=None, group=None) -> tuple[float, float]:
    """(max, min) over ranks of a rank's timed region: max/min is the load imbalance of the head or problem
    partition (per-head sparsity differs). Identity with one rank."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(time_ms), float(time_ms)
    hi = torch.tensor([float(time_ms)], dtype=torch.float64, device=device)
    lo = hi.clone()
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    return float(hi.item()), float(lo.item())
