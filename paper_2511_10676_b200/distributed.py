"""Data-parallel plumbing (torch.distributed; NCCL on B200, gloo for CPU tests).

The path shards by token: rows are independent, so inference and
evaluation run on contiguous token ranges per rank with weight replicas and a
single int64 all-reduce of the packed counters (integer sums — identical to a
single GPU). Training is data parallel: each rank takes a strided slice of
every minibatch; the loss partial sums {loss, hinge, n_pairs} are all-reduced
before the batch-global normalisers are applied (N*E for BCE, the batch pair
count for the hinge — losses.py:129-130, 214-216), then gradients are summed.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) token range of `rank` (sizes differ by at most one)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def allreduce_counters(counters: torch.Tensor, group=None) -> torch.Tensor:
    """Sum int64 evaluation counters over ranks in place (one collective)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(counters, op=dist.ReduceOp.SUM, group=group)
    return counters


def dp_hooks(group=None, host_staged: bool = False):
    """(grad_allreduce, loss_allreduce) callables for trainer.train / DeviceTrainer.

    host_staged: copy through host memory around the collective (a gloo
    process group; the CPU tests and the one-GPU multi-process test)."""

    def _ar(t: torch.Tensor):
        if host_staged and t.is_cuda:
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    return _ar, _ar


def allreduce_counters_host(counters: torch.Tensor, group=None) -> torch.Tensor:
    """allreduce_counters through host memory (gloo)."""
    h = counters.cpu()
    allreduce_counters(h, group)
    counters.copy_(h)
    return counters
