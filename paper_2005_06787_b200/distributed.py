"""Slice sharding over the GPUs of one box (one process per GPU, NCCL).

Replaces the reference's file-queue harness (queue.hpp:156-336): instead of
envelopes [lo, hi) claimed through a shared directory and summed by
`agent_collect` in ascending envelope order, every rank owns one contiguous
slice range, keeps its branch cache resident in HBM, and only the
2*out_elements fp64 accumulator (1 KiB for 64 amplitudes) crosses GPUs.

Two reductions:
  deterministic=True  every rank keeps its per-slice roots; the ascending fold
                      of run_scheme (runtime.hpp:601-605) starts on rank 0 and
                      each rank continues it with the accumulator handed over
                      by the previous rank (one 1 KiB send/recv per hop), then
                      the last rank broadcasts it: the SAME BITS as the
                      single-process run_scheme for any number of GPUs.
  deterministic=False each rank folds its own range in ascending order and one
                      NCCL all-reduce adds the partial sums; results agree to
                      rounding across GPU counts.
The in-process variant of the same scheme (one host thread per GPU, NCCL via
the C ABI) is stn_multi_* / runtime.MultiPlan.
"""
from __future__ import annotations

from typing import Callable

import numpy as np


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced range of slices owned by `rank` (ascending ranks
    own ascending ranges, so rank order is assignment order)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def distributed_sum(n_slices: int, out_elements: int,
                    compute: Callable[[int, int, object, object], None],
                    fold: Callable[[object, int, object], None] | None,
                    device, deterministic: bool = True, group=None):
    """Host-side sharding + exchange. `compute(lo, hi, per_slice, acc)` fills
    this rank's rows (per_slice: [hi-lo, 2*out] tensor) or folds them into
    acc; `fold(rows, n, acc)` continues acc's ascending fold over n rows on the
    device (the executor's stn_fold_slices_ordered; a torch loop when None).
    Returns the sum on every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_range(n_slices, rank, world)
    acc = torch.zeros(2 * out_elements, dtype=torch.float64, device=device)
    if not deterministic:
        if hi > lo:
            compute(lo, hi, None, acc)
        if world > 1:
            dist.all_reduce(acc, group=group)
        return acc
    rows = torch.zeros((max(hi - lo, 1), 2 * out_elements), dtype=torch.float64, device=device)
    if hi > lo:
        compute(lo, hi, rows[: hi - lo], None)
    ranks = dist.get_process_group_ranks(group) if (world > 1 and group is not None) else None
    glob = (lambda r: ranks[r]) if ranks else (lambda r: r)  # noqa: E731
    if rank > 0:
        dist.recv(acc, src=glob(rank - 1), group=group)
    if hi > lo:
        if fold is not None:
            fold(rows, hi - lo, acc)
        else:
            for a in range(hi - lo):
                acc += rows[a]
    if rank < world - 1:
        dist.send(acc, dst=glob(rank + 1), group=group)
    if world > 1:
        dist.broadcast(acc, src=glob(world - 1), group=group)
    return acc


def run_scheme_distributed(plan, cache, deterministic: bool = True, group=None, stream=None):
    """All slices of `plan` over every rank of the default process group; each
    rank passes its own device plan and branch cache. Returns the summed root
    tensor (numpy complex128, out_dims) on every rank."""
    import torch

    from .runtime import fold_slices_ordered, run_slices

    device = torch.device("cuda", torch.cuda.current_device())
    if stream is None:  # the stream the zero-fills and the NCCL calls are ordered on
        stream = torch.cuda.current_stream(device)

    def compute(lo, hi, per_slice, acc):
        run_slices(plan, cache, lo, hi, acc=acc, per_slice=per_slice, stream=stream)

    def fold(rows, n, acc):
        fold_slices_ordered(rows, n, plan.out_elements, acc, stream=stream)

    out = distributed_sum(plan.subtasks, plan.out_elements, compute, fold, device,
                          deterministic, group)
    return out.cpu().numpy().view(np.complex128).reshape(plan.out_dims)
