"""Host-side multi-GPU logic on the CPU: world sizes 2 and 3 (uneven shards) over gloo.

The per-rank compute is the CPU oracle (test infrastructure standing in for the
GPU executor); what is tested is the product's sharding and exchange logic in
paper_2005_06787_b200/distributed.py: balanced contiguous ranges, the chained
ascending fold (1 KiB accumulator handed rank to rank) giving the SAME BITS as
the single-process run_scheme sum (runtime.hpp:601-605) for any world size, and
the one-all-reduce fast reduction.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2005_06787_b200.distributed import distributed_sum, shard_range

CASE = "rt_grid3x4_m8_sliced"


def test_shard_range_partitions_in_order():
    for n in (0, 1, 5, 64, 1000):
        for w in (1, 2, 3, 8):
            ranges = [shard_range(n, r, w) for r in range(w)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c and b >= a
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, deterministic, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from golden_io import plan_path
    from oracle.oracle import OraclePlan
    p = OraclePlan(plan_path(CASE, "single"))
    cache = p.build_cache()

    def compute(lo, hi, per_slice, acc):
        vals, s = p.run_slices(lo, hi, cache)
        v = torch.from_numpy(np.ascontiguousarray(vals).view(np.float64).reshape(hi - lo, -1))
        if per_slice is not None:
            per_slice.copy_(v)
        else:
            acc += torch.from_numpy(s.view(np.float64).copy())

    out = distributed_sum(p.subtasks, p.out_elements, compute, None, torch.device("cpu"),
                          deterministic)
    if rank == 0:
        q.put(out.numpy().copy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("deterministic", [True, False])
def test_gloo_sum_matches_single_process(deterministic, world):
    from golden_io import read_ref
    _, _, want, _, _ = read_ref(CASE, "single")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, deterministic, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    got = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    got = got.view(np.complex128)
    if deterministic:
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    else:
        assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
