"""Host logic of the N>1 path with two gloo processes on CPU: head slices partition the
heads, weak-scaling seeds differ per rank, and the timing reduction is max-over-ranks / sum-of-FLOPs."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_01085_b200.shard import head_range, problem_seed, rank_time_spread, reduce_step_stats


def test_head_range_partitions():
    for H in (1, 2, 12, 40, 41):
        for world in (1, 2, 3, 4, 8):
            if world > H:
                continue
            spans = [head_range(H, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == H
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        head_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        t, f = reduce_step_stats(10.0 + rank, 100.0 * (rank + 1))
        h = head_range(40, world, rank)
        out[rank] = (t, f, h, problem_seed(7, rank), rank_time_spread(10.0 + 3 * rank))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0][0] == res[1][0] == 11.0  # max over ranks
    assert res[0][1] == res[1][1] == 300.0  # FLOPs summed
    assert res[0][2] == (0, 20) and res[1][2] == (20, 40)
    assert res[0][3] != res[1][3]
    assert res[0][4] == res[1][4] == (13.0, 10.0)  # (max, min) over ranks


def test_single_process_identity():
    assert reduce_step_stats(3.5, 42.0) == (3.5, 42.0)
