"""World-size-2 gloo test of the multi-GPU host logic (sharding + global min-loc)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2204_10562_b200.distributed import global_best, min_loc, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = shard(10, rank, world)
        # makespans chosen so that the global winner is a tie on makespan broken by xi
        mk = {0: 5.0, 1: 3.0, 2: 4.0, 3: 3.0, 4: 9.0, 5: 3.0, 6: 7.0, 7: 8.0, 8: 6.0, 9: 3.5}
        xi = {0: 1, 1: 4, 2: 2, 3: 2, 4: 1, 5: 2, 6: 3, 7: 1, 8: 2, 9: 1}
        got = global_best([mk[k] for k in mine], [xi[k] for k in mine], mine)
        q.put((rank, mine, got))
    finally:
        dist.destroy_process_group()


def test_sharded_min_loc_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shards = {r: m for r, m, _ in res}
    assert sorted(shards[0] + shards[1]) == list(range(10))
    assert set(shards[0]).isdisjoint(shards[1])
    # makespan 3.0 at instances 1 (xi 4), 3 (xi 2), 5 (xi 2): smallest xi, then lowest instance
    for _, _, got in res:
        assert got == (3.0, 2, 3)


def _worker_uneven(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = shard(n, rank, world)
        mk = [float((7 * k) % 5) + (0.5 if k % 3 else 0.0) for k in range(n)]
        xi = [1 + (k * 5) % 4 for k in range(n)]
        got = global_best([mk[k] for k in mine], [xi[k] for k in mine], mine)
        q.put((rank, mine, got))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [10, 2, 0])
def test_uneven_and_empty_shards_world3(n):
    """10 items over 3 ranks (4/3/3), 2 items (one rank empty), 0 items (all
    empty): counts are gathered first and short shards padded with +inf rows."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_uneven, args=(r, 3, port, n, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shards = {r: m for r, m, _ in res}
    assert sorted(sum(shards.values(), [])) == list(range(n))
    mk = [float((7 * k) % 5) + (0.5 if k % 3 else 0.0) for k in range(n)]
    xi = [1 + (k * 5) % 4 for k in range(n)]
    want = min_loc(np.array([[mk[k], xi[k], k] for k in range(n)])) if n else None
    for _, _, got in res:
        assert got == want


def test_min_loc_single_process():
    assert min_loc(np.zeros((0, 3))) is None
    assert global_best([], [], []) is None
    assert min_loc(np.array([[2.0, 3, 0], [2.0, 1, 5], [1.5, 9, 2]])) == (1.5, 9, 2)
    assert global_best([1.0, 1.0], [2, 2], [7, 3]) == (1.0, 2, 3)
