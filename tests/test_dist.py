"""Multi-rank host logic on CPU (gloo, world_size 2): sharding, timing max,
gather of per-rank results -- the control plane bench.py and
paper_1407_8315_b200.dist use around the per-GPU solves."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1407_8315_b200 import dist as D


def test_shard_covers_and_balances():
    for total in (0, 1, 7, 4096, 4097):
        for size in (1, 2, 3, 8):
            parts = [D.shard(total, r, size) for r in range(size)]
            assert parts[0][0] == 0 and parts[-1][1] == total
            assert all(parts[i][1] == parts[i + 1][0] for i in range(size - 1))
            lens = [hi - lo for lo, hi in parts]
            assert max(lens) - min(lens) <= 1
    with pytest.raises(ValueError):
        D.shard(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, size, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        m = D.max_over_ranks(1.5 + rank)
        lo, hi = D.shard(10, rank, size)
        parts = D.gather_to_root((lo, [{lo + i: complex(i)} for i in range(hi - lo)]))
        if rank == 0:
            q.put((m, parts))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    m, parts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert m == 2.5
    assert [lo for lo, _ in parts] == [0, 5]
    merged = [e for _, es in sorted(parts) for e in es]
    assert [list(e)[0] for e in merged] == list(range(10))
