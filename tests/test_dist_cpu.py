"""CPU, world_size 2 over gloo: the multi-rank plumbing of bench.py / slab.py
(instance sharding, max-over-ranks timing, the config-5 tile all-to-all layout)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_03326_b200.slab import tile_layout
    from paper_2503_03326_b200.parallel import max_over_ranks, shard_range
    lo, hi = shard_range(64, rank, world)
    # slab exchange: the send block for peer d carries (src, dest, pair, row, col) tags
    R = 4
    per_peer, total = tile_layout(R, world)
    send = torch.zeros(total, dtype=torch.float64)
    for d in range(world):
        for p in range(4):
            for i in range(R):
                for j in range(R):
                    send[d * per_peer + (p * R + i) * R + j] = rank * 1e4 + d * 1e3 + p * 100 + i * 10 + j
    recv = torch.zeros_like(send)
    dist.all_to_all_single(recv, send)
    ok = True
    for src in range(world):
        for p in range(4):
            for i in range(R):
                for j in range(R):
                    ok &= recv[src * per_peer + (p * R + i) * R + j].item() == src * 1e4 + rank * 1e3 + p * 100 + i * 10 + j
    t = max_over_ranks(1.0 + rank, group=None)
    q.put((rank, lo, hi, ok, t))
    dist.destroy_process_group()


def test_two_rank_plumbing():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert [r[1:3] for r in res] == [(0, 32), (32, 64)]
    assert all(r[3] for r in res)
    assert all(r[4] == 2.0 for r in res)
