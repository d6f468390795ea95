"""Multi-process (world size 2, gloo, CPU) test of the row-block sharding host
logic: block ranges, per-rank strips, padded all-gather and reassembly give
exactly the single-process result.  Local multiplies use the CPU oracle (the
GPU path of the same logic is tested in test_gpu_shard.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import rsr_oracle as orc
from paper_2603_27462_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, n, k, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = orc.random_matrix(m, n, "ternary", 11)
        ranges = shard.row_ranges(m, k, world)
        pad = max(r1 - r0 for r0, r1 in ranges)
        r0, r1 = ranges[rank]
        vi = np.random.default_rng(5).integers(-128, 128, n).astype(np.int8)
        y_local = torch.zeros(pad, dtype=torch.int32)
        if r1 > r0:
            strip = orc.Packed(r1 - r0, n, "ternary", full.data[r0:r1])
            a = orc.preprocess(strip, k)
            y_local[:r1 - r0] = torch.from_numpy(orc.matvec_i8(a, vi))
        y_all = torch.zeros(pad * world, dtype=torch.int32)
        dist.all_gather_into_tensor(y_all, y_local)
        y = y_all[torch.from_numpy(shard.gather_index(ranges, pad))].numpy()
        q.put((rank, y))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,n,k", [(37, 300, 5), (64, 1000, 6), (5, 50, 4)])
def test_sharded_int_matvec_gloo_world2(m, n, k):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = orc.random_matrix(m, n, "ternary", 11)
    ref = orc.matvec_i8(orc.preprocess(full, k),
                        np.random.default_rng(5).integers(-128, 128, n).astype(np.int8))
    for r in range(world):
        assert np.array_equal(outs[r], ref)


def test_block_ranges_balance_and_cover():
    assert shard.block_ranges(10, 3) == [(0, 3), (3, 6), (6, 10)]
    assert shard.block_ranges(2, 4) == [(0, 0), (0, 1), (1, 1), (1, 2)]
    w = np.array([1, 1, 1, 1, 10, 1, 1, 1], float)
    rg = shard.block_ranges(8, 2, w)
    assert rg[0][0] == 0 and rg[-1][1] == 8 and rg[0][1] == rg[1][0]
    assert rg == [(0, 5), (5, 8)] or rg == [(0, 4), (4, 8)]
    assert shard.row_ranges(10, 4, 2) == [(0, 4), (4, 10)]
    # byte-weighted row ranges: a heavy first block moves the cut forward
    assert shard.row_ranges(12, 4, 2, np.array([5.0, 1.0, 1.0])) == [(0, 4), (4, 12)]
    idx = shard.gather_index([(0, 4), (4, 10)], 6)
    assert list(idx) == [0, 1, 2, 3, 6, 7, 8, 9, 10, 11]


def _peer_worker(rank, world, port, m, n, k, q):
    """gather="peer" host logic: every rank's strip lands, through
    peer_row_addresses, at its global rows of every rank's full buffer (peer
    memory emulated: the stores are exchanged with all_gather_object and
    applied at the computed addresses of a flat buffer per rank)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = orc.random_matrix(m, n, "ternary", 11)
        r0, r1 = shard.row_ranges(m, k, world)[rank]
        vi = np.random.default_rng(5).integers(-128, 128, n).astype(np.int8)
        rows = np.zeros(0, np.int32)
        if r1 > r0:
            rows = orc.matvec_i8(orc.preprocess(orc.Packed(r1 - r0, n, "ternary",
                                                           full.data[r0:r1]), k), vi)
        esz, base = 4, 1 << 20  # every rank's buffer at the same fake base
        addrs = shard.peer_row_addresses([base * (j + 1) for j in range(world)], r0, esz)
        sent = [None] * world
        dist.all_gather_object(sent, (addrs, rows))
        mine = np.full(m, -7, np.int64)
        for peer_addrs, peer_rows in sent:  # the stores other ranks made into my buffer
            start = (peer_addrs[rank] - base * (rank + 1)) // esz
            mine[start:start + len(peer_rows)] = peer_rows
        q.put((rank, mine))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,n,k", [(37, 300, 5), (5, 50, 4)])
def test_peer_gather_addresses_gloo_world2(m, n, k):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, m, n, k, q))
             for r in range(world)]
    for p in procs:
        p.start()
    outs = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = orc.random_matrix(m, n, "ternary", 11)
    ref = orc.matvec_i8(orc.preprocess(full, k),
                        np.random.default_rng(5).integers(-128, 128, n).astype(np.int8))
    for r in range(world):
        assert np.array_equal(outs[r], ref)
