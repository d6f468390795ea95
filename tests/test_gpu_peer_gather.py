"""The sharded path's all-gather fused into the multiply (rsr_matvec_peers,
ShardedMatrix(gather="peer")): each output row is stored by the multiply's
epilogue into every rank's full output buffer over peer memory.

* emulated peers on one GPU: the launch fans out to several local buffers at
  a strip's global row offset (single-tile epilogue and multi-tile finalize
  both), every copy equal to the plain multiply, rows outside the strip
  untouched;
* torch symmetric memory end to end: ShardedMatrix(gather="peer") on
  min(2, #GPUs) ranks equals the single-GPU result bit for bit (integer
  path) and the NCCL gather's float result (one rank on a one-GPU box: the
  rendezvous, the one-peer store and the barrier).
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rsr():
    import torch
    import paper_2603_27462_b200 as pkg
    torch.cuda.set_device(0)
    return pkg


@pytest.mark.parametrize("tile_width", [None, 512])
def test_peer_stores_emulated(rsr, tile_width):
    import torch
    from paper_2603_27462_b200 import kernels as kn
    from paper_2603_27462_b200 import shard
    from paper_2603_27462_b200.devicepack import random_ternary_device
    m, n, k = 1000, 1500, 5
    r0, r1 = 300, 705  # a strip starting on a block boundary
    strip = random_ternary_device(r1 - r0, n, 4, 0.5, row0=r0)
    a = rsr.preprocess(rsr.PackedMatrix(r1 - r0, n, "ternary", strip.data), k, tile_width)
    g = torch.Generator(device="cuda").manual_seed(1)
    for vt, odt in ((torch.randint(-128, 128, (n,), dtype=torch.int8, device="cuda",
                                   generator=g), torch.int32),
                    (torch.randn(n, device="cuda", generator=g).to(torch.bfloat16), torch.float32)):
        ref = torch.empty(r1 - r0, dtype=odt, device="cuda")
        kn.matvec_into(a, vt, ref)
        ys = [torch.full((m,), -7, dtype=odt, device="cuda") for _ in range(3)]
        rows = torch.tensor(shard.peer_row_addresses([y.data_ptr() for y in ys], r0,
                                                     ys[0].element_size()),
                            dtype=torch.int64, device="cuda")
        kn.matvec_peers_into(a, vt, rows, len(ys))
        torch.cuda.synchronize()
        for y in ys:
            assert torch.equal(y[r0:r1], ref)
            assert bool((y[:r0] == -7).all()) and bool((y[r1:] == -7).all())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        from paper_2603_27462_b200 import shard
        from paper_2603_27462_b200.devicepack import random_ternary_device
        m, n, k = 1203, 40000, 6
        strip = lambda r0, r1: random_ternary_device(r1 - r0, n, 9, 0.5, row0=r0)
        sp = shard.ShardedMatrix(m, n, "ternary", k, strip, rank, world, gather="peer",
                                 tile_width=16384)
        sn = shard.ShardedMatrix(m, n, "ternary", k, strip, rank, world, tile_width=16384)
        g = torch.Generator(device="cuda").manual_seed(3)
        vi = torch.randint(-128, 128, (n,), dtype=torch.int8, device="cuda", generator=g)
        vf = torch.randn(n, device="cuda", generator=g).to(torch.bfloat16)
        outs = []
        for _ in range(3):  # both alternating buffers, then the first again
            yi = sp.matvec(vi).cpu().numpy()
            yf = sp.matvec(vf).cpu().numpy()
            outs.append((yi, yf))
        yf_nccl = sn.matvec(vf).cpu().numpy()
        q.put((rank, outs, yf_nccl))
    finally:
        dist.destroy_process_group()


def test_symmetric_memory_gather_equals_single_gpu(rsr):
    import torch
    import torch.multiprocessing as mp
    from paper_2603_27462_b200.devicepack import random_ternary_device
    world = min(2, torch.cuda.device_count())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {r: (outs, yfn) for r, outs, yfn in (q.get(timeout=300) for _ in range(world))}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m, n, k = 1203, 40000, 6
    full = random_ternary_device(m, n, 9, 0.5)
    a = rsr.preprocess(rsr.PackedMatrix(m, n, "ternary", full.data), k, 16384)
    g = torch.Generator(device="cuda").manual_seed(3)
    vi = torch.randint(-128, 128, (n,), dtype=torch.int8, device="cuda", generator=g)
    ref_i = rsr.rsr_matvec(a, vi).cpu().numpy()
    for r in range(world):
        outs, yf_nccl = res[r]
        for yi, yf in outs:
            assert np.array_equal(yi, ref_i)
            assert np.array_equal(yf, yf_nccl)
