"""Row-block sharded multiply over NCCL on two GPUs (SURVEY 8e, C5's path):
each rank preprocesses only its strip, multiplies, and the all-gathered,
reassembled output equals the single-GPU result (bit-exact on the integer
and fused paths).  Needs two GPUs; skipped otherwise (the host logic is
covered by the gloo world-2 test on CPU)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


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
        sm = shard.ShardedMatrix(m, n, "ternary", k, strip, rank, world, weight_scale=0.5)
        g = torch.Generator(device="cuda").manual_seed(3)
        vi = torch.randint(-128, 128, (n,), dtype=torch.int8, device="cuda", generator=g)
        vf = torch.randn(n, device="cuda", generator=g).to(torch.bfloat16)
        yi = sm.matvec(vi)
        yq = sm.matvec(vf, fused=True)
        q.put((rank, yi.cpu().numpy(), yq.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_nccl_world2_equals_single_gpu():
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    import torch.multiprocessing as mp
    import paper_2603_27462_b200 as rsr
    from paper_2603_27462_b200.devicepack import random_ternary_device
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = {r: (yi, yq) for r, yi, yq in (q.get(timeout=300) for _ in range(world))}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    torch.cuda.set_device(0)
    m, n, k = 1203, 40000, 6
    full = random_ternary_device(m, n, 9, 0.5)
    a = rsr.preprocess(rsr.PackedMatrix(m, n, "ternary", full.data, 0.5), k)
    g = torch.Generator(device="cuda").manual_seed(3)
    vi = torch.randint(-128, 128, (n,), dtype=torch.int8, device="cuda", generator=g)
    vf = torch.randn(n, device="cuda", generator=g).to(torch.bfloat16)
    ref_i = rsr.rsr_matvec(a, vi).cpu().numpy()
    ref_q = rsr.rsr_matvec_fused(a, vf).cpu().numpy()
    for r in range(world):
        assert np.array_equal(outs[r][0], ref_i)
        assert np.array_equal(outs[r][1], ref_q)
