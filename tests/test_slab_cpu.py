"""Multi-GPU host logic on CPU (gloo, world_size 2 and 3): z-slab partition, slab layout, ghost-layer
exchange and the owned-row reductions of paper_2410_09497_b200.slab. The CUDA slab
operator itself is covered by tests/test_gpu_parity.py::test_slab_vmult_matches_global."""
import os
import socket

import numpy as np
import pytest

import paper_2410_09497_b200 as smg
from paper_2410_09497_b200 import slab

torch = pytest.importorskip("torch")


def test_partition_properties():
    for level in (1, 2, 3, 5, 6):
        m = 2 << level
        for world in (1, 2, 3, 4, 8):
            if m < world:
                continue
            b = slab.partition(level, world)
            assert b[0][0] == 0 and b[-1][1] == m
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            assert all(z1 > z0 for z0, z1 in b)
    assert slab.partition(5, 8) == [(8 * r, 8 * r + 8) for r in range(8)]


@pytest.mark.parametrize("k,level,z0,z1", [(1, 2, 0, 4), (2, 3, 4, 8), (3, 3, 8, 16), (2, 1, 0, 4)])
def test_slab_layout_matches_library(k, level, z0, z1):
    L = slab.SlabLayout(k, level, z0, z1)
    assert slab.slab_sizes(k, level, z0, z1) == L.size + [L.total]
    if (z0, z1) == (0, 2 << level):  # whole level == the stored global layout
        assert L.size + [L.total] == smg.level_sizes(k, level)


def test_extract_insert_roundtrip():
    k, level = 2, 3
    g = np.random.default_rng(0).uniform(size=smg.level_sizes(k, level)[4])
    out = np.zeros_like(g)
    for z0, z1 in slab.partition(level, 3):
        L = slab.SlabLayout(k, level, z0, z1)
        L.insert_owned(out, L.extract(g))
    assert np.array_equal(out, g)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, k, level, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        z0, z1 = slab.partition(level, world)[rank]
        L = slab.SlabLayout(k, level, z0, z1)
        g = torch.from_numpy(np.random.default_rng(42).uniform(-1, 1, smg.level_sizes(k, level)[4]))
        want = L.extract(g)
        v = torch.zeros_like(want)
        for c in range(4):  # only the owned rows are known before the exchange
            a, b = L.owned_planes(c)
            L.block(v, c)[a:b] = L.block(want, c)[a:b]
        slab.HaloExchange(L, rank, world).exchange(v)
        if L.zhi < L.m:  # u_z's extra top plane (the next slab's face) is never read: not exchanged
            L.block(v, 2)[-1] = L.block(want, 2)[-1]
        ok_ghost = bool(torch.equal(v, want))
        # owned-row dot, all-reduced == global dot
        part = 0.0
        for c in range(4):
            a, b = L.owned_planes(c)
            part += float((L.block(v, c)[a:b] ** 2).sum())
        t = torch.tensor([part], dtype=torch.float64)
        dist.all_reduce(t)
        ok_dot = abs(float(t) - float((g * g).sum())) <= 1e-9 * float((g * g).sum())
        q.put((rank, ok_ghost, ok_dot))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,k,level", [(2, 2, 2), (3, 1, 3), (2, 3, 1)])
def test_halo_exchange_gloo(world, k, level):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, k, level, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_ghost, ok_dot in res:
        assert ok_ghost, f"rank {rank}: ghost layers differ from the global vector"
        assert ok_dot, f"rank {rank}: owned-row dot does not add up"


class _CtxStub:
    degree = 2
    device = 0


def _mg_worker(rank, world, port, k, level, q):
    import torch.distributed as dist
    from paper_2410_09497_b200 import slab_mg
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx = _CtxStub()
        ctx.degree = k
        mg = slab_mg.SlabMG(ctx, level, slab.partition(level, world), [rank], world=world)
        ok = True
        for lvl in range(mg.la + 1, level + 1):
            S = mg.slabs[rank][lvl]
            g = torch.from_numpy(np.random.default_rng(lvl).uniform(-1, 1, smg.level_sizes(k, lvl)[4]))
            want = S.extract(g)
            v = torch.zeros_like(want)
            for c in range(4):
                a, b = S.owned_planes(c)
                S.block(v, c)[a:b] = S.block(want, c)[a:b]
            mg.exchange(lvl, {rank: v})
            if S.zhi < S.m:  # the held range's top u_z plane is never read: not exchanged
                S.block(v, 2)[-1] = S.block(want, 2)[-1]
            ok = ok and bool(torch.equal(v, want))
        q.put((rank, ok, mg.la))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,k,level", [(2, 2, 4), (4, 1, 4), (3, 2, 4)])
def test_slab_multigrid_exchange_gloo(world, k, level):
    # 3 ghost cell layers per interior side at every partitioned level
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mg_worker, args=(r, world, port, k, level, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, la in res:
        assert ok, f"rank {rank}: ghost layers differ"
        assert la < level
