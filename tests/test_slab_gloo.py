"""Multi-rank host logic of the slab decomposition on CPU (gloo, world size 2 and 3).

Each rank takes its own particles (particles owned by cell), computes its owned rows and
ghost planes (here from the oracle restricted to its particles, standing in for the
device kernel), runs the real exchange (slab.exchange_ghosts over torch.distributed) and
the result must equal the whole-domain oracle of all particles."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2604_19286_b200 import slab


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, order, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.Config("t", n, order, "tensor", 5, seed=21)
        widths = [slab.slab_bounds(n[0], world, r)[1] - slab.slab_bounds(n[0], world, r)[0] for r in range(world)]
        xb, xe = slab.slab_bounds(n[0], world, rank)
        d = synth.particles(cfg, xb, xe)
        loc = oracle.assemble(n, order, 9, d["pos"], d["q"], d["B"])          # whole-domain rows of MY particles
        plane = n[1] * n[2]
        S = (2 * order + 1) ** 3
        loc = loc.reshape(n[0], plane * S * 9)
        owned = torch.from_numpy(loc[xb:xe].copy())
        gplanes = [xe % n[0]] if order == 1 else [(xb - 1) % n[0], xe % n[0], (xe + 1) % n[0]]
        ghost = torch.from_numpy(loc[gplanes].copy())
        # rows outside owned+ghost planes must be empty (particles owned by cell)
        others = [x for x in range(n[0]) if not (xb <= x < xe) and x not in gplanes]
        assert not loc[others].any()

        def add(k, src):
            owned[k] += src

        slab.exchange_ghosts(owned, ghost, order, plane * S * 9, rank, world, widths, add=add)
        q.put((rank, xb, xe, owned.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("order", [1, 2])
def test_slab_exchange_gloo(world, order):
    n = (12, 5, 6) if world == 2 else (11, 5, 5)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, order, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = synth.Config("t", n, order, "tensor", 5, seed=21)
    d = synth.particles(cfg)
    ref = oracle.assemble(n, order, 9, d["pos"], d["q"], d["B"]).reshape(n[0], -1)
    for rank, xb, xe, owned in res:
        scale = np.abs(ref[xb:xe]).max()
        assert np.abs(owned - ref[xb:xe]).max() <= 1e-13 * scale, rank


def test_slab_bounds_cover():
    for n0 in (5, 12, 64, 257):
        for w in (1, 2, 3, 8):
            if n0 < 2 * w:
                continue
            b = [slab.slab_bounds(n0, w, r) for r in range(w)]
            assert b[0][0] == 0 and b[-1][1] == n0
            assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))


# ------------------------------------------------------------- particle migration (NEXT-1)
def partition_reference(n0, h, xb, xe):
    """Stable 3-way partition by slab (the rule of include/mm.h mm_slab_partition), in torch."""
    def part(pos, q, B):
        c = torch.floor(pos[:, 0] / h).long()
        u = (c - xb) % n0
        w = xe - xb
        cls = torch.where(u < w, 0, torch.where((u - w) < (n0 - w + 1) // 2, 2, 1))
        idx = torch.cat([torch.nonzero(cls == k).flatten() for k in range(3)])
        cnt = tuple(int((cls == k).sum()) for k in range(3))
        return pos[idx], q[idx], (B[idx] if B is not None else None), cnt
    return part


def _migrate_worker(rank, world, port, n, q, reach=1.5):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.Config("t", n, 1, "tensor", 4, seed=33)
        xb, xe = slab.slab_bounds(n[0], world, rank)
        d = synth.particles(cfg, xb, xe)
        # the mover: every particle displaced by up to `reach` cells along x (periodic)
        rng = np.random.default_rng(100 + rank)
        pos = d["pos"].copy()
        pos[:, 0] = (pos[:, 0] + rng.uniform(-reach, reach, len(pos))) % n[0]
        pos[:, 0] = np.where(pos[:, 0] >= n[0], 0.0, pos[:, 0])
        t = {k: torch.from_numpy(v) for k, v in (("pos", pos), ("q", d["q"]), ("B", d["B"]))}
        p2, q2, B2 = slab.migrate(t["pos"], t["q"], t["B"], rank, world, partition_reference(n[0], 1.0, xb, xe))
        q.put((rank, xb, xe, p2.numpy(), q2.numpy(), B2.numpy(), pos, d["q"], d["B"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,reach", [(2, 1.5), (3, 1.5), (4, 7.0), (5, 10.0)])
def test_slab_migration_gloo(world, reach):
    # reach > slab width: particles cross several slabs and are forwarded over several rounds
    n = (12, 4, 5) if world < 4 else (20, 4, 3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_migrate_worker, args=(r, world, port, n, q, reach)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    before = np.concatenate([np.column_stack([r[6], r[7], r[8]]) for r in res])
    after = np.concatenate([np.column_stack([r[3], r[4], r[5]]) for r in res])
    # particles owned by cell after the exchange, none lost or duplicated (rows as multisets)
    for rank, xb, xe, p2, q2, B2, *_ in res:
        cx = np.floor(p2[:, 0]).astype(int)
        assert ((cx >= xb) & (cx < xe)).all(), rank
    key = lambda a: a[np.lexsort(a.T[::-1])]
    assert after.shape == before.shape
    assert (key(after) == key(before)).all()
