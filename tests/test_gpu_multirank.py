"""Multi-rank slab step with the real kernels: world 2 and 3, every rank on cuda:0.

One PIC-cycle step per rank, as bench.py runs it at N > 1 plus the migration of NEXT-1:
the mover displaces the rank's particles across slab boundaries, slab.migrate exchanges the
leavers (mm_slab_partition on the device), mm_sort_by_cell + mm_assemble run on the slab grid,
slab.exchange_ghosts sums the ghost planes into their owners with mm_ghost_add.  The owned
rows of all ranks together must equal the whole-domain oracle of all moved particles.

The box has one GPU and NCCL refuses two ranks on one device, so the transport is gloo over
host-staged copies; the device work is the product path.
"""
import os
import socket

import numpy as np
import pytest

import oracle
import synth
from tests.helpers import rel_err

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

N = (12, 6, 7)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _moved_particles(order, world, rank):
    """The rank's particles after the mover: owned by cell, then x displaced by up to 1.5 cells."""
    from paper_2604_19286_b200 import slab
    cfg = synth.Config("t", N, order, "tensor", 6, seed=40 + order)
    xb, xe = slab.slab_bounds(N[0], world, rank)
    d = synth.particles(cfg, xb, xe)
    rng = np.random.default_rng(1000 * world + rank)
    pos = d["pos"].copy()
    pos[:, 0] = (pos[:, 0] + rng.uniform(-1.5, 1.5, len(pos))) % N[0]
    pos[:, 0] = np.where(pos[:, 0] >= N[0], 0.0, pos[:, 0])
    return pos, d["q"], d["B"]


def _worker(rank, world, port, order, q):
    import torch.distributed as dist
    import paper_2604_19286_b200 as m
    from paper_2604_19286_b200 import slab
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        xb, xe = slab.slab_bounds(N[0], world, rank)
        widths = [slab.slab_bounds(N[0], world, r)[1] - slab.slab_bounds(N[0], world, r)[0] for r in range(world)]
        g = m.Grid(N, x_begin=xb, x_end=xe)
        pos, qq, B = (torch.from_numpy(np.ascontiguousarray(a)) for a in _moved_particles(order, world, rank))

        def partition(p, c, b):   # device partition, host-staged for the gloo transport
            po, qo, bo, cnt = m.mm_slab_partition(g, p.cuda(), c.cuda(), b.cuda())
            return po.cpu(), qo.cpu(), bo.cpu(), cnt

        pos, qq, B = slab.migrate(pos, qq, B, rank, world, partition)
        h = m.mm_sort_by_cell(g, order, 4, pos.cuda(), qq.cuda(), B.cuda())
        out = torch.full(m.out_shape(g, order, 9), float("nan"), dtype=torch.float64, device="cuda")
        ghost = torch.full(m.ghost_shape(g, order, 9), float("nan"), dtype=torch.float64, device="cuda")
        m.mm_assemble(h, 9, m.MM_FP64, m.Species(), out, ghost)
        plane_elems = N[1] * N[2] * (2 * order + 1) ** 3 * 9

        def add(k, src):
            m.mm_ghost_add(g, order, 9, out, src.cuda().contiguous(), k, 1)

        slab.exchange_ghosts(out, ghost.cpu(), order, plane_elems, rank, world, widths, add=add)
        torch.cuda.synchronize()
        q.put((rank, xb, xe, len(qq), out.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("order", [1, 2])
def test_multirank_step(world, order):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, order, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts = [_moved_particles(order, world, r) for r in range(world)]
    pos = np.concatenate([p[0] for p in parts])
    qq = np.concatenate([p[1] for p in parts])
    B = np.concatenate([p[2] for p in parts])
    assert sum(r[3] for r in res) == len(qq)     # migration neither lost nor duplicated particles
    ref = oracle.assemble(N, order, 9, pos, qq, B)
    S = (2 * order + 1) ** 3
    ref = ref.reshape(N[0], N[1] * N[2], S, 9)
    full = np.full_like(ref, np.nan)
    for rank, xb, xe, _, owned in res:
        full[xb:xe] = owned.reshape(xe - xb, N[1] * N[2], S, 9)
    assert not np.isnan(full).any()
    assert rel_err(full.reshape(-1, S, 9), ref.reshape(-1, S, 9)) <= 1e-12
