"""GPU tests of the multi-GPU boundary inside libmm (include/mm.h: mm_comm_*, mm_ghost_exchange,
mm_assemble_slab) and of the TF32 paths on slab grids.

The box has one GPU, so the NCCL path runs as the SELF RING: a communicator of one rank is its
own slab neighbour on both sides, the whole grid is treated as a slab [0, n0) whose ghost planes
travel through ncclSend/ncclRecv to the same rank and are added into its own rows.  That is the
code path of N ranks (same routing, same overlap of the boundary-bin exchange with the interior
bins), and its result must equal the periodic whole-domain oracle.  The multi-rank routing is
covered by the gloo tests of slab.py (tests/test_slab_gloo.py), which use the same table.
"""
import numpy as np
import pytest

import oracle
import synth
from tests.helpers import rel_err, to_dev

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def mm():
    import paper_2604_19286_b200 as m
    return m


@pytest.fixture(scope="module")
def comm1():
    m = mm()
    c = m.mm_comm_create(1, 0, m.mm_comm_unique_id())
    yield c
    m.mm_comm_free(c)


@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("kind", [9, 1])
@pytest.mark.parametrize("prec", [0, 1, 2])
def test_assemble_slab_self_ring(comm1, order, kind, prec):
    m = mm()
    n = (9, 6, 7)
    cfg = synth.Config("t", n, order, "tensor", 17, seed=90 + order)
    d = synth.particles(cfg)
    g = m.Grid(n)
    dd = to_dev(d)
    h = m.mm_sort_by_cell(g, order, 4, dd["pos"], dd["q"], dd["B"] if kind == 9 else None)
    dt = torch.float64 if prec == 0 else torch.float32
    out = torch.full(m.out_shape(g, order, kind), float("nan"), dtype=dt, device="cuda")
    ghost = torch.full(m.ghost_shape(g, order, kind), float("nan"), dtype=dt, device="cuda")
    m.mm_assemble_slab(h, kind, prec, m.Species(), out, ghost, comm1)
    torch.cuda.synchronize()
    ref = oracle.assemble(n, order, kind, d["pos"], d["q"], d["B"] if kind == 9 else None)
    tol = {0: 1e-12, 1: 2e-3, 2: 2e-5}[prec]
    assert rel_err(out.cpu().numpy().astype(np.float64), ref) <= tol
    # accumulate = 1 adds a second copy (the ghost scratch is re-zeroed by the call)
    m.mm_assemble_slab(h, kind, prec, m.Species(), out, ghost, comm1, accumulate=True)
    torch.cuda.synchronize()
    assert rel_err(out.cpu().numpy().astype(np.float64), 2 * ref) <= tol


def test_assemble_slab_self_ring_c2_full(comm1):
    # c2 at full size through the overlapped path: sampled node planes against the oracle
    m = mm()
    cfg = synth.config("c2")
    d = synth.particles(cfg)
    g = m.Grid(cfg.n)
    dd = to_dev(d)
    h = m.mm_sort_by_cell(g, 1, 4, dd["pos"], dd["q"], dd["B"])
    out = torch.full(m.out_shape(g, 1, 9), float("nan"), dtype=torch.float64, device="cuda")
    ghost = torch.empty(m.ghost_shape(g, 1, 9), dtype=torch.float64, device="cuda")
    m.mm_assemble_slab(h, 9, m.MM_FP64, m.Species(), out, ghost, comm1)
    ref_out = torch.empty_like(out)
    m.mm_assemble(h, 9, m.MM_FP64, m.Species(), ref_out)
    torch.cuda.synchronize()
    o = out.view(cfg.n[0], -1, 27, 9)
    cx = np.floor(d["pos"][:, 0]).astype(np.int64)
    for X in (0, 63):  # the planes that receive the exchanged ghost plane
        sel = (cx == X) | (cx == (X - 1) % cfg.n[0])
        sub = {k: v[sel] for k, v in d.items()}
        ref = oracle.assemble(cfg.n, 1, 9, sub["pos"], sub["q"], sub["B"]).reshape(cfg.n[0], -1, 27, 9)[X]
        assert rel_err(o[X].cpu().numpy(), ref) <= 1e-12, X
    assert rel_err(out.cpu().numpy(), ref_out.cpu().numpy()) <= 1e-13


@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("prec", [0, 1])
def test_ghost_exchange_routing_self_ring(comm1, order, prec):
    # routing table of include/mm.h on the self ring: order 1: out[0] += ghost[0];
    # order 2: out[0] += ghost[1], out[1] += ghost[2], out[w-1] += ghost[0]
    m = mm()
    n = (7, 5, 6)
    g = m.Grid(n)
    dt = torch.float64 if prec == 0 else torch.float32
    S = (2 * order + 1) ** 3
    plane = n[1] * n[2] * S * 9
    gen = torch.Generator(device="cuda").manual_seed(3)
    out = torch.rand((n[0] * n[1] * n[2], S, 9), generator=gen, dtype=dt, device="cuda")
    ghost = torch.rand(m.ghost_shape(g, order, 9), generator=gen, dtype=dt, device="cuda")
    o0, g0 = out.clone().view(n[0], plane), ghost.clone().view(-1, plane)
    m.mm_ghost_exchange(comm1, g, order, 9, prec, out, ghost)
    torch.cuda.synchronize()
    exp = o0.clone()
    if order == 1:
        exp[0] += g0[0]
    else:
        exp[0] += g0[1]
        exp[1] += g0[2]
        exp[n[0] - 1] += g0[0]
    assert torch.equal(out.view(n[0], plane), exp)
    assert torch.equal(ghost.view(-1, plane), g0)   # the sent planes are not modified


def test_comm_argument_errors(comm1):
    m = mm()
    with pytest.raises(m.MMError) as e:
        m.mm_comm_create(2, 5, bytes(128))
    assert e.value.status == m.MM_ERR_INVALID_ARG
    n = (8, 6, 6)
    gs = m.Grid(n, (1.0, 1.0, 1.0), 2, 5)          # a slab grid with a one-rank communicator
    d = to_dev(synth.particles(synth.Config("t", n, 1, "tensor", 3, seed=2), 2, 5))
    h = m.mm_sort_by_cell(gs, 1, 4, d["pos"], d["q"], d["B"])
    out = torch.zeros(m.out_shape(gs, 1, 9), dtype=torch.float64, device="cuda")
    ghost = torch.zeros(m.ghost_shape(gs, 1, 9), dtype=torch.float64, device="cuda")
    with pytest.raises(m.MMError) as e:
        m.mm_assemble_slab(h, 9, m.MM_FP64, m.Species(), out, ghost, comm1)
    assert e.value.status == m.MM_ERR_INCOMPATIBLE


@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("x3,tol", [(False, 2e-3), (True, 2e-5)])
def test_tf32_slab_decomposition_single_gpu(order, x3, tol):
    """TF32 / 3xTF32 on slab grids (ghost planes in FP32): k slabs on one GPU, ghost planes
    folded into their owners, equals the whole-domain oracle."""
    m = mm()
    n = (12, 6, 7)
    cfg = synth.Config("t", n, order, "tensor", 9, seed=4)
    cuts = [0, 3, 7, 9, 12]
    plane = n[1] * n[2]
    S = (2 * order + 1) ** 3
    full = torch.zeros((n[0], plane, S, 9), dtype=torch.float32, device="cuda")
    prec = m.MM_TF32X3 if x3 else m.MM_TF32
    for r in range(len(cuts) - 1):
        xb, xe = cuts[r], cuts[r + 1]
        d = to_dev(synth.particles(cfg, xb, xe))
        g = m.Grid(n, (1.0, 1.0, 1.0), xb, xe)
        h = m.mm_sort_by_cell(g, order, 4, d["pos"], d["q"], d["B"])
        out = torch.full(m.out_shape(g, order, 9), float("nan"), dtype=torch.float32, device="cuda")
        ghost = torch.full(m.ghost_shape(g, order, 9), float("nan"), dtype=torch.float32, device="cuda")
        m.mm_assemble(h, 9, prec, m.Species(), out, ghost)
        full[xb:xe] += out.view(xe - xb, plane, S, 9)
        gh = ghost.view(-1, plane, S, 9)
        if order == 1:
            full[xe % n[0]] += gh[0]
        else:
            full[(xb - 1) % n[0]] += gh[0]
            full[xe % n[0]] += gh[1]
            full[(xe + 1) % n[0]] += gh[2]
    torch.cuda.synchronize()
    ref = oracle.assemble(n, order, 9, *[synth.particles(cfg)[k] for k in ("pos", "q", "B")])
    assert rel_err(full.view(-1, S, 9).cpu().numpy().astype(np.float64), ref) <= tol
