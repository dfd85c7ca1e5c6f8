"""GPU parity of the two-phase deposit (csrc/mm_nodesum.cu): the assembly kernels store one
pair-product block per bin and a node-row kernel sums the blocks of the bins around each node
(DESIGN.md §7).  Default for the TF32 / 3xTF32 order-2 assembly; MM_TWO_PHASE selects it for the
FP64 order-2 kernels (bit 2) and TF32 order 1 (bit 1).

Checked against the oracle (whole periodic grids incl. the smallest legal n = 5 where the
unwrapped x bins 0 and n0 share a window, sparse inputs with empty bins, accumulate) and against
the RED deposit on slab grids (owned rows and ghost planes), with NaN-filled outputs so that an
element the node kernel missed fails.
"""
import os

import numpy as np
import pytest

import oracle
import synth
from tests.helpers import rel_err, to_dev

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {"fp64": 1e-12, "tf32": 2e-3, "tf32x3": 2e-5}
MODES = {  # precision, order -> MM_TWO_PHASE value that selects the two-phase deposit
    ("fp64", 2): "4", ("tf32", 2): "1", ("tf32x3", 2): "1", ("tf32", 1): "2", ("tf32x3", 1): "2"}


def mm():
    import paper_2604_19286_b200 as m
    return m


def _prec(m, name):
    return {"fp64": m.MM_FP64, "tf32": m.MM_TF32, "tf32x3": m.MM_TF32X3}[name]


def assemble(n, order, kind, d, prec, mode, x_begin=0, x_end=None, accumulate_with=None):
    m = mm()
    old = os.environ.get("MM_TWO_PHASE")
    os.environ["MM_TWO_PHASE"] = mode
    try:
        g = m.Grid(n, x_begin=x_begin, x_end=x_end)
        dd = to_dev(d)
        h = m.mm_sort_by_cell(g, order, 4, dd["pos"], dd["q"], dd["B"] if kind == 9 else None)
        dt = torch.float64 if prec == "fp64" else torch.float32
        if accumulate_with is not None:
            out = torch.from_numpy(accumulate_with).to("cuda", dt)
        else:
            out = torch.full(m.out_shape(g, order, kind), float("nan"), dtype=dt, device="cuda")
        ghost = None
        if m.is_slab(g):
            ghost = torch.full(m.ghost_shape(g, order, kind), float("nan"), dtype=dt, device="cuda")
        m.mm_assemble(h, kind, _prec(m, prec), m.Species(), out, ghost, accumulate=accumulate_with is not None)
        torch.cuda.synchronize()
        return (out.cpu().numpy().astype(np.float64),
                None if ghost is None else ghost.cpu().numpy().astype(np.float64))
    finally:
        if old is None:
            os.environ.pop("MM_TWO_PHASE", None)
        else:
            os.environ["MM_TWO_PHASE"] = old


CASES = [("fp64", 2), ("tf32", 2), ("tf32x3", 2), ("tf32", 1)]


@pytest.mark.parametrize("prec,order", CASES)
@pytest.mark.parametrize("kind", [9, 1])
@pytest.mark.parametrize("n,ppc,keep", [((5, 6, 5), 6, 1.0), ((8, 7, 9), 40, 1.0), ((9, 5, 6), 1, 0.3)])
def test_two_phase_vs_oracle(prec, order, kind, n, ppc, keep):
    """Whole periodic grids: n0 = 5 (bins 0 and n0 share a window), ragged bins, and a sparse
    input (30% of one particle per cell: most bins empty, skipped by the node kernel)."""
    cfg = synth.Config("t", n, order, "tensor", ppc, seed=21 + order)
    d = synth.particles(cfg)
    if keep < 1.0:
        sel = np.random.default_rng(3).random(len(d["q"])) < keep
        d = {k: np.ascontiguousarray(v[sel]) for k, v in d.items()}
    out, _ = assemble(n, order, kind, d, prec, MODES[(prec, order)])
    ref = oracle.assemble(n, order, kind, d["pos"], d["q"], d["B"] if kind == 9 else None)
    assert np.isfinite(out).all()
    assert rel_err(out, ref) <= TOL[prec]


@pytest.mark.parametrize("prec,order", CASES)
def test_two_phase_accumulate(prec, order):
    n = (6, 5, 7)
    cfg = synth.Config("t", n, order, "tensor", 12, seed=31)
    d = synth.particles(cfg)
    ref = oracle.assemble(n, order, 9, d["pos"], d["q"], d["B"])
    pre = np.random.default_rng(5).uniform(-1, 1, ref.shape)
    if prec != "fp64":
        pre = pre.astype(np.float32).astype(np.float64)
    out, _ = assemble(n, order, 9, d, prec, MODES[(prec, order)], accumulate_with=pre)
    assert rel_err(out - pre, ref) <= TOL[prec] * (1 if prec == "fp64" else 4)


@pytest.mark.parametrize("prec,order", CASES)
@pytest.mark.parametrize("kind", [9, 1])
@pytest.mark.parametrize("cut", [(0, 4), (3, 9), (5, 12)])
def test_two_phase_slab_vs_red(prec, order, kind, cut):
    """Slab grids through mm_assemble: owned rows and every ghost plane equal the RED deposit
    (MM_TWO_PHASE=0) to rounding."""
    n = (12, 6, 7)
    cfg = synth.Config("t", n, order, "tensor", 9, seed=4)
    d = synth.particles(cfg, cut[0], cut[1])
    o2, g2 = assemble(n, order, kind, d, prec, MODES[(prec, order)], *cut)
    o0, g0 = assemble(n, order, kind, d, prec, "0", *cut)
    assert np.isfinite(o2).all() and np.isfinite(g2).all()
    tol = 1e-13 if prec == "fp64" else 1e-5
    scale = max(np.abs(o0).max(), 1e-300)
    assert np.abs(o2 - o0).max() <= tol * scale
    assert np.abs(g2 - g0).max() <= tol * scale


@pytest.mark.parametrize("prec", ["fp64", "tf32"])
def test_two_phase_c3_sampled_planes(prec):
    """c3 at full size (the bench's launch configuration): sampled node planes against the
    oracle fed with the particles that reach them."""
    m = mm()
    cfg = synth.config("c3")
    d = synth.particles(cfg)
    out, _ = assemble(cfg.n, 2, 9, d, prec, MODES[(prec, 2)])
    n = cfg.n
    plane = n[1] * n[2]
    out = out.reshape(n[0], plane, 125, 9)
    cx = np.floor(d["pos"][:, 0]).astype(np.int64)
    for X in (0, 40):
        sel = np.zeros(len(cx), dtype=bool)
        for c in range(X - 3, X + 3):
            sel |= cx == (c % n[0])
        sub = {k: v[sel] for k, v in d.items()}
        ref = oracle.assemble(n, 2, 9, sub["pos"], sub["q"], sub["B"]).reshape(n[0], plane, 125, 9)
        assert rel_err(out[X], ref[X]) <= TOL[prec], X
    del m
