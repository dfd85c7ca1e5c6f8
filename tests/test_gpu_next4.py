"""GPU parity of NEXT-4: moment deposition on the assembly's DMMA machinery and
the field gather that feeds alpha (include/mm.h mm_deposit_moments, mm_gather_field), against the
oracle's or_moments / or_gather (pinned in tests/test_oracle_pins.py)."""
import numpy as np
import pytest

import oracle
import synth
from tests.helpers import to_dev

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def mm():
    import paper_2604_19286_b200 as m
    return m


def mom_err(got, ref, ref_abs):
    """max |got - ref| / R with R = sigma sum_p |Q_p^m| W_pg (the robust scale; R = 0 -> exact 0)."""
    diff = np.abs(got - ref)
    zero = ref_abs == 0
    if np.any(zero & (diff > 0)):
        return float("inf")
    return float(np.where(zero, 0.0, diff / np.where(zero, 1.0, ref_abs)).max()) if diff.size else 0.0


def _velocities(npart, seed):
    return np.random.default_rng(seed).uniform(-2.0, 2.0, (npart, 3))


def run_moments(n, order, nq, d, v, sigma=1.0, xb=0, xe=None, accumulate_into=None):
    m = mm()
    g = m.Grid(n, (1.0, 1.0, 1.0), xb, xe)
    dd = to_dev(d)
    h = m.mm_sort_by_cell(g, order, 4, dd["pos"], dd["q"], None)
    out = torch.full(m.moments_shape(g, nq), float("nan"), dtype=torch.float64, device="cuda") \
        if accumulate_into is None else accumulate_into
    ghost = None
    if m.is_slab(g):
        ghost = torch.full(m.moments_ghost_shape(g, order, nq), float("nan"), dtype=torch.float64, device="cuda")
    m.mm_deposit_moments(h, nq, m.Species(sigma=sigma), torch.from_numpy(v).cuda(), out, ghost,
                         accumulate=accumulate_into is not None)
    torch.cuda.synchronize()
    return out.cpu().numpy(), None if ghost is None else ghost.cpu().numpy()


@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("nq", [4, 10])
@pytest.mark.parametrize("n,ppc", [((8, 8, 8), 64), ((7, 9, 6), 13), ((5, 5, 5), 3)])
def test_moments_parity(order, nq, n, ppc):
    d = synth.particles(synth.Config("t", n, order, "tensor", ppc, seed=31 + nq))
    v = _velocities(len(d["q"]), 5)
    got, _ = run_moments(n, order, nq, d, v, sigma=0.75)
    ref = oracle.moments(n, order, nq, d["pos"], d["q"], v, sigma=0.75)
    ref_abs = oracle.moments(n, order, nq, d["pos"], np.abs(d["q"]), np.abs(v), sigma=0.75)
    assert mom_err(got, ref, ref_abs) <= 1e-12


@pytest.mark.parametrize("order", [1, 2])
def test_moments_lattice_bit_exact(order):
    n = (6, 5, 7)
    d = synth.particles(synth.Config("t", n, order, "tensor", 24, seed=12), lattice=True)
    v = np.random.default_rng(2).integers(-4, 5, (len(d["q"]), 3)) / 4.0   # dyadic velocities
    got, _ = run_moments(n, order, 10, d, v)
    assert (got == oracle.moments(n, order, 10, d["pos"], d["q"], v)).all()


@pytest.mark.parametrize("order", [1, 2])
def test_moments_slabs_and_accumulate(order):
    # slabs with ghost planes folded into their owners (loopback) equal the whole domain; accumulate
    n = (12, 6, 7)
    cfg = synth.Config("t", n, order, "tensor", 9, seed=4)
    plane = n[1] * n[2]
    full = np.zeros((n[0], plane, 10))
    for xb, xe in ((0, 3), (3, 7), (7, 9), (9, 12)):
        d = synth.particles(cfg, xb, xe)
        v = _velocities(len(d["q"]), xb)
        o, gh = run_moments(n, order, 10, d, v, xb=xb, xe=xe)
        full[xb:xe] += o.reshape(xe - xb, plane, 10)
        gh = gh.reshape(-1, plane, 10)
        if order == 1:
            full[xe % n[0]] += gh[0]
        else:
            full[(xb - 1) % n[0]] += gh[0]
            full[xe % n[0]] += gh[1]
            full[(xe + 1) % n[0]] += gh[2]
    allp = [synth.particles(cfg, a, b) for a, b in ((0, 3), (3, 7), (7, 9), (9, 12))]
    pos = np.concatenate([d["pos"] for d in allp])
    q = np.concatenate([d["q"] for d in allp])
    v = np.concatenate([_velocities(len(d["q"]), xb) for d, xb in zip(allp, (0, 3, 7, 9))])
    ref = oracle.moments(n, order, 10, pos, q, v)
    ref_abs = oracle.moments(n, order, 10, pos, np.abs(q), np.abs(v))
    assert mom_err(full.reshape(-1, 10), ref, ref_abs) <= 1e-12
    # accumulate: a second species on top
    d = allp[0]
    m = mm()
    base = torch.from_numpy(ref.copy()).cuda()
    d2 = synth.particles(synth.Config("t", n, order, "tensor", 5, seed=8))
    v2 = _velocities(len(d2["q"]), 77)
    got, _ = run_moments(n, order, 10, d2, v2, accumulate_into=base)
    ref2 = oracle.moments(n, order, 10, d2["pos"], d2["q"], v2, out=ref.copy(), accumulate=True)
    ref2_abs = ref_abs + oracle.moments(n, order, 10, d2["pos"], np.abs(d2["q"]), np.abs(v2))
    assert mom_err(got, ref2, ref2_abs) <= 1e-12


def test_moments_c2_full_size_sampled_planes():
    m = mm()
    cfg = synth.config("c2")
    d = synth.particles(cfg)
    v = _velocities(len(d["q"]), 9)
    got, _ = run_moments(cfg.n, 1, 10, d, v)
    got = got.reshape(cfg.n[0], -1, 10)
    cx = np.floor(d["pos"][:, 0]).astype(np.int64)
    for X in (0, 40):
        sel = (cx == X) | (cx == (X - 1) % cfg.n[0])
        ref = oracle.moments(cfg.n, 1, 10, d["pos"][sel], d["q"][sel], v[sel]).reshape(cfg.n[0], -1, 10)[X]
        ref_abs = oracle.moments(cfg.n, 1, 10, d["pos"][sel], np.abs(d["q"][sel]), np.abs(v[sel])).reshape(
            cfg.n[0], -1, 10)[X]
        assert mom_err(got[X], ref, ref_abs) <= 1e-12, X


# ---------------------------------------------------------------------------- gather
@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("xb,xe", [(0, None), (3, 8)])
def test_gather_feeds_assembly(order, xb, xe):
    """B at the nodes -> mm_gather_field -> the records' B and Fp (caller's order) equal
    oracle.gather; a following mm_assemble equals the oracle assembly with the gathered B."""
    m = mm()
    n = (10, 6, 7)
    cfg = synth.Config("t", n, order, "tensor", 11, seed=60 + order)
    d = synth.particles(cfg, xb, xe)
    nn = int(np.prod(n))
    F = np.random.default_rng(4).uniform(-1.5, 1.5, (nn, 3))
    g = m.Grid(n, (1.0, 1.0, 1.0), xb, xe)
    dd = to_dev(d)
    h = m.mm_sort_by_cell(g, order, 4, dd["pos"], dd["q"], dd["B"])
    Fp = torch.full((len(d["q"]), 3), float("nan"), dtype=torch.float64, device="cuda")
    m.mm_gather_field(h, torch.from_numpy(F).cuda(), Fp)
    torch.cuda.synchronize()
    ref = oracle.gather(n, order, d["pos"], F)
    fp = Fp.cpu().numpy()
    assert np.abs(fp - ref).max() <= 1e-14 * 8
    v = m.mm_sorted_view(h)
    perm = v["perm"].cpu().numpy()
    rec = v["rec"].cpu().numpy()
    assert (rec[perm >= 0, 4:7] == fp[perm[perm >= 0]]).all()   # the records hold the same values
    assert (rec[perm < 0, 4:7] == 0).all()
    if xe is None:
        out = torch.full(m.out_shape(g, order, 9), float("nan"), dtype=torch.float64, device="cuda")
        m.mm_assemble(h, 9, m.MM_FP64, m.Species(), out)
        torch.cuda.synchronize()
        from tests.helpers import rel_err
        assert rel_err(out.cpu().numpy(), oracle.assemble(n, order, 9, d["pos"], d["q"], fp)) <= 1e-12


def test_gather_needs_B_handle():
    m = mm()
    n = (6, 6, 6)
    d = to_dev(synth.particles(synth.Config("t", n, 1, "tensor", 3, seed=2)))
    h = m.mm_sort_by_cell(m.Grid(n), 1, 4, d["pos"], d["q"], None)
    with pytest.raises(m.MMError) as e:
        m.mm_gather_field(h, torch.zeros((216, 3), dtype=torch.float64, device="cuda"))
    assert e.value.status == m.MM_ERR_INCOMPATIBLE
