"""GPU: incremental re-binning (mm_resort_by_cell) of moved particles is
bit-identical to the oracle's stable sort of the new positions (perm, seg_begin, seg_count and
record bits) over several steps, on whole and slab grids, with bins that empty, fill, and grow
past the warp / CTA fix-up sizes; the assembly from the re-binned handle matches the oracle;
errors and the asynchronous variant."""
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


def check_sort(h, n, order, k_pad, d, x_begin=0, x_end=None):
    m = mm()
    v = m.mm_sorted_view(h)
    kw = {} if x_end is None else {"x_begin": x_begin, "x_end": x_end}
    r = oracle.sort(n, order, k_pad, d["pos"], d["q"], d["B"], **kw)
    assert v["np_padded"] == r["np_padded"]
    assert (v["seg_count"].cpu().numpy() == r["seg_count"]).all()
    assert (v["seg_begin"].cpu().numpy() == r["seg_begin"]).all()
    assert (v["perm"].cpu().numpy() == r["perm"]).all()
    assert (v["rec"].cpu().numpy().view(np.uint64) == r["rec"].view(np.uint64)).all()


def move(d, n, rng, frac, scale, lo=None, hi=None):
    """Move a fraction of the particles by up to `scale` cells (periodic; optionally kept in
    the x-slab [lo, hi))."""
    pos = d["pos"].copy()
    np_ = len(pos)
    sel = rng.random(np_) < frac
    pos[sel] += rng.uniform(-scale, scale, (sel.sum(), 3))
    L = np.array(n, dtype=np.float64)
    pos = np.mod(pos, L)
    pos = np.where(pos >= L, 0.0, pos)
    if lo is not None:
        w = hi - lo
        pos[:, 0] = lo + np.mod(pos[:, 0] - lo, w)
        pos[:, 0] = np.where(pos[:, 0] >= hi, lo, pos[:, 0])
    return dict(d, pos=pos)


@pytest.mark.parametrize("order,k_pad", [(1, 4), (2, 4), (1, 8), (2, 8)])
def test_resort_steps_bit_exact(order, k_pad):
    m = mm()
    n = (9, 7, 8)
    rng = np.random.default_rng(order * 10 + k_pad)
    d = synth.particles(synth.Config("r", n, order, "tensor", 24, seed=5 + order))
    g = m.Grid(n)
    dd = to_dev(d)
    h = m.mm_sort_by_cell(g, order, k_pad, dd["pos"], dd["q"], dd["B"])
    for step in range(4):
        d = move(d, n, rng, 0.15 if step % 2 == 0 else 0.6, 0.7 if step < 3 else 3.5)
        dd = to_dev(d)
        m.mm_resort_by_cell(h, dd["pos"], dd["q"], dd["B"])
        check_sort(h, n, order, k_pad, d)
    out = torch.empty(m.out_shape(g, order, 9), dtype=torch.float64, device="cuda")
    m.mm_assemble(h, m.MM_TENSOR, m.MM_FP64, m.Species(), out)
    torch.cuda.synchronize()
    ref = oracle.assemble(n, order, 9, d["pos"], d["q"], d["B"])
    assert rel_err(out.cpu().numpy(), ref) <= 1e-12
    m.mm_free(h)


@pytest.mark.parametrize("order", [1, 2])
def test_resort_slab_scalar_handle(order):
    m = mm()
    n, xb, xe = (12, 6, 7), 3, 8
    rng = np.random.default_rng(7 + order)
    d = synth.particles(synth.Config("r", n, order, "tensor", 20, seed=9), x_begin=xb, x_end=xe)
    g = m.Grid(n, (1.0, 1.0, 1.0), xb, xe)
    dd = to_dev(d)
    h = m.mm_sort_by_cell(g, order, 4, dd["pos"], dd["q"], None)
    for _ in range(3):
        d = move(d, n, rng, 0.3, 1.2, xb, xe)
        dd = to_dev(d)
        m.mm_resort_by_cell(h, dd["pos"], dd["q"], None)
        v = m.mm_sorted_view(h)
        r = oracle.sort(n, order, 4, d["pos"], d["q"], d["B"], x_begin=xb, x_end=xe)
        assert (v["perm"].cpu().numpy() == r["perm"]).all()
        assert (v["seg_begin"].cpu().numpy() == r["seg_begin"]).all()
        # 32-B records {xi, q} of a handle sorted without B: the oracle's first four fields
        assert (v["rec"].cpu().numpy().view(np.uint64) == r["rec"][:, :4].view(np.uint64)).all()
    m.mm_free(h)


def test_resort_bins_grow_past_fixup_sizes():
    """Particles converge into one cell step by step: that bin passes the warp (1024) and CTA
    (16384) fix-up sizes; the others empty."""
    m = mm()
    n = (5, 5, 5)
    rng = np.random.default_rng(3)
    d = synth.particles(synth.Config("r", n, 1, "tensor", 160, seed=13))  # 20000 particles
    g = m.Grid(n)
    dd = to_dev(d)
    h = m.mm_sort_by_cell(g, 1, 4, dd["pos"], dd["q"], dd["B"])
    target = np.array([2.0, 3.0, 1.0])
    for frac in (0.04, 0.5, 0.95):
        pos = d["pos"].copy()
        sel = rng.random(len(pos)) < frac
        pos[sel] = target + rng.random((sel.sum(), 3))
        d = dict(d, pos=pos)
        dd = to_dev(d)
        m.mm_resort_by_cell(h, dd["pos"], dd["q"], dd["B"])
        check_sort(h, n, 1, 4, d)
    m.mm_free(h)


def test_resort_errors_and_async():
    m = mm()
    n = (6, 5, 7)
    rng = np.random.default_rng(1)
    d = synth.particles(synth.Config("r", n, 2, "tensor", 10, seed=2))
    g = m.Grid(n)
    dd = to_dev(d)
    h = m.mm_sort_by_cell(g, 2, 4, dd["pos"], dd["q"], dd["B"])
    # asynchronous variant, several steps, one wait
    for _ in range(3):
        d = move(d, n, rng, 0.3, 1.0)
        dd = to_dev(d)
        m.mm_resort_by_cell(h, dd["pos"], dd["q"], dd["B"], wait=False)
    m.mm_sort_wait(h)
    check_sort(h, n, 2, 4, d)
    # B presence and np must match the handle
    with pytest.raises(m.MMError) as ei:
        m.mm_resort_by_cell(h, dd["pos"], dd["q"], None)
    assert ei.value.status == m.MM_ERR_INCOMPATIBLE
    with pytest.raises(m.MMError) as ei:
        m.mm_resort_by_cell(h, dd["pos"][:-1], dd["q"][:-1], dd["B"][:-1])
    assert ei.value.status == m.MM_ERR_INCOMPATIBLE
    # a particle leaving the domain: MM_ERR_DOMAIN, the handle becomes invalid
    bad = dd["pos"].clone()
    bad[4, 2] = 7.5
    with pytest.raises(m.MMError) as ei:
        m.mm_resort_by_cell(h, bad, dd["q"], dd["B"])
    assert ei.value.status == m.MM_ERR_DOMAIN
    with pytest.raises(m.MMError) as ei:
        m.mm_resort_by_cell(h, dd["pos"], dd["q"], dd["B"])
    assert ei.value.status == m.MM_ERR_INCOMPATIBLE
    # a full sort makes it valid again
    h = m.mm_sort_by_cell(g, 2, 4, dd["pos"], dd["q"], dd["B"], handle=h)
    m.mm_resort_by_cell(h, dd["pos"], dd["q"], dd["B"])  # nobody moved
    check_sort(h, n, 2, 4, d)
    m.mm_free(h)
