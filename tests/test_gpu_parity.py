"""GPU parity: the CUDA path through the C ABI against the oracle (run on a B200).

Bars: sort/binning bit-exact (perm, seg_begin, seg_count,
record bits); FP64 assembly within 1e-12 of the oracle normalised by the
global row-abs-sum (north_star); dyadic-lattice inputs bit-exact.
"""
import numpy as np
import pytest

import oracle
import synth
from tests.helpers import rel_err, to_dev

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-12


def mm():
    import paper_2604_19286_b200 as m
    return m


def run_gpu(n, order, kind, d, k_pad=4, species=None, x_begin=0, x_end=None, h=(1.0, 1.0, 1.0)):
    m = mm()
    g = m.Grid(n, h, x_begin, x_end)
    dd = to_dev(d)
    B = dd["B"] if kind == 9 else None
    h_ = m.mm_sort_by_cell(g, order, k_pad, dd["pos"], dd["q"], B)
    out = torch.full(m.out_shape(g, order, kind), float("nan"), dtype=torch.float64, device="cuda")
    ghost = None
    if m.is_slab(g):
        ghost = torch.full(m.ghost_shape(g, order, kind), float("nan"), dtype=torch.float64, device="cuda")
    m.mm_assemble(h_, kind, m.MM_FP64, species or m.Species(), out, ghost)
    torch.cuda.synchronize()
    return out.cpu().numpy(), (None if ghost is None else ghost.cpu().numpy()), h_


def run_oracle(n, order, kind, d, **kw):
    return oracle.assemble(n, order, kind, d["pos"], d["q"], d["B"] if kind == 9 else None, **kw)


# ------------------------------------------------------------------ sort
@pytest.mark.parametrize("order,k_pad", [(1, 4), (1, 8), (2, 4), (2, 8)])
@pytest.mark.parametrize("lattice", [False, True])
def test_sort_bit_exact(order, k_pad, lattice):
    n = (6, 5, 7)
    d = synth.particles(synth.Config("t", n, order, "tensor", 13, seed=3), lattice=lattice)
    _, _, h = run_gpu(n, order, 9, d, k_pad=k_pad)
    v = mm().mm_sorted_view(h)
    r = oracle.sort(n, order, k_pad, d["pos"], d["q"], d["B"])
    assert v["np_padded"] == r["np_padded"]
    assert (v["seg_count"].cpu().numpy() == r["seg_count"]).all()
    assert (v["seg_begin"].cpu().numpy() == r["seg_begin"]).all()
    assert (v["perm"].cpu().numpy() == r["perm"]).all()
    rec = v["rec"].cpu().numpy()
    assert (rec.view(np.uint64) == r["rec"].view(np.uint64)).all()


@pytest.mark.parametrize("order", [1, 2])
def test_sort_bit_exact_nonpow2_spacing(order):
    # xi = x/h - floor(x/h) must be bit-identical to the oracle's IEEE division for any h
    # (R5)
    n, h = (7, 9, 6), (0.3, 1.7, 0.77)
    rng = np.random.default_rng(17 + order)
    npart = 300000
    pos = rng.random((npart, 3)) * np.array(n) * np.array(h)
    # plus positions on and next to nodes
    k = rng.integers(0, 6, (20000, 3)) * np.array(h)
    pos[:20000] = np.nextafter(k, k + rng.choice([-1.0, 1.0, 0.0], size=k.shape) * 10) % (np.array(n) * h)
    pos[20000:40000] = k % (np.array(n) * h)
    L = np.array(n) * np.array(h)
    pos = np.where(pos >= L, 0.0, pos)
    d = {"pos": pos, "q": rng.uniform(-1, 1, npart), "B": rng.uniform(-1, 1, (npart, 3))}
    _, _, hd = run_gpu(n, order, 9, d, h=h)
    v = mm().mm_sorted_view(hd)
    r = oracle.sort(n, order, 4, d["pos"], d["q"], d["B"], h=h)
    assert (v["perm"].cpu().numpy() == r["perm"]).all()
    assert (v["seg_begin"].cpu().numpy() == r["seg_begin"]).all()
    assert (v["rec"].cpu().numpy().view(np.uint64) == r["rec"].view(np.uint64)).all()


def test_sort_bit_exact_c2_full():
    cfg = synth.config("c2")
    d = synth.particles(cfg)
    m = mm()
    g = m.Grid(cfg.n)
    dd = to_dev(d)
    h = m.mm_sort_by_cell(g, 1, 4, dd["pos"], dd["q"], dd["B"])
    v = m.mm_sorted_view(h)
    r = oracle.sort(cfg.n, 1, 4, d["pos"], d["q"], d["B"], records=False)
    assert (v["seg_count"].cpu().numpy() == r["seg_count"]).all()
    assert (v["seg_begin"].cpu().numpy() == r["seg_begin"]).all()
    assert (v["perm"].cpu().numpy() == r["perm"]).all()


@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("ppc", [13, 100, 300, 1500])
@pytest.mark.parametrize("input_order", ["sorted", "nearly", "reversed"])
def test_sort_bit_exact_input_order(order, ppc, input_order):
    """Cell-ordered inputs (the PIC regime): a warp's particles share bins, so the key pass
    takes one atomic per run of equal keys and the fix-up finds ascending slices.  Bins of
    ~ppc particles reach every fix-up path: warp networks (<= 64, <= 512), the shared-memory
    warp sort (<= 1024) and the CTA sort (> 1024)."""
    n = (6, 5, 7)
    cfg = synth.Config("t", n, order, "tensor", ppc, seed=50 + ppc)
    d = synth.particles(cfg, shuffle=(input_order == "nearly" and "nearly") or False)
    if input_order == "reversed":
        d = {k: np.ascontiguousarray(v[::-1]) for k, v in d.items()}
    _, _, h = run_gpu(n, order, 9, d)
    v = mm().mm_sorted_view(h)
    r = oracle.sort(n, order, 4, d["pos"], d["q"], d["B"])
    assert (v["seg_begin"].cpu().numpy() == r["seg_begin"]).all()
    assert (v["perm"].cpu().numpy() == r["perm"]).all()
    assert (v["rec"].cpu().numpy().view(np.uint64) == r["rec"].view(np.uint64)).all()


@pytest.mark.parametrize("order", [1, 2])
def test_parity_cell_ordered_input(order):
    n = (7, 6, 5)
    d = synth.particles(synth.Config("t", n, order, "tensor", 40, seed=9), shuffle="nearly")
    out, _, _ = run_gpu(n, order, 9, d)
    assert rel_err(out, run_oracle(n, order, 9, d)) <= TOL


@pytest.mark.parametrize("npart,order", [(3000, 1), (20000, 1), (20000, 2)])
def test_sort_large_bins(npart, order):
    # all particles in one cell: exercises the CTA (<= 16384) and huge (> 16384) fix-up paths
    n = (5, 5, 5)
    rng = np.random.default_rng(5)
    pos = np.array([2.0, 3.0, 1.0]) + rng.random((npart, 3)) * 0.999
    d = {"pos": pos, "q": rng.uniform(0.5, 1.5, npart), "B": rng.uniform(-1, 1, (npart, 3))}
    _, _, h = run_gpu(n, order, 9, d)
    v = mm().mm_sorted_view(h)
    r = oracle.sort(n, order, 4, d["pos"], d["q"], d["B"])
    assert (v["perm"].cpu().numpy() == r["perm"]).all()
    assert (v["seg_begin"].cpu().numpy() == r["seg_begin"]).all()


# -------------------------------------------------------------- assembly
@pytest.mark.parametrize("name,kind", [("c1", 9), ("c1", 1)])
def test_c1_parity(name, kind):
    cfg = synth.config(name)
    d = synth.particles(cfg)
    out, _, _ = run_gpu(cfg.n, cfg.order, kind, d)
    ref = run_oracle(cfg.n, cfg.order, kind, d)
    assert rel_err(out, ref) <= TOL


@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("kind", [9, 1])
@pytest.mark.parametrize("n,ppc", [((8, 8, 8), 64), ((7, 9, 6), 13), ((5, 5, 5), 3)])
def test_parity_uniform(order, kind, n, ppc):
    cfg = synth.Config("t", n, order, "tensor" if kind == 9 else "scalar", ppc, seed=77)
    d = synth.particles(cfg)
    out, _, _ = run_gpu(n, order, kind, d)
    ref = run_oracle(n, order, kind, d)
    assert rel_err(out, ref) <= TOL


@pytest.mark.parametrize("order", [1, 2])
def test_parity_clustered(order):
    cfg = synth.Config("t", (6, 24, 6), order, "scalar", 64, dist="clustered", seed=31)
    d = synth.particles(cfg)
    out, _, _ = run_gpu(cfg.n, order, 1, d)
    ref = run_oracle(cfg.n, order, 1, d)
    assert rel_err(out, ref) <= TOL


@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("kind", [9, 1])
def test_lattice_bit_exact(order, kind):
    cfg = synth.Config("t", (6, 5, 7), order, "tensor", 24, seed=12)
    d = synth.particles(cfg, lattice=True)
    out, _, _ = run_gpu(cfg.n, order, kind, d)
    ref = run_oracle(cfg.n, order, kind, d)
    assert (out == ref).all()


def test_species_constants_and_sigma():
    n = (6, 6, 6)
    cfg = synth.Config("t", n, 1, "tensor", 10, seed=2)
    d = synth.particles(cfg)
    sp = dict(qom=-2.5, dt=0.3, c=1.7, sigma=0.25)
    out, _, _ = run_gpu(n, 1, 9, d, species=mm().Species(**sp))
    ref = run_oracle(n, 1, 9, d, **sp)
    assert rel_err(out, ref) <= TOL


def test_nonunit_spacing():
    n, h = (6, 5, 7), (0.5, 2.0, 0.125)
    rng = np.random.default_rng(8)
    pos = rng.random((4000, 3)) * np.array(n) * np.array(h)
    d = {"pos": pos, "q": rng.uniform(-1, 1, 4000), "B": rng.uniform(-2, 2, (4000, 3))}
    for order in (1, 2):
        out, _, _ = run_gpu(n, order, 9, d, h=h)
        ref = oracle.assemble(n, order, 9, d["pos"], d["q"], d["B"], h=h)
        assert rel_err(out, ref) <= TOL


def test_accumulate_species_sum():
    m = mm()
    n = (6, 6, 6)
    d1 = synth.particles(synth.Config("t", n, 1, "tensor", 8, seed=1))
    d2 = synth.particles(synth.Config("t", n, 1, "tensor", 5, seed=2))
    g = m.Grid(n)
    out = torch.empty(m.out_shape(g, 1, 9), dtype=torch.float64, device="cuda")
    e1, e2 = to_dev(d1), to_dev(d2)
    h1 = m.mm_sort_by_cell(g, 1, 4, e1["pos"], e1["q"], e1["B"])
    m.mm_assemble(h1, 9, m.MM_FP64, m.Species(qom=1.0), out)
    h2 = m.mm_sort_by_cell(g, 1, 4, e2["pos"], e2["q"], e2["B"])
    m.mm_assemble(h2, 9, m.MM_FP64, m.Species(qom=-256.0), out, accumulate=True)
    ref = oracle.assemble(n, 1, 9, d1["pos"], d1["q"], d1["B"], qom=1.0)
    ref = oracle.assemble(n, 1, 9, d2["pos"], d2["q"], d2["B"], qom=-256.0, out=ref, accumulate=True)
    assert rel_err(out.cpu().numpy(), ref) <= TOL


def test_handle_reuse():
    m = mm()
    n = (6, 6, 6)
    g = m.Grid(n)
    h = None
    for seed, ppc in ((1, 9), (2, 30), (3, 4)):
        d = synth.particles(synth.Config("t", n, 2, "tensor", ppc, seed=seed))
        dd = to_dev(d)
        h = m.mm_sort_by_cell(g, 2, 4, dd["pos"], dd["q"], dd["B"], handle=h)
        out = torch.empty(m.out_shape(g, 2, 9), dtype=torch.float64, device="cuda")
        m.mm_assemble(h, 9, m.MM_FP64, m.Species(), out)
        assert rel_err(out.cpu().numpy(), run_oracle(n, 2, 9, d)) <= TOL


# ----------------------------------------------------------- edge cases
def test_empty_input():
    m = mm()
    g = m.Grid((5, 5, 5))
    e = torch.empty((0, 3), dtype=torch.float64, device="cuda")
    h = m.mm_sort_by_cell(g, 2, 4, e, torch.empty(0, dtype=torch.float64, device="cuda"), e)
    assert m.mm_sorted_view(h)["np_padded"] == 0
    out = torch.full(m.out_shape(g, 2, 9), 7.0, dtype=torch.float64, device="cuda")
    m.mm_assemble(h, 9, m.MM_FP64, m.Species(), out)
    assert (out == 0).all()


def test_special_positions():
    # xi exactly 0 and 1/2 (TSC tie, reading R4), particles on the last cell, ppc not a multiple of K
    n = (5, 6, 7)
    pts = []
    for x in (0.0, 0.5, 4.5, 4.999999999, 2.0):
        for y in (0.0, 0.5, 5.5, 3.25):
            for z in (0.0, 0.5, 6.75, 6.5):
                pts.append((x, y, z))
    pos = np.array(pts * 3)
    rng = np.random.default_rng(1)
    d = {"pos": pos, "q": rng.uniform(-1, 2, len(pos)), "B": rng.uniform(-1, 1, (len(pos), 3))}
    for order in (1, 2):
        for kind in (9, 1):
            out, _, h = run_gpu(n, order, kind, d, k_pad=8)
            assert rel_err(out, run_oracle(n, order, kind, d)) <= TOL
            v = mm().mm_sorted_view(h)
            r = oracle.sort(n, order, 8, d["pos"], d["q"], d["B"] if kind == 9 else None)
            assert (v["perm"].cpu().numpy() == r["perm"]).all()


@pytest.mark.parametrize("bad,status", [("domain_hi", 2), ("domain_lo", 2), ("nan_pos", 3), ("inf_q", 3),
                                        ("nan_B", 3)])
def test_errors(bad, status):
    m = mm()
    n = (5, 5, 5)
    d = synth.particles(synth.Config("t", n, 1, "tensor", 4, seed=1))
    d = {k: v.copy() for k, v in d.items()}
    if bad == "domain_hi":
        d["pos"][7, 1] = 5.0
    elif bad == "domain_lo":
        d["pos"][3, 2] = -1e-9
    elif bad == "nan_pos":
        d["pos"][9, 0] = np.nan
    elif bad == "inf_q":
        d["q"][2] = np.inf
    else:
        d["B"][5, 2] = np.nan
    dd = to_dev(d)
    with pytest.raises(m.MMError) as e:
        m.mm_sort_by_cell(m.Grid(n), 1, 4, dd["pos"], dd["q"], dd["B"])
    assert e.value.status == status


def test_invalid_arguments():
    m = mm()
    d = to_dev(synth.particles(synth.Config("t", (5, 5, 5), 1, "tensor", 2, seed=1)))
    with pytest.raises(m.MMError) as e:
        m.mm_sort_by_cell(m.Grid((4, 5, 5)), 2, 4, d["pos"], d["q"], d["B"])   # n < 2R+1
    assert e.value.status == m.MM_ERR_INVALID_ARG
    with pytest.raises(m.MMError):
        m.mm_sort_by_cell(m.Grid((5, 5, 5)), 1, 6, d["pos"], d["q"], d["B"])   # k_pad not multiple of 4
    h = m.mm_sort_by_cell(m.Grid((5, 5, 5)), 1, 4, d["pos"], d["q"], None)     # scalar-only handle
    out = torch.empty(m.out_shape(m.Grid((5, 5, 5)), 1, 9), dtype=torch.float64, device="cuda")
    with pytest.raises(m.MMError) as e:
        m.mm_assemble(h, 9, m.MM_FP64, m.Species(), out)
    assert e.value.status == m.MM_ERR_INCOMPATIBLE
    with pytest.raises(m.MMError) as e:
        m.mm_sort_by_cell(m.Grid((6, 5, 5)), 1, 4, d["pos"], d["q"], d["B"], handle=h)   # other grid
    assert e.value.status == m.MM_ERR_INCOMPATIBLE


# ------------------------------------------------------ slab (ghost planes)
@pytest.mark.parametrize("order", [1, 2])
def test_slab_decomposition_single_gpu(order):
    """k slabs on one GPU, ghost planes folded into their owners with mm_ghost_add:
    equals the whole-domain oracle (loopback)."""
    m = mm()
    n = (12, 6, 7)
    cfg = synth.Config("t", n, order, "tensor", 9, seed=4)
    cuts = [0, 3, 7, 9, 12]
    full = torch.zeros(m.out_shape(m.Grid(n), order, 9), dtype=torch.float64, device="cuda")
    plane = n[1] * n[2]
    ghosts = []
    for r in range(len(cuts) - 1):
        xb, xe = cuts[r], cuts[r + 1]
        d = synth.particles(cfg, xb, xe)
        out, ghost, _ = run_gpu(n, order, 9, d, x_begin=xb, x_end=xe)
        full[xb * plane:xe * plane] += torch.from_numpy(out).cuda()
        ghosts.append((xb, xe, torch.from_numpy(ghost).cuda()))
    # exchange: ghost planes are added into the owner's rows (periodic ring)
    nr = len(cuts) - 1
    for r, (xb, xe, gh) in enumerate(ghosts):
        gh = gh.reshape(-1, plane, gh.shape[1], gh.shape[2])
        nxt = ghosts[(r + 1) % nr]
        prv = ghosts[(r - 1) % nr]
        g_next = m.Grid(n, x_begin=nxt[0], x_end=nxt[1])
        g_prev = m.Grid(n, x_begin=prv[0], x_end=prv[1])
        owned_next = full[nxt[0] * plane:nxt[1] * plane]
        owned_prev = full[prv[0] * plane:prv[1] * plane]
        if order == 1:
            m.mm_ghost_add(g_next, order, 9, owned_next, gh[0].contiguous(), 0, 1)
        else:
            m.mm_ghost_add(g_prev, order, 9, owned_prev, gh[0].contiguous(), prv[1] - prv[0] - 1, 1)
            m.mm_ghost_add(g_next, order, 9, owned_next, gh[1:3].contiguous(), 0, 2)
    d_all = synth.particles(cfg)
    ref = run_oracle(n, order, 9, d_all)
    torch.cuda.synchronize()
    assert rel_err(full.cpu().numpy(), ref) <= TOL


# ------------------------------------------- full-size configs (sampled rows)
@pytest.mark.parametrize("name", ["c2", "c3"])
def test_full_size_sampled_planes(name):
    """BASELINE configs at full size in the launch configuration bench.py times; the oracle
    computes the exact rows of sampled node planes from the particles that can reach them."""
    cfg = synth.config(name)
    d = synth.particles(cfg)
    out, _, _ = run_gpu(cfg.n, cfg.order, 9, d)
    n = cfg.n
    plane = n[1] * n[2]
    S = (2 * cfg.order + 1) ** 3
    out = out.reshape(n[0], plane, S, 9)
    cx = np.floor(d["pos"][:, 0]).astype(np.int64)
    for X in (0, 17, n[0] - 1):
        lo, hi = X - cfg.order - 1, X + cfg.order      # cells whose support can reach node plane X
        sel = np.zeros(len(cx), dtype=bool)
        for c in range(lo, hi + 1):
            sel |= cx == (c % n[0])
        sub = {k: v[sel] for k, v in d.items()}
        ref = run_oracle(n, cfg.order, 9, sub).reshape(n[0], plane, S, 9)
        assert rel_err(out[X], ref[X]) <= TOL, X


# ---------------------------------------------- TF32 / 3xTF32 (tcgen05) variant
def run_gpu_tf32(n, order, kind, d, prec, species=None):
    m = mm()
    g = m.Grid(n)
    dd = to_dev(d)
    h_ = m.mm_sort_by_cell(g, order, 4, dd["pos"], dd["q"], dd["B"] if kind == 9 else None)
    out = torch.full(m.out_shape(g, order, kind), float("nan"), dtype=torch.float32, device="cuda")
    m.mm_assemble(h_, kind, prec, species or m.Species(), out)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


TOL_TF32 = 2e-3      # north_star (row-normalised)
TOL_TF32X3 = 2e-5    # split TF32 with FP32 accumulation and FP32 output


@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("kind", [9, 1])
@pytest.mark.parametrize("x3", [False, True])
def test_tf32_parity(order, kind, x3):
    m = mm()
    cfg = synth.Config("t", (8, 7, 9), order, "tensor", 40, seed=5)
    d = synth.particles(cfg)
    out = run_gpu_tf32(cfg.n, order, kind, d, m.MM_TF32X3 if x3 else m.MM_TF32)
    ref = run_oracle(cfg.n, order, kind, d)
    assert rel_err(out, ref) <= (TOL_TF32X3 if x3 else TOL_TF32)


@pytest.mark.parametrize("order,den", [(1, 4), (2, 2)])
@pytest.mark.parametrize("kind", [9, 1])
def test_tf32_lattice_bit_exact(order, den, kind):
    # xi in {k/4} (order 1) or {0, 1/2} (order 2): operands exact in TF32, sums exact in FP32
    m = mm()
    cfg = synth.Config("t", (6, 5, 7), order, "tensor", 20, seed=13)
    d = synth.particles(cfg, lattice=True, lattice_den=den)
    out = run_gpu_tf32(cfg.n, order, kind, d, m.MM_TF32)
    ref = run_oracle(cfg.n, order, kind, d)
    assert (out == ref.astype(np.float32).astype(np.float64)).all()


def test_tf32_c3_sampled_planes():
    m = mm()
    cfg = synth.config("c3")
    d = synth.particles(cfg)
    out = run_gpu_tf32(cfg.n, 2, 9, d, m.MM_TF32)
    n = cfg.n
    plane = n[1] * n[2]
    out = out.reshape(n[0], plane, 125, 9)
    cx = np.floor(d["pos"][:, 0]).astype(np.int64)
    X = 33
    sel = np.zeros(len(cx), dtype=bool)
    for c in range(X - 3, X + 3):
        sel |= cx == (c % n[0])
    sub = {k: v[sel] for k, v in d.items()}
    ref = run_oracle(n, 2, 9, sub).reshape(n[0], plane, 125, 9)
    assert rel_err(out[X], ref[X]) <= TOL_TF32


# ------------------------------------------------------------- operator apply (NEXT-3)
@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("kind", [9, 1])
def test_apply_random_matrix(order, kind):
    # y = M E for an arbitrary (random) stencil matrix: the CUDA product vs the oracle's loops
    m = mm()
    n = (7, 5, 6)
    S = (2 * order + 1) ** 3
    nn = int(np.prod(n))
    rng = np.random.default_rng(17 + order)
    M = rng.standard_normal((nn, S, kind))
    E = rng.standard_normal((nn, 3) if kind == 9 else (nn,))
    ref = oracle.apply(n, order, kind, M, E)
    g = m.Grid(n)
    Md, Ed = torch.from_numpy(M).cuda(), torch.from_numpy(E).cuda()
    y = torch.full(E.shape, float("nan"), dtype=torch.float64, device="cuda")
    m.mm_apply(g, order, kind, Md, Ed, y)
    y0 = torch.from_numpy(ref).cuda()
    m.mm_apply(g, order, kind, Md, Ed, y0, accumulate=True)
    torch.cuda.synchronize()
    scale = np.abs(M).reshape(nn, -1).sum(1).max() * np.abs(E).max()
    assert np.abs(y.cpu().numpy() - ref).max() <= 1e-14 * scale
    assert np.abs(y0.cpu().numpy() - 2 * ref).max() <= 2e-14 * scale


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_apply_pipeline_full_size(name):
    # sort -> assemble -> apply on the GPU at full size vs the oracle applied to the GPU's own
    # matrix (apply is exact up to rounding for any M), plus the partition-of-unity pin
    # M 1 = sum_p s_p W_pg checked on sampled rows against the oracle's assembly of a slab
    m = mm()
    cfg = synth.config(name)
    d = synth.particles(cfg)
    g = m.Grid(cfg.n)
    dd = to_dev(d)
    h_ = m.mm_sort_by_cell(g, cfg.order, 4, dd["pos"], dd["q"], dd["B"])
    M = torch.empty(m.out_shape(g, cfg.order, 9), dtype=torch.float64, device="cuda")
    m.mm_assemble(h_, 9, m.MM_FP64, m.Species(), M)
    nn = int(np.prod(cfg.n))
    E = torch.from_numpy(np.random.default_rng(3).standard_normal((nn, 3))).cuda()
    y = torch.empty((nn, 3), dtype=torch.float64, device="cuda")
    m.mm_apply(g, cfg.order, 9, M, E, y)
    torch.cuda.synchronize()
    Mh = M.cpu().numpy()
    ref = oracle.apply(cfg.n, cfg.order, 9, Mh, E.cpu().numpy())
    scale = np.abs(Mh).reshape(nn, -1).sum(1).max() * 5.0
    assert np.abs(y.cpu().numpy() - ref).max() <= 1e-13 * scale


def test_apply_rejects_slab():
    m = mm()
    g = m.Grid((8, 8, 8), (1.0, 1.0, 1.0), 0, 4)
    t = torch.zeros(8, dtype=torch.float64, device="cuda")
    with pytest.raises(m.MMError):
        m.mm_apply(g, 1, 9, t, t, t)


@pytest.mark.parametrize("order", [1, 2])
def test_sort_scalar_handle_records(order):
    # a handle sorted without B stores 32-B records {xi, q}: bit-identical to the oracle's
    # first four record fields; assembling a B-handle as MM_SCALAR reads the 64-B records
    n = (6, 5, 7)
    d = synth.particles(synth.Config("t", n, order, "tensor", 13, seed=9))
    m = mm()
    g = m.Grid(n)
    dd = to_dev(d)
    h = m.mm_sort_by_cell(g, order, 4, dd["pos"], dd["q"], None)
    v = m.mm_sorted_view(h)
    r = oracle.sort(n, order, 4, d["pos"], d["q"], d["B"])
    assert v["rec"].shape[1] == 4
    assert (v["perm"].cpu().numpy() == r["perm"]).all()
    assert (v["rec"].cpu().numpy().view(np.uint64) == r["rec"][:, :4].view(np.uint64)).all()
    hB = m.mm_sort_by_cell(g, order, 4, dd["pos"], dd["q"], dd["B"])
    ref = run_oracle(n, order, 1, d)
    for hh in (h, hB):
        for prec, dt, tol in ((m.MM_FP64, torch.float64, TOL), (m.MM_TF32, torch.float32, 2e-3)):
            out = torch.full(m.out_shape(g, order, 1), float("nan"), dtype=dt, device="cuda")
            m.mm_assemble(hh, 1, prec, m.Species(), out)
            torch.cuda.synchronize()
            assert rel_err(out.cpu().numpy().astype(np.float64), ref) <= tol


# ------------------------------------------------------------- mixed-precision inputs (NEXT-2)
@pytest.mark.parametrize("order", [1, 2])
def test_mixed_precision_inputs(order):
    # FP32 positions and B, FP64 charges: the sort and the FP64 assembly equal the
    # oracle run on the exactly widened arrays (sort bit-exact, entries <= 1e-12)
    m = mm()
    n = (7, 6, 5)
    d = synth.particles(synth.Config("t", n, order, "tensor", 20, seed=41))
    pos32, B32 = d["pos"].astype(np.float32), d["B"].astype(np.float32)
    pos32 = np.where(np.floor(pos32.astype(np.float64)) >= np.array(n), 0.0, pos32).astype(np.float32)
    w = {"pos": pos32.astype(np.float64), "q": d["q"], "B": B32.astype(np.float64)}
    g = m.Grid(n)
    h = m.mm_sort_by_cell(g, order, 4, torch.from_numpy(pos32).cuda(), torch.from_numpy(d["q"]).cuda(),
                          torch.from_numpy(B32).cuda())
    v = m.mm_sorted_view(h)
    r = oracle.sort(n, order, 4, w["pos"], w["q"], w["B"])
    assert (v["perm"].cpu().numpy() == r["perm"]).all()
    assert (v["rec"].cpu().numpy().view(np.uint64) == r["rec"].view(np.uint64)).all()
    out = torch.full(m.out_shape(g, order, 9), float("nan"), dtype=torch.float64, device="cuda")
    m.mm_assemble(h, 9, m.MM_FP64, m.Species(), out)
    torch.cuda.synchronize()
    assert rel_err(out.cpu().numpy(), run_oracle(n, order, 9, w)) <= TOL


@pytest.mark.parametrize("order", [1, 2])
def test_c4_full_size_sampled_planes(order):
    # config c4 at full size (128^3, clustered, 134.7 M particles drawn on the device as bench.py
    # does), scalar kind, FP64 and (order 2) TF32: sampled node planes against the oracle run on
    # the particles that can reach them
    m = mm()
    cfg = synth.config("c4o1")
    d = synth.particles_device(cfg, "cuda", with_B=False)
    n = cfg.n
    g = m.Grid(n)
    h = m.mm_sort_by_cell(g, order, 4, d["pos"], d["q"], None)
    S = (2 * order + 1) ** 3
    plane = n[1] * n[2]
    precs = [(m.MM_FP64, torch.float64, TOL)] + ([(m.MM_TF32, torch.float32, 2e-3)] if order == 2 else [])
    outs = []
    for prec, dt, tol in precs:
        out = torch.empty(m.out_shape(g, order, 1), dtype=dt, device="cuda")
        m.mm_assemble(h, 1, prec, m.Species(), out)
        outs.append((out.view(n[0], plane, S), tol))
    torch.cuda.synchronize()
    cx = torch.floor(d["pos"][:, 0]).long()
    for X in (0, 37):
        sel = torch.zeros_like(cx, dtype=torch.bool)
        for c in range(X - order - 1, X + order + 1):
            sel |= cx == (c % n[0])
        sub = {"pos": d["pos"][sel].cpu().numpy(), "q": d["q"][sel].cpu().numpy(), "B": None}
        ref = oracle.assemble(n, order, 1, sub["pos"], sub["q"]).reshape(n[0], plane, S)[X]
        for o, tol in outs:
            got = o[X].cpu().numpy().astype(np.float64)
            assert rel_err(got[:, :, None], ref[:, :, None]) <= tol, (X, tol)


# ------------------------------------------------------------- slab migration (NEXT-1)
@pytest.mark.parametrize("xb,xe", [(0, 16), (5, 9), (12, 16), (0, 3)])
def test_slab_partition(xb, xe):
    # stable 3-way partition by slab (include/mm.h): classes and order against numpy
    m = mm()
    n = (16, 6, 7)
    rng = np.random.default_rng(xb * 31 + xe)
    npart = 50000
    pos = rng.random((npart, 3)) * np.array(n)
    pos = np.where(pos >= np.array(n), 0.0, pos)
    qq = rng.uniform(-1, 1, npart)
    B = rng.uniform(-1, 1, (npart, 3))
    g = m.Grid(n, (1.0, 1.0, 1.0), xb, xe)
    po, qo, Bo, cnt = m.mm_slab_partition(g, torch.from_numpy(pos).cuda(), torch.from_numpy(qq).cuda(),
                                          torch.from_numpy(B).cuda())
    c = np.floor(pos[:, 0]).astype(int)
    u = (c - xb) % n[0]
    w = xe - xb
    cls = np.where(u < w, 0, np.where((u - w) < (n[0] - w + 1) // 2, 2, 1))
    idx = np.concatenate([np.nonzero(cls == k)[0] for k in range(3)])
    assert cnt == tuple(int((cls == k).sum()) for k in range(3))
    assert (po.cpu().numpy() == pos[idx]).all()
    assert (qo.cpu().numpy() == qq[idx]).all()
    assert (Bo.cpu().numpy() == B[idx]).all()
