"""GPU: the record-first sort path (csrc/mm_sort.cu k_scatter0 / k_fixrec_*), which the library
takes from MM_SORT_RECFIRST_MIN particles on (default 48 M: c4 and the weak row), forced here on
small inputs with MM_SORT_RECFIRST_MIN=1.  Bit-exact against the oracle's stable sort (perm,
seg_begin, seg_count, record bits incl. zero pads) on every fix-up path (register networks,
shared-memory CTA sort > 512, huge-bin compaction > 16384), scalar handles (32-B records), slab
grids, FP32 inputs; the assembly from such a handle; a re-binning (mm_resort_by_cell) after it,
which first rebuilds the inverse permutation; and the c2 full-size sort against the classic path.
"""
import numpy as np
import pytest

import oracle
import synth
from tests.helpers import rel_err, to_dev

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def recfirst(monkeypatch):
    monkeypatch.setenv("MM_SORT_RECFIRST_MIN", "1")


def mm():
    import paper_2604_19286_b200 as m
    return m


def check(h, n, order, k_pad, d, with_B=True, **kw):
    v = mm().mm_sorted_view(h)
    r = oracle.sort(n, order, k_pad, d["pos"], d["q"], d["B"], **kw)
    assert v["np_padded"] == r["np_padded"]
    assert (v["seg_count"].cpu().numpy() == r["seg_count"]).all()
    assert (v["seg_begin"].cpu().numpy() == r["seg_begin"]).all()
    assert (v["perm"].cpu().numpy() == r["perm"]).all()
    rec = v["rec"].cpu().numpy()
    ref = r["rec"] if with_B else r["rec"][:, :4]
    assert (rec.view(np.uint64) == np.ascontiguousarray(ref).view(np.uint64)).all()


@pytest.mark.parametrize("order,k_pad", [(1, 4), (2, 4), (1, 8), (2, 8)])
@pytest.mark.parametrize("ppc", [13, 100, 300, 1500])
@pytest.mark.parametrize("with_B", [True, False])
def test_recfirst_bit_exact(order, k_pad, ppc, with_B):
    m = mm()
    n = (6, 5, 7)
    d = synth.particles(synth.Config("t", n, order, "tensor", ppc, seed=60 + ppc + order))
    dd = to_dev(d)
    h = m.mm_sort_by_cell(m.Grid(n), order, k_pad, dd["pos"], dd["q"], dd["B"] if with_B else None)
    check(h, n, order, k_pad, d, with_B)


@pytest.mark.parametrize("npart,order", [(3000, 1), (20000, 1), (20000, 2)])
def test_recfirst_large_bins(npart, order):
    # one cell holds everything: the CTA (<= 16384) and huge (> 16384) paths
    m = mm()
    n = (5, 5, 5)
    rng = np.random.default_rng(5)
    pos = np.array([2.0, 3.0, 1.0]) + rng.random((npart, 3)) * 0.999
    d = {"pos": pos, "q": rng.uniform(0.5, 1.5, npart), "B": rng.uniform(-1, 1, (npart, 3))}
    dd = to_dev(d)
    h = m.mm_sort_by_cell(m.Grid(n), order, 4, dd["pos"], dd["q"], dd["B"])
    check(h, n, order, 4, d)


@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("xb,xe", [(0, 4), (3, 9)])
def test_recfirst_slab(order, xb, xe):
    m = mm()
    n = (12, 6, 7)
    d = synth.particles(synth.Config("t", n, order, "tensor", 9, seed=4), xb, xe)
    dd = to_dev(d)
    h = m.mm_sort_by_cell(m.Grid(n, x_begin=xb, x_end=xe), order, 4, dd["pos"], dd["q"], dd["B"])
    check(h, n, order, 4, d, x_begin=xb, x_end=xe)


@pytest.mark.parametrize("order", [1, 2])
def test_recfirst_fp32_inputs_and_assembly(order):
    m = mm()
    n = (7, 6, 5)
    d = synth.particles(synth.Config("t", n, order, "tensor", 20, seed=41))
    pos32, B32 = d["pos"].astype(np.float32), d["B"].astype(np.float32)
    pos32 = np.where(np.floor(pos32.astype(np.float64)) >= np.array(n), 0.0, pos32).astype(np.float32)
    w = {"pos": pos32.astype(np.float64), "q": d["q"], "B": B32.astype(np.float64)}
    g = m.Grid(n)
    h = m.mm_sort_by_cell(g, order, 4, torch.from_numpy(pos32).cuda(), torch.from_numpy(d["q"]).cuda(),
                          torch.from_numpy(B32).cuda())
    check(h, n, order, 4, w)
    out = torch.full(m.out_shape(g, order, 9), float("nan"), dtype=torch.float64, device="cuda")
    m.mm_assemble(h, 9, m.MM_FP64, m.Species(), out)
    torch.cuda.synchronize()
    ref = oracle.assemble(n, order, 9, w["pos"], w["q"], w["B"])
    assert rel_err(out.cpu().numpy(), ref) <= 1e-12


@pytest.mark.parametrize("order", [1, 2])
def test_recfirst_then_resort(order):
    # the record-first sort leaves no inverse permutation; the re-binning rebuilds it
    m = mm()
    n = (9, 7, 8)
    rng = np.random.default_rng(order)
    d = synth.particles(synth.Config("r", n, order, "tensor", 24, seed=5 + order))
    g = m.Grid(n)
    dd = to_dev(d)
    h = m.mm_sort_by_cell(g, order, 4, dd["pos"], dd["q"], dd["B"])
    check(h, n, order, 4, d)
    for _ in range(2):
        pos = d["pos"].copy()
        sel = rng.random(len(pos)) < 0.1
        pos[sel] += rng.uniform(-1.5, 1.5, (sel.sum(), 3))
        L = np.array(n, dtype=np.float64)
        pos = np.mod(pos, L)
        pos = np.where(pos >= L, 0.0, pos)
        d = dict(d, pos=pos)
        dd = to_dev(d)
        m.mm_resort_by_cell(h, dd["pos"], dd["q"], dd["B"])
        check(h, n, order, 4, d)


def test_recfirst_c2_full_equals_classic(monkeypatch):
    m = mm()
    cfg = synth.config("c2")
    d = synth.particles(cfg)
    dd = to_dev(d)
    g = m.Grid(cfg.n)
    h1 = m.mm_sort_by_cell(g, 1, 4, dd["pos"], dd["q"], dd["B"])
    v1 = {k: x.cpu().numpy() for k, x in m.mm_sorted_view(h1).items() if hasattr(x, "cpu")}
    m.mm_free(h1)
    monkeypatch.setenv("MM_SORT_RECFIRST_MIN", str(10 ** 12))
    h0 = m.mm_sort_by_cell(g, 1, 4, dd["pos"], dd["q"], dd["B"])
    v0 = {k: x.cpu().numpy() for k, x in m.mm_sorted_view(h0).items() if hasattr(x, "cpu")}
    for k in ("seg_count", "seg_begin", "perm"):
        assert (v1[k] == v0[k]).all(), k
    assert (v1["rec"].view(np.uint64) == v0["rec"].view(np.uint64)).all()


@pytest.mark.parametrize("bad,status", [("domain_hi", 2), ("domain_lo", 2), ("nan_pos", 3), ("inf_q", 3),
                                        ("nan_B", 3)])
def test_recfirst_errors(bad, status):
    # the status words are raised by k_key (domain, positions) and k_scatter0 (q, B) as on the
    # classic path; the asynchronous variant reports them at mm_sort_wait
    m = mm()
    n = (5, 5, 5)
    d = {k: v.copy() for k, v in synth.particles(synth.Config("t", n, 1, "tensor", 4, seed=1)).items()}
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
    h = m.mm_sort_by_cell(m.Grid(n), 1, 4, dd["pos"], dd["q"], dd["B"], wait=False)
    with pytest.raises(m.MMError) as e:
        m.mm_sort_wait(h)
    assert e.value.status == status
