"""GPU: mm_assemble (accumulate=0) leaves no stale value behind, whatever the buffer held before
(the memset, or k_asm_o1t's in-kernel first-writer zeroing), on whole and slab
grids, across repeated launches on one handle (the flag epoch), with the zeroing lookahead both
larger and smaller than the number of bins; accumulate=1 still adds to what the buffer holds."""
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


def _particles(n, order, ppc, seed, x_begin=0, x_end=None):
    d = synth.particles(synth.Config("z", n, order, "tensor", ppc, seed=seed))
    if x_end is not None:
        cx = np.floor(d["pos"][:, 0]).astype(int)
        keep = (cx >= x_begin) & (cx < x_end)
        d = {k: v[keep] for k, v in d.items()}
    return d


@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("n,ppc", [((5, 6, 7), 9), ((40, 36, 32), 3)])
def test_repeated_launches_garbage_buffers(order, n, ppc):
    m = mm()
    d = _particles(n, order, ppc, seed=11 + order)
    ref = oracle.assemble(n, order, 9, d["pos"], d["q"], d["B"])
    g = m.Grid(n)
    dd = to_dev(d)
    h = m.mm_sort_by_cell(g, order, 4, dd["pos"], dd["q"], dd["B"])
    bufs = [torch.full(m.out_shape(g, order, 9), v, dtype=torch.float64, device="cuda")
            for v in (float("nan"), 1e300)]
    for it in range(5):
        out = bufs[it % 2]
        if it >= 2:
            out.fill_(float("nan") if it % 2 == 0 else -7.0)
        m.mm_assemble(h, m.MM_TENSOR, m.MM_FP64, m.Species(), out)
        torch.cuda.synchronize()
        assert rel_err(out.cpu().numpy(), ref) <= 1e-12, it
    m.mm_free(h)


@pytest.mark.parametrize("order", [1, 2])
def test_slab_garbage_ghost(order):
    m = mm()
    n, xb, xe = (12, 7, 9), 3, 8
    d = _particles(n, order, 11, seed=5, x_begin=xb, x_end=xe)
    g = m.Grid(n, (1.0, 1.0, 1.0), xb, xe)
    dd = to_dev(d)
    h = m.mm_sort_by_cell(g, order, 4, dd["pos"], dd["q"], dd["B"])
    out = torch.full(m.out_shape(g, order, 9), float("nan"), dtype=torch.float64, device="cuda")
    ghost = torch.full(m.ghost_shape(g, order, 9), float("nan"), dtype=torch.float64, device="cuda")
    for _ in range(2):
        m.mm_assemble(h, m.MM_TENSOR, m.MM_FP64, m.Species(), out, ghost)
    torch.cuda.synchronize()
    # whole-domain oracle of the slab's particles: owned rows equal it on [xb, xe); the ghost
    # planes hold the contributions to the rows outside the slab
    full = oracle.assemble(n, order, 9, d["pos"], d["q"], d["B"])
    plane = n[1] * n[2]
    own = full.reshape(n[0], plane, *full.shape[1:])
    assert rel_err(out.cpu().numpy(), own[xb:xe].reshape(-1, *full.shape[1:])) <= 1e-12
    gx = [xe] if order == 1 else [xb - 1, xe, xe + 1]
    gh = ghost.cpu().numpy().reshape(len(gx), plane, *full.shape[1:])
    for i, x in enumerate(gx):
        assert rel_err(gh[i], own[x % n[0]]) <= 1e-12


def test_accumulate_keeps_prefill():
    m = mm()
    n = (6, 6, 6)
    d = _particles(n, 1, 8, seed=9)
    ref = oracle.assemble(n, 1, 9, d["pos"], d["q"], d["B"])
    g = m.Grid(n)
    dd = to_dev(d)
    h = m.mm_sort_by_cell(g, 1, 4, dd["pos"], dd["q"], dd["B"])
    out = torch.full(m.out_shape(g, 1, 9), 0.0, dtype=torch.float64, device="cuda")
    m.mm_assemble(h, m.MM_TENSOR, m.MM_FP64, m.Species(), out)
    m.mm_assemble(h, m.MM_TENSOR, m.MM_FP64, m.Species(), out, accumulate=1)
    torch.cuda.synchronize()
    assert rel_err(out.cpu().numpy(), 2 * ref) <= 1e-12


def test_in_kernel_zeroing_subprocess():
    """The same checks with k_asm_o1t's in-kernel first-writer zeroing switched on (MM_ZERO_O1=1,
    read once per process, hence a child process); off by default (slower than the memset)."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, MM_ZERO_O1="1")
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.abspath(__file__), "-q", "-x", "-m", "gpu",
                        "-k", "not subprocess"], env=env, capture_output=True, text=True, timeout=600,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
