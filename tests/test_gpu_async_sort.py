"""GPU: mm_sort_by_cell_async (no host round trip) produces the same binning as the oracle
(bit-exact) and the same assembly; its domain / finiteness errors are reported by mm_sort_wait,
sticky over several sorts, and cleared by it."""
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


@pytest.mark.parametrize("order", [1, 2])
def test_async_sort_equals_oracle(order):
    m = mm()
    n = (7, 6, 9)
    d = synth.particles(synth.Config("a", n, order, "tensor", 21, seed=31 + order))
    dd = to_dev(d)
    g = m.Grid(n)
    h = None
    for _ in range(3):  # reused handle, several sorts in flight without a wait
        h = m.mm_sort_by_cell(g, order, 4, dd["pos"], dd["q"], dd["B"], handle=h, wait=False)
        out = torch.empty(m.out_shape(g, order, 9), dtype=torch.float64, device="cuda")
        m.mm_assemble(h, m.MM_TENSOR, m.MM_FP64, m.Species(), out)
    m.mm_sort_wait(h)
    r = oracle.sort(n, order, 4, d["pos"], d["q"], d["B"])
    v = m.mm_sorted_view(h)
    assert v["np_padded"] == r["np_padded"]
    assert (v["perm"].cpu().numpy() == r["perm"]).all()
    assert (v["seg_begin"].cpu().numpy() == r["seg_begin"]).all()
    ref = oracle.assemble(n, order, 9, d["pos"], d["q"], d["B"])
    assert rel_err(out.cpu().numpy(), ref) <= 1e-12
    m.mm_free(h)


def test_async_sort_deferred_errors():
    m = mm()
    n = (5, 5, 5)
    d = synth.particles(synth.Config("a", n, 1, "tensor", 8, seed=3))
    g = m.Grid(n)
    good = to_dev(d)
    bad = to_dev(d)
    bad["pos"][7, 1] = 5.5  # outside [0, n1 h)
    nan = to_dev(d)
    nan["q"][3] = float("nan")
    h = m.mm_sort_by_cell(g, 1, 4, good["pos"], good["q"], good["B"], wait=False)
    m.mm_sort_wait(h)  # OK
    # an invalid sort followed by a valid one: the error is sticky until mm_sort_wait
    h = m.mm_sort_by_cell(g, 1, 4, bad["pos"], bad["q"], bad["B"], handle=h, wait=False)
    h = m.mm_sort_by_cell(g, 1, 4, good["pos"], good["q"], good["B"], handle=h, wait=False)
    with pytest.raises(m.MMError) as ei:
        m.mm_sort_wait(h)
    assert ei.value.status == m.MM_ERR_DOMAIN
    # cleared: a valid sort now reports OK
    h = m.mm_sort_by_cell(g, 1, 4, good["pos"], good["q"], good["B"], handle=h, wait=False)
    m.mm_sort_wait(h)
    h = m.mm_sort_by_cell(g, 1, 4, nan["pos"], nan["q"], nan["B"], handle=h, wait=False)
    with pytest.raises(m.MMError) as ei:
        m.mm_sort_wait(h)
    assert ei.value.status == m.MM_ERR_NONFINITE
    # the synchronous sort reports its own error and leaves nothing sticky behind
    with pytest.raises(m.MMError):
        m.mm_sort_by_cell(g, 1, 4, bad["pos"], bad["q"], bad["B"], handle=h)
    h = m.mm_sort_by_cell(g, 1, 4, good["pos"], good["q"], good["B"], handle=h, wait=False)
    m.mm_sort_wait(h)
    m.mm_free(h)
