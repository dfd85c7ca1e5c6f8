"""Input generators (synth/): every input order is a permutation of the same particle set."""
import numpy as np
import pytest

import synth


@pytest.mark.parametrize("order_kind", [True, "nearly"])
def test_orders_are_permutations(order_kind):
    cfg = synth.config("c2", n=(8, 8, 8))
    base = synth.particles(cfg, shuffle=False)
    other = synth.particles(cfg, shuffle=order_kind)
    n = len(base["q"])
    assert len(other["q"]) == n == synth.num_particles(cfg)
    rows = lambda d: np.concatenate([d["pos"], d["q"][:, None], d["B"]], axis=1)
    a, b = rows(base), rows(other)
    ka, kb = np.lexsort(a.T[::-1]), np.lexsort(b.T[::-1])
    assert np.array_equal(a[ka], b[kb])
    if order_kind == "nearly":
        moved = np.any(a != b, axis=1).mean()
        assert 0.05 < moved <= 0.1
    # exactly ppc particles per cell
    cells = np.floor(other["pos"]).astype(np.int64)
    lin = (cells[:, 0] * 8 + cells[:, 1]) * 8 + cells[:, 2]
    assert np.all(np.bincount(lin, minlength=512) == cfg.ppc)
