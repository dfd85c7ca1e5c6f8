"""Pins of the oracle against what the paper and the mathematics fix (CPU only).

Each test names the passage it pins.  None of them re-types the oracle's
formula: the pins are worked examples (SPEC.md / hand-derived fractions in
tests/golden/), closed forms, identities, a dense W S W^T brute force built
from the explicit periodic B-spline definition, and invariants the paper
states (partition of unity, spatial symmetry, exactness of the sum).
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "single_particle.json")))


def slot(d, R):
    L = 2 * R + 1
    return ((d[0] + R) * L + (d[1] + R)) * L + (d[2] + R)


def lin(g, n):
    return (g[0] * n[1] + g[1]) * n[2] + g[2]


# ----------------------------------------------------------------- locate (R5)
@pytest.mark.parametrize("x,h,cell,xi", [
    (2.25, 1.0, 2, 0.25),
    (3.0, 1.0, 3, 0.0),        # SPEC.md:47 (a node maps to the upper cell)
    (1.75, 0.5, 3, 0.5),
])
def test_locate_spec_examples(x, h, cell, xi):
    c, f = oracle.locate([x, 0.0, 0.0], n=(8, 8, 8), h=(h, 1.0, 1.0))
    assert c[0] == cell and f[0] == xi


def test_locate_domain_errors():
    with pytest.raises(oracle.OracleError) as e:
        oracle.locate([8.0, 0.0, 0.0], n=(8, 8, 8))
    assert e.value.code == oracle.OR_ERR_DOMAIN
    with pytest.raises(oracle.OracleError) as e:
        oracle.locate([-1e-300, 0.0, 0.0], n=(8, 8, 8))
    assert e.value.code == oracle.OR_ERR_DOMAIN
    with pytest.raises(oracle.OracleError) as e:
        oracle.locate([float("nan"), 0.0, 0.0], n=(8, 8, 8))
    assert e.value.code == oracle.OR_ERR_NONFINITE
    # slab ownership: cell 2 is outside [3, 6)
    with pytest.raises(oracle.OracleError):
        oracle.locate([2.5, 0.0, 0.0], n=(8, 8, 8), x_begin=3, x_end=6)


# ----------------------------------------------------------- shape functions
def test_phi_values():
    # SPEC.md:111-113; order-2 values follow from the quadratic B-spline (R3)
    assert oracle.phi(1, 0.0) == 1.0
    assert oracle.phi(2, 0.0) == 0.75
    assert oracle.phi(2, 1.0) == 0.125
    assert oracle.phi(2, 1.5) == 0.0 and oracle.phi(1, 1.0) == 0.0


@pytest.mark.parametrize("order,xi,base,w", [
    (1, 0.25, 0, [0.75, 0.25]),
    (2, 0.0, -1, [0.125, 0.75, 0.125]),
    (2, 0.25, -1, [1 / 32, 11 / 16, 9 / 32]),   # hand-derived (golden order2 x-axis)
    (2, 0.5, 0, [0.5, 0.5, 0.0]),               # tie -> ">=" branch, PAPER.md:168 (R4)
    (2, 0.3, -1, None),
    (2, 0.7, 0, None),
])
def test_support_and_weights(order, xi, base, w):
    b, ww = oracle.support_1d(order, xi)
    assert b == base
    if w is not None:
        assert list(ww) == w


def test_partition_of_unity_and_nonnegativity():
    # sum_g W_pg = 1, W >= 0
    rng = np.random.default_rng(1)
    for order in (1, 2):
        for xi in rng.random(2000):
            _, w = oracle.support_1d(order, float(xi))
            assert (w >= 0).all()
            assert abs(w.sum() - 1.0) <= 4.5e-16     # a few ulp of 1
    # 2D product example SPEC.md:131: (0.25, 0.5) -> (.375, .375, .125, .125)
    _, wx = oracle.support_1d(1, 0.25)
    _, wy = oracle.support_1d(1, 0.5)
    assert list(np.outer(wx, wy).ravel()) == [0.375, 0.375, 0.125, 0.125]


# ------------------------------------------------------------------ alpha
def test_alpha_closed_forms():
    # PAPER.md:91-96
    assert (oracle.alpha([0, 0, 0]) == np.eye(3)).all()
    assert (oracle.alpha([0, 0, 1]) == 0.5 * np.array([[1, 1, 0], [-1, 1, 0], [0, 0, 2]])).all()
    assert (oracle.alpha([1, 1, 1]) == 0.25 * np.array([[2, 2, 0], [0, 2, 2], [2, 0, 2]])).all()


def test_alpha_is_inverse_of_I_plus_cross():
    # alpha = (I + C(omega))^-1 with C(omega) u = omega x u (reading R8); C built from np.cross,
    # the inverse by LAPACK — an independent route to eq_alpha_matrix.
    rng = np.random.default_rng(2)
    for om in rng.normal(size=(2000, 3)) * 2.0:
        C = np.stack([np.cross(om, e) for e in np.eye(3)], axis=1)
        a = oracle.alpha(om)
        assert np.abs(a @ (np.eye(3) + C) - np.eye(3)).max() < 1e-14
        assert np.abs(a - np.linalg.inv(np.eye(3) + C)).max() < 1e-14
        assert (oracle.alpha(-om) == a.T).all()       # alpha(-omega) = alpha(omega)^T exactly


# --------------------------------------------------- single-particle goldens
def _frac(v):
    return float(Fraction(v[0], v[1]))


@pytest.mark.parametrize("key", ["order1", "order2"])
def test_single_particle_golden(key):
    gd = GOLD[key]
    order = 1 if key == "order1" else 2
    n = gd["grid"]
    out = oracle.assemble(n, order, 9, [gd["x"]], [gd["q"]], [gd["B"]])
    g = lin(gd["node"], n)
    d0 = slot((0, 0, 0), order)
    for c, v in gd["diag"].items():
        assert out[g, d0, int(c)] == _frac(v)
    for c, v in gd["row_sum"].items():
        assert out[g, :, int(c)].sum() == _frac(v)
    assert np.count_nonzero(out) == gd["nonzeros"]
    assert out[:, :, 8].sum() == gd["total_comp8"]
    assert oracle.keys(n, order, [gd["x"]], [gd["q"]], [gd["B"]])[0] == gd["sort_key"]


def test_cic_1d_spec_example():
    gd = GOLD["cic_1d_spec"]
    n = gd["grid"]
    out = oracle.assemble(n, 1, 1, [gd["x"]], [gd["q"]])
    for node, d, v in gd["entries"]:
        assert out[lin(node, n), slot(d, 1), 0] == v
    assert np.count_nonzero(out) == len(gd["entries"])


# ------------------------------------------------------ dense brute force
def dense_W(n, pos, order):
    """W[g, p] = prod_mu phi(t_mu) with t the periodic-image distance in cell units
    (eq_weight_matrix PAPER.md:123-128 with eq_shape_bspline); phi written from its
    textbook piecewise definition, independent of the oracle."""
    n = np.asarray(n)
    gs = np.stack(np.meshgrid(*[np.arange(k) for k in n], indexing="ij"), -1).reshape(-1, 3)
    t = pos[None, :, :] - gs[:, None, :]
    t = (t + n / 2) % n - n / 2            # nearest periodic image
    a = np.abs(t)
    if order == 1:
        f = np.clip(1 - a, 0, None)
    else:
        f = np.where(a <= 0.5, 0.75 - a ** 2, np.where(a <= 1.5, 0.5 * (1.5 - a) ** 2, 0.0))
    return f.prod(-1)


def stencil_to_dense(out, n, order):
    R = order
    nn = int(np.prod(n))
    C = out.shape[2]
    D = np.zeros((C, nn, nn))
    rng = range(-R, R + 1)
    gs = np.stack(np.meshgrid(*[np.arange(k) for k in n], indexing="ij"), -1).reshape(-1, 3)
    for g, gv in enumerate(gs):
        for dx in rng:
            for dy in rng:
                for dz in rng:
                    h = ((gv[0] + dx) % n[0], (gv[1] + dy) % n[1], (gv[2] + dz) % n[2])
                    D[:, g, lin(h, n)] += out[g, slot((dx, dy, dz), R)]
    return D


@pytest.mark.parametrize("order,n,np_", [(1, (4, 4, 4), 300), (1, (3, 5, 4), 200), (2, (5, 5, 5), 300),
                                          (2, (6, 5, 7), 200)])
def test_dense_brute_force(order, n, np_):
    # eq_D_WSW: M^{ij} = W S^{ij} W^T, S^{ij} = diag(q alpha^{ij}),
    # alpha via LAPACK inverse of (I + C(omega)).
    d = synth.random_particles(n, np_, seed=7 + order, bscale=2.0, qrange=(-1.5, 1.5))
    out = oracle.assemble(n, order, 9, d["pos"], d["q"], d["B"])
    W = dense_W(n, d["pos"], order)
    s = np.empty((np_, 9))
    for p in range(np_):
        om = d["B"][p] / 2.0
        C = np.stack([np.cross(om, e) for e in np.eye(3)], axis=1)
        s[p] = (d["q"][p] * np.linalg.inv(np.eye(3) + C)).ravel()
    D = stencil_to_dense(out, n, order)
    scale = np.abs(W).sum(0).max() ** 2 * np.abs(s).max()
    for c in range(9):
        ref = (W * s[:, c]) @ W.T
        assert np.abs(D[c] - ref).max() <= 1e-13 * scale, c
    # row sparsity bound: at most (2n+1)^3 nonzeros per row
    assert (np.count_nonzero(D[0], axis=1) <= (2 * order + 1) ** 3).all()


# ------------------------------------------------------------- invariants
def _cfg_particles(order, n=(6, 5, 7), ppc=6, seed=11):
    cfg = synth.Config("t", n, order, "tensor", ppc, seed=seed)
    return synth.particles(cfg)


@pytest.mark.parametrize("order", [1, 2])
def test_partition_of_unity_moment(order):
    # PAPER.md:164 with eq_mass_matrix_general: sum_{g'} M^{ij}_{gg'} = sum_p s_p^{ij} W_pg.
    n = (6, 5, 7)
    d = _cfg_particles(order, n)
    out = oracle.assemble(n, order, 9, d["pos"], d["q"], d["B"])
    W = dense_W(n, d["pos"], order)
    s = np.stack([d["q"][p] * oracle.alpha(d["B"][p] / 2).ravel() for p in range(len(d["q"]))])
    mom = W @ s
    assert np.abs(out.sum(1) - mom).max() <= 1e-13 * np.abs(mom).max()
    assert np.abs(out.sum((0, 1)) - s.sum(0)).max() <= 1e-12 * np.abs(s).sum()


@pytest.mark.parametrize("order", [1, 2])
def test_spatial_symmetry_bit_exact(order):
    # eq_spatial_symmetry: out[g][d][ij] == out[g+d][-d][ij] exactly
    n = (6, 5, 7)
    d = _cfg_particles(order, n)
    out = oracle.assemble(n, order, 9, d["pos"], d["q"], d["B"])
    R = order
    gs = np.stack(np.meshgrid(*[np.arange(k) for k in n], indexing="ij"), -1).reshape(-1, 3)
    rr = range(-R, R + 1)
    for dd in [(a, b, c) for a in rr for b in rr for c in rr]:
        nb = np.array([lin(((g[0] + dd[0]) % n[0], (g[1] + dd[1]) % n[1], (g[2] + dd[2]) % n[2]), n)
                       for g in gs])
        assert (out[:, slot(dd, R)] == out[nb, slot(tuple(-x for x in dd), R)]).all()


@pytest.mark.parametrize("order", [1, 2])
def test_B_reversal_transposes_components(order):
    # alpha(-omega) = alpha(omega)^T (eq_alpha_matrix) => M^{ij}(B) = M^{ji}(-B)
    n = (5, 5, 5)
    d = _cfg_particles(order, n)
    a = oracle.assemble(n, order, 9, d["pos"], d["q"], d["B"])
    b = oracle.assemble(n, order, 9, d["pos"], d["q"], -d["B"])
    assert (a.reshape(-1, 3, 3) == b.reshape(-1, 3, 3).transpose(0, 2, 1)).all()


@pytest.mark.parametrize("order", [1, 2])
def test_B_zero_reduces_to_scalar(order):
    # alpha = I when B = 0 (eq_alpha_matrix) => M = M_scalar (x) I
    n = (5, 6, 5)
    d = _cfg_particles(order, n)
    t = oracle.assemble(n, order, 9, d["pos"], d["q"], np.zeros_like(d["B"]))
    s = oracle.assemble(n, order, 1, d["pos"], d["q"])
    for c in range(9):
        if c in (0, 4, 8):
            assert (t[:, :, c] == s[:, :, 0]).all()
        else:
            assert (t[:, :, c] == 0).all()


@pytest.mark.parametrize("order", [1, 2])
def test_linearity_and_charge_scaling(order):
    n = (5, 5, 6)
    d = _cfg_particles(order, n)
    full = oracle.assemble(n, order, 9, d["pos"], d["q"], d["B"])
    h = len(d["q"]) // 3
    a = oracle.assemble(n, order, 9, d["pos"][:h], d["q"][:h], d["B"][:h])
    b = oracle.assemble(n, order, 9, d["pos"][h:], d["q"][h:], d["B"][h:])
    assert np.abs(a + b - full).max() <= 1e-13 * np.abs(full).max()
    acc = oracle.assemble(n, order, 9, d["pos"][h:], d["q"][h:], d["B"][h:], out=a.copy(), accumulate=True)
    assert np.abs(acc - full).max() <= 1e-13 * np.abs(full).max()
    two = oracle.assemble(n, order, 9, d["pos"], 2 * d["q"], d["B"])
    assert (two == 2 * full).all()


@pytest.mark.parametrize("order", [1, 2])
def test_translation_by_one_cell(order):
    n = (5, 6, 7)
    d = _cfg_particles(order, n)
    lattice = synth.particles(synth.Config("t", n, order, "tensor", 3, seed=5), lattice=True)
    for dd in (d, lattice):
        base = oracle.assemble(n, order, 9, dd["pos"], dd["q"], dd["B"])
        sh = dd["pos"].copy()
        sh[:, 1] = (sh[:, 1] + 1.0) % n[1]
        moved = oracle.assemble(n, order, 9, sh, dd["q"], dd["B"])
        b4 = base.reshape(n[0], n[1], n[2], -1)
        m4 = moved.reshape(n[0], n[1], n[2], -1)
        tol = 0 if dd is lattice else 1e-13 * np.abs(base).max()
        assert np.abs(np.roll(b4, 1, axis=1) - m4).max() <= tol


@pytest.mark.parametrize("order", [1, 2])
def test_permutation_invariance(order):
    n = (5, 5, 5)
    d = _cfg_particles(order, n)
    a = oracle.assemble(n, order, 9, d["pos"], d["q"], d["B"])
    p = np.random.default_rng(3).permutation(len(d["q"]))
    b = oracle.assemble(n, order, 9, d["pos"][p], d["q"][p], d["B"][p])
    assert np.abs(a - b).max() <= 1e-13 * np.abs(a).max()


@pytest.mark.parametrize("order", [1, 2])
def test_lattice_inputs_order_independent_exactly(order):
    # dyadic lattice: every product and partial sum is exact, so any summation order gives the
    # same bits (the property the GPU lattice parity test relies on)
    n = (5, 5, 5)
    d = synth.particles(synth.Config("t", n, order, "tensor", 8, seed=9), lattice=True)
    a = oracle.assemble(n, order, 9, d["pos"], d["q"], d["B"])
    p = np.random.default_rng(4).permutation(len(d["q"]))
    b = oracle.assemble(n, order, 9, d["pos"][p], d["q"][p], d["B"][p])
    assert (a == b).all()
    W = dense_W(n, d["pos"], order)
    s = np.stack([d["q"][i] * oracle.alpha(d["B"][i] / 2).ravel() for i in range(len(d["q"]))])
    D = stencil_to_dense(a, n, order)
    for c in (0, 1, 5, 8):
        assert (D[c] == (W * s[:, c]) @ W.T).all()


# --------------------------------------------------------------------- sort
def test_sort_spec_example():
    # particles in cells [2,0,2,1] -> order [1,3,0,2]
    n = (5, 5, 5)
    pos = np.array([[2.5, 0.5, 0.5], [0.5, 0.5, 0.5], [2.25, 0.5, 0.5], [1.5, 0.5, 0.5]])
    r = oracle.sort(n, 1, 1, pos, np.ones(4))
    assert list(r["perm"]) == [1, 3, 0, 2]
    cells = [lin((k, 0, 0), n) for k in (0, 1, 2)]
    assert [int(r["seg_count"][c]) for c in cells] == [1, 1, 2]
    assert [int(r["seg_begin"][c]) for c in cells] == [0, 1, 2]


@pytest.mark.parametrize("order,k", [(1, 4), (1, 8), (2, 4), (2, 8), (1, 1)])
def test_sort_against_numpy_stable_argsort(order, k):
    n = (6, 5, 7)
    d = synth.random_particles(n, 2000, seed=21)
    # repeat some particles to force equal keys
    d["pos"][1000:1400] = d["pos"][:400]
    r = oracle.sort(n, order, k, d["pos"], d["q"], d["B"])
    key = oracle.keys(n, order, d["pos"], d["q"], d["B"])
    ref = np.argsort(key, kind="stable")
    perm = r["perm"]
    assert sorted(perm[perm >= 0].tolist()) == list(range(2000))
    assert (perm[perm >= 0] == ref).all()
    counts = np.bincount(key, minlength=oracle.nbins(n, order))
    assert (r["seg_count"] == counts).all()
    padded = (counts + k - 1) // k * k
    assert (r["seg_begin"] == np.concatenate([[0], np.cumsum(padded)])).all()
    assert r["np_padded"] == padded.sum()
    rec = r["rec"]
    assert (rec[perm < 0] == 0).all()
    src = perm[perm >= 0]
    assert (rec[perm >= 0, 3] == d["q"][src]).all()
    assert (rec[perm >= 0, 4:7] == d["B"][src]).all()
    u = d["pos"][src] / 1.0
    assert (rec[perm >= 0, :3] == u - np.floor(u)).all()


def test_keys_group_support_identity():
    # eq_group_partition: equal key <=> identical support node set.  For TSC the
    # 3-node window of an axis is centred on the nearest node, so the support set is
    # identified by the nearest node (axis 0 unwrapped, reading R12).
    n = (6, 6, 6)
    d = synth.random_particles(n, 3000, seed=3)
    key = oracle.keys(n, 2, d["pos"], d["q"], d["B"])
    centre = np.floor(d["pos"] + 0.5)
    centre[:, 1:] %= np.asarray(n[1:])
    ck = ((centre[:, 0] * n[1] + centre[:, 1]) * n[2] + centre[:, 2]).astype(np.int64)
    pairs = set(zip(key.tolist(), ck.tolist()))
    assert len({k for k, _ in pairs}) == len(pairs) == len({c for _, c in pairs})


def test_sort_errors():
    n = (5, 5, 5)
    with pytest.raises(oracle.OracleError):
        oracle.sort(n, 1, 4, [[5.0, 0, 0]], [1.0])
    with pytest.raises(oracle.OracleError) as e:
        oracle.sort(n, 1, 4, [[1.0, 0, 0]], [float("inf")])
    assert e.value.code == oracle.OR_ERR_NONFINITE
    with pytest.raises(oracle.OracleError) as e:
        oracle.sort((4, 5, 5), 2, 4, [[1.0, 0, 0]], [1.0])
    assert e.value.code == oracle.OR_ERR_INVALID_ARG
    r = oracle.sort(n, 1, 4, np.zeros((0, 3)), np.zeros(0))
    assert r["np_padded"] == 0 and (r["seg_count"] == 0).all()


# ------------------------------------------------------------- operator apply
@pytest.mark.parametrize("order,n", [(1, (4, 5, 3)), (2, (5, 6, 5))])
def test_apply_against_dense_WSW(order, n):
    # eq_field_eq: y = M E with M^{ij} = W diag(q alpha^{ij}) W^T (eq_D_WSW,
    # PAPER.md:141-144) built densely from the particles, independent of the stencil storage;
    # a transposed block (alpha^T) or a wrong slot/neighbour mapping fails it.
    np_ = 250
    d = synth.random_particles(n, np_, seed=31 + order, bscale=2.0, qrange=(-1.5, 1.5))
    out = oracle.assemble(n, order, 9, d["pos"], d["q"], d["B"])
    rng = np.random.default_rng(5)
    nn = int(np.prod(n))
    E = rng.standard_normal((nn, 3))
    y = oracle.apply(n, order, 9, out, E)
    W = dense_W(n, d["pos"], order)
    s = np.empty((np_, 3, 3))
    for p in range(np_):
        om = d["B"][p] / 2.0
        C = np.stack([np.cross(om, e) for e in np.eye(3)], axis=1)
        s[p] = d["q"][p] * np.linalg.inv(np.eye(3) + C)
    e_p = W.T @ E                                   # field at the particles, [np, 3]
    ref = W @ np.einsum("pij,pj->pi", s, e_p)       # sum_p W_pg s_p e_p
    scale = np.abs(W).sum(0).max() ** 2 * np.abs(s).max() * np.abs(E).max()
    assert np.abs(y - ref).max() <= 1e-13 * scale
    # accumulate adds; scalar kind applies the scalar matrix
    y2 = oracle.apply(n, order, 9, out, E, y=y.copy(), accumulate=True)
    assert np.allclose(y2, 2 * y, rtol=0, atol=1e-13 * scale)
    outs = oracle.assemble(n, order, 1, d["pos"], d["q"])
    f = E[:, 0]
    ys = oracle.apply(n, order, 1, outs, f)
    refs = W @ (d["q"] * (W.T @ f))
    assert np.abs(ys - refs).max() <= 1e-13 * np.abs(W).sum(0).max() ** 2 * 1.5 * np.abs(f).max()


def test_apply_constant_field_is_moment():
    # partition of unity: M 1 = sum_p s_p W_pg  (row sums), per component row i
    n, order = (5, 5, 6), 2
    d = _cfg_particles(order, n)
    out = oracle.assemble(n, order, 9, d["pos"], d["q"], d["B"])
    y = oracle.apply(n, order, 9, out, np.ones((int(np.prod(n)), 3)))
    W = dense_W(n, d["pos"], order)
    s = np.stack([d["q"][p] * oracle.alpha(d["B"][p] / 2) for p in range(len(d["q"]))])  # [np,3,3]
    ref = W @ s.sum(axis=2)
    assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()


def test_keys_on_a_slab_hand_derived():
    # Reading R12 on a slab: bx = c_x + b_x - x_begin + order - 1 (unwrapped, local),
    # by/bz wrapped; key = (bx n1 + by) n2 + bz.  Keys worked out by hand for grid (10, 5, 6),
    # slab [3, 7):
    #   (3.25, 1.5, 5.75): cell (3,1,5), xi (.25,.5,.75); CIC bx 0 -> key 11;
    #                      TSC base (-1, 0, 0) (xi_y = 1/2 ties to base 0, R4) -> bx 0 -> 11
    #   (6.9, 4.2, 0.1):   cell (6,4,0); CIC bx 3 -> (3*5+4)*6+0 = 114;
    #                      TSC base (0,-1,-1) -> bx 4, by 3, bz 5 -> (4*5+3)*6+5 = 143
    #   (3.0, 0.0, 0.0):   cell (3,0,0), xi 0; CIC key 0; TSC base -1: bx 0, by 4, bz 5 -> 29
    n, xb, xe = (10, 5, 6), 3, 7
    pos = np.array([[3.25, 1.5, 5.75], [6.9, 4.2, 0.1], [3.0, 0.0, 0.0]])
    q = np.ones(3)
    assert oracle.keys(n, 1, pos, q, x_begin=xb, x_end=xe).tolist() == [11, 114, 0]
    assert oracle.keys(n, 2, pos, q, x_begin=xb, x_end=xe).tolist() == [11, 143, 29]
    assert oracle.nbins(n, 1, xb, xe) == 4 * 5 * 6
    assert oracle.nbins(n, 2, xb, xe) == 5 * 5 * 6
    # outside the slab along x: a domain error (never clamped), also for the plane below x_begin
    for x in (2.99, 7.0, 9.5):
        with pytest.raises(oracle.OracleError) as e:
            oracle.keys(n, 1, [[x, 1.0, 1.0]], [1.0], x_begin=xb, x_end=xe)
        assert e.value.code == oracle.OR_ERR_DOMAIN
    # the slab sort places these three exactly as the hand keys say (K = 4 padding)
    r = oracle.sort(n, 2, 4, pos, q, x_begin=xb, x_end=xe)
    assert r["seg_count"][[11, 29, 143]].tolist() == [1, 1, 1] and r["seg_count"].sum() == 3
    assert r["seg_begin"][12] == 4 and r["seg_begin"][30] == 8 and r["seg_begin"][144] == 12
    assert r["perm"].tolist() == [0, -1, -1, -1, 2, -1, -1, -1, 1, -1, -1, -1]


@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("n", [(12, 5, 6), (9, 7, 5), (16, 5, 5)])
def test_assemble_omp_equals_serial(order, n):
    # the all-core timing variant of the oracle is the same sum in another order (x-slab
    # colouring): equal within rounding, bit-identical on the dyadic lattice
    from tests.helpers import rel_err
    d = synth.particles(synth.Config("t", n, order, "tensor", 9, seed=5 + order))
    a = oracle.assemble(n, order, 9, d["pos"], d["q"], d["B"])
    b, th = oracle.assemble_omp(n, order, 9, d["pos"], d["q"], d["B"])
    assert th >= 1 and rel_err(b, a) <= 1e-13
    dl = synth.particles(synth.Config("t", n, order, "tensor", 9, seed=6), lattice=True)
    a = oracle.assemble(n, order, 1, dl["pos"], dl["q"])
    b, _ = oracle.assemble_omp(n, order, 1, dl["pos"], dl["q"])
    assert (a == b).all()


# ------------------------------------------------- NEXT-4: moments and field gather
def test_moments_single_particle_hand_values():
    # CIC, grid 4^3, x = (1.25, 2.5, 3.75), q = 2, v = (1, -2, 1/2): weights x {1: 3/4, 2: 1/4},
    # y {2: 1/2, 3: 1/2}, z {3: 1/4, 0: 3/4} (z wraps).  At node (1, 2, 3): W = 3/32, rho = q W = 3/16,
    # J = rho v = (3/16, -3/8, 3/32), second moments rho (vx vx, vx vy, vx vz, vy vy, vy vz, vz vz)
    # = (3/16, -3/8, 3/32, 3/4, -3/16, 3/64); 8 nonzero nodes, total charge q
    n = (4, 4, 4)
    m = oracle.moments(n, 1, 10, [[1.25, 2.5, 3.75]], [2.0], [[1.0, -2.0, 0.5]])
    exp = [Fraction(3, 16), Fraction(3, 16), Fraction(-3, 8), Fraction(3, 32), Fraction(3, 16), Fraction(-3, 8),
           Fraction(3, 32), Fraction(3, 4), Fraction(-3, 16), Fraction(3, 64)]
    assert [Fraction(x) for x in m[lin((1, 2, 3), n)]] == exp
    assert np.count_nonzero(m[:, 0]) == 8 and m[:, 0].sum() == 2.0
    m4 = oracle.moments(n, 1, 4, [[1.25, 2.5, 3.75]], [2.0], [[1.0, -2.0, 0.5]])
    assert (m4 == m[:, :4]).all()
    # TSC: x = (1.25, 2.5, 3.75) on 5^3: x {0: 1/32, 1: 11/16, 2: 9/32}, y {2: 1/2, 3: 1/2},
    # z {3: 9/32, 4: 11/16, 0: 1/32}; rho at (1, 3, 4) = 2 (11/16)(1/2)(11/16) = 121/256
    m2 = oracle.moments((5, 5, 5), 2, 4, [[1.25, 2.5, 3.75]], [2.0], [[1.0, -2.0, 0.5]])
    assert Fraction(m2[lin((1, 3, 4), (5, 5, 5)), 0]) == Fraction(121, 256)
    assert Fraction(m2[lin((1, 3, 4), (5, 5, 5)), 2]) == Fraction(-121, 128)


@pytest.mark.parametrize("order,n", [(1, (4, 5, 3)), (2, (5, 6, 5)), (2, (7, 5, 6))])
def test_moments_dense_and_totals(order, n):
    # mom = W^T Q with the dense periodic W of the explicit B-spline definition (eq_weight_matrix)
    d = synth.random_particles(n, 300, seed=17 + order, qrange=(-1.5, 1.5))
    v = np.random.default_rng(3).uniform(-2, 2, (300, 3))
    m = oracle.moments(n, order, 10, d["pos"], d["q"], v, sigma=0.5)
    W = dense_W(n, d["pos"], order)
    Q = d["q"][:, None] * np.column_stack([np.ones(300), v, v[:, 0] * v[:, 0], v[:, 0] * v[:, 1], v[:, 0] * v[:, 2],
                                          v[:, 1] * v[:, 1], v[:, 1] * v[:, 2], v[:, 2] * v[:, 2]])
    ref = 0.5 * W @ Q
    assert np.abs(m - ref).max() <= 1e-13 * np.abs(Q).max() * 8
    # partition of unity: sum over nodes = sigma sum_p Q_p
    assert np.allclose(m.sum(0), 0.5 * Q.sum(0), rtol=1e-13, atol=1e-13 * np.abs(Q).sum())


@pytest.mark.parametrize("order", [1, 2])
def test_charge_density_is_scalar_mass_row_sum(order):
    # rho_g = sum_p q_p W_pg = sum_{g'} M_{gg'} of the scalar mass matrix (partition of unity,
    # PAPER.md:164, applied to the pinned assembly)
    n = (6, 5, 7)
    d = _cfg_particles(order)
    v = np.zeros_like(d["pos"])
    rho = oracle.moments(n, order, 4, d["pos"], d["q"], v)[:, 0]
    M = oracle.assemble(n, order, 1, d["pos"], d["q"])
    assert np.allclose(rho, M[:, :, 0].sum(1), rtol=1e-13, atol=1e-14)


@pytest.mark.parametrize("order", [1, 2])
def test_gather_dense_constant_linear_and_adjoint(order):
    n = (6, 7, 5)
    rng = np.random.default_rng(9 + order)
    d = synth.random_particles(n, 400, seed=23 + order)
    nn = int(np.prod(n))
    F = rng.standard_normal((nn, 3))
    Fp = oracle.gather(n, order, d["pos"], F)
    W = dense_W(n, d["pos"], order)
    assert np.abs(Fp - W.T @ F).max() <= 1e-13 * np.abs(F).max() * 8
    # a constant field is reproduced (partition of unity)
    Fc = np.tile([1.5, -0.25, 3.0], (nn, 1))
    assert np.abs(oracle.gather(n, order, d["pos"], Fc) - [1.5, -0.25, 3.0]).max() <= 1e-14
    # a linear field is reproduced exactly by both B-splines away from the periodic seam
    nl = (10, 9, 11)
    gs = np.stack(np.meshgrid(*[np.arange(k) for k in nl], indexing="ij"), -1).reshape(-1, 3).astype(float)
    A = np.array([[0.5, 1.0, 0.0], [-1.0, 0.25, 2.0], [0.0, 3.0, -0.5]])
    Fl = gs @ A + [1.0, 2.0, 3.0]
    xp = 2.0 + rng.random((300, 3)) * (np.array(nl) - 5.0)      # support windows never wrap
    assert np.abs(oracle.gather(nl, order, xp, Fl) - (xp @ A + [1.0, 2.0, 3.0])).max() <= 1e-12
    # adjointness: the gather is the transpose of the deposit, sum_p F(x_p).(q v)_p = sum_g F_g.J_g
    v = rng.uniform(-1, 1, (400, 3))
    J = oracle.moments(n, order, 4, d["pos"], d["q"], v)[:, 1:4]
    lhs = np.sum(Fp * d["q"][:, None] * v)
    assert abs(lhs - np.sum(F * J)) <= 1e-12 * np.sum(np.abs(F).max() * np.abs(d["q"][:, None] * v))
