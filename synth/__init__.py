"""Seeded synthetic plasma generators shared by the oracle checks and the CUDA path.

This module holds NONE of the method's arithmetic (no shape functions, no
alpha, no binning): it only draws particle positions, charges and magnetic
fields with numpy's counter-based Philox generator, with the shapes, sizes
and distributions of the paper's isolation runs (uniform
ppc, pre-sorted cells; here the input order is a random shuffle, the sort's
worst case) and of its production run (a double Harris sheet,
imitated by the clustered profile of config c4).  The recipe is stated in
DESIGN.md §Inputs.

Each x-plane of cells has its own Philox stream keyed by (seed, plane), so
the particle set of a slab is the same for any number of ranks.
"""
from __future__ import annotations

import dataclasses
import numpy as np

SEED0 = 19286


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n: tuple                  # cells = nodes per axis
    order: int                # B-spline order (1 CIC, 2 TSC)
    kind: str                 # "tensor" (ECSIM, 9 comps) | "scalar" (MPM, 1 comp)
    ppc: int                  # particles per cell (mean for "clustered")
    dist: str = "uniform"     # "uniform" | "clustered"
    bfield: str = "random"    # "random" U[-1,1]^3 per particle | "uniform" B=(0,0,2)
    seed: int = SEED0
    h: tuple = (1.0, 1.0, 1.0)
    qom: float = 1.0
    dt: float = 1.0
    c: float = 1.0
    sigma: float = 1.0

    @property
    def ncomp(self):
        return 9 if self.kind == "tensor" else 1

    @property
    def ncells(self):
        return self.n[0] * self.n[1] * self.n[2]


# BASELINE.json "configs" (index = list position); c4 and c5 come in an order-1 and an order-2 flavour.
CONFIGS = {
    "c1": Config("c1", (4, 4, 4), 1, "tensor", 16, bfield="uniform", seed=SEED0 + 0),
    "c2": Config("c2", (64, 64, 64), 1, "tensor", 64, seed=SEED0 + 1),
    "c3": Config("c3", (64, 64, 64), 2, "tensor", 64, seed=SEED0 + 2),
    "c4o1": Config("c4o1", (128, 128, 128), 1, "scalar", 64, dist="clustered", seed=SEED0 + 3),
    "c4o2": Config("c4o2", (128, 128, 128), 2, "scalar", 64, dist="clustered", seed=SEED0 + 3),
    "c5o1": Config("c5o1", (256, 256, 256), 1, "tensor", 64, seed=SEED0 + 4),
    "c5o2": Config("c5o2", (256, 256, 256), 2, "tensor", 64, seed=SEED0 + 4),
}


def config(name: str, **over) -> Config:
    return dataclasses.replace(CONFIGS[name], **over)


def clustered_counts(ny: int, ppc: int, lam: float = 2.9) -> np.ndarray:
    """Per-y-row particle count of a double-Harris-like profile:
    f(y) = 0.1 + sech^2((y - Ly/4)/lam) + sech^2((y - 3Ly/4)/lam), y at the cell centre,
    count = round(ppc * f / mean f)."""
    y = np.arange(ny) + 0.5
    f = 0.1 + np.cosh((y - ny / 4) / lam) ** -2 + np.cosh((y - 3 * ny / 4) / lam) ** -2
    return np.rint(ppc * f / f.mean()).astype(np.int64)


def _stream(seed: int, plane: int, salt: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=(int(seed) << 24) ^ (int(plane) << 2) ^ salt))


def particles(cfg: Config, x_begin: int = 0, x_end: int | None = None, shuffle=True,
              lattice: bool = False, lattice_den: int | None = None) -> dict:
    """Particles located in the cell slab [x_begin, x_end) x [0,n1) x [0,n2).

    Returns dict(pos[np,3], q[np], B[np,3]) as float64 numpy arrays.  Input order: a uniform
    random shuffle (shuffle=True, the sort's worst case), cell-sorted (False) or "nearly"
    sorted (a random 10% of the particles permuted among themselves, the PIC-step regime).
    lattice=True draws the dyadic variant: xi in {k/16} (order 1)
    or {k/4} (order 2) (lattice_den overrides the denominator), q in {1, 2, -1}, B = 2*omega with omega in
    {0, +-e_i, (+-1,+-1,+-1)} so that every product and partial sum of the
    assembly is exact in FP64.
    """
    n0, n1, n2 = cfg.n
    x_end = n0 if x_end is None else x_end
    if cfg.dist == "uniform":
        row_counts = np.full(n1, cfg.ppc, dtype=np.int64)
    elif cfg.dist == "clustered":
        row_counts = clustered_counts(n1, cfg.ppc)
    else:
        raise ValueError(cfg.dist)
    per_plane = int(row_counts.sum()) * n2
    # cell (y, z) index of each particle inside one x-plane (identical for every plane)
    cy = np.repeat(np.arange(n1, dtype=np.int64), row_counts * n2)
    cz = np.concatenate([np.repeat(np.arange(n2, dtype=np.int64), int(c)) for c in row_counts])
    nplanes = x_end - x_begin
    total = per_plane * nplanes
    pos = np.empty((total, 3))
    q = np.empty(total)
    B = np.empty((total, 3))
    h = np.asarray(cfg.h, dtype=np.float64)
    omega_set = np.array([[0, 0, 0], [1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1],
                          [1, 1, 1], [-1, 1, -1], [1, -1, -1], [-1, -1, 1]], dtype=np.float64)
    for k, ix in enumerate(range(x_begin, x_end)):
        rng = _stream(cfg.seed, ix)
        sl = slice(k * per_plane, (k + 1) * per_plane)
        if lattice:
            den = lattice_den or (16 if cfg.order == 1 else 4)
            xi = rng.integers(0, den, size=(per_plane, 3)).astype(np.float64) / den
            qq = np.array([1.0, 2.0, -1.0])[rng.integers(0, 3, size=per_plane)]
            om = omega_set[rng.integers(0, len(omega_set), size=per_plane)]
            bb = 2.0 * om * (cfg.c / (cfg.qom * cfg.dt))
        else:
            xi = rng.random((per_plane, 3))
            qq = rng.uniform(0.5, 1.5, size=per_plane)
            if cfg.bfield == "uniform":
                bb = np.broadcast_to(np.array([0.0, 0.0, 2.0]), (per_plane, 3))
            else:
                bb = rng.uniform(-1.0, 1.0, size=(per_plane, 3))
        cell = np.stack([np.full(per_plane, ix, dtype=np.int64), cy, cz], axis=1).astype(np.float64)
        x = (cell + xi) * h
        # guard the (rare) rounding of c + xi up to c + 1: keep the particle in its cell
        bad = np.floor(x / h) != cell
        x[bad] = (cell * h)[bad]
        pos[sl] = x
        q[sl] = qq
        B[sl] = bb
    if shuffle == "nearly" and total > 1:
        # generation order is cell-sorted; a PIC step leaves particles nearly sorted:
        # a random 10% of them are permuted among themselves (a true permutation: every
        # particle appears exactly once)
        rng = _stream(cfg.seed, x_begin, salt=2)
        k = total // 10
        idx = rng.choice(total, size=k, replace=False)
        perm = np.arange(total)
        perm[idx] = idx[rng.permutation(k)]
        pos, q, B = pos[perm], q[perm], B[perm]
    elif shuffle and total > 1:
        perm = _stream(cfg.seed, x_begin, salt=1).permutation(total)
        pos, q, B = pos[perm], q[perm], B[perm]
    return {"pos": np.ascontiguousarray(pos), "q": np.ascontiguousarray(q), "B": np.ascontiguousarray(B)}


def particles_device(cfg: Config, device, with_B: bool = True, x_begin: int = 0, x_end: int | None = None) -> dict:
    """The same recipe as particles() (cell counts, xi ~ U[0,1)^3, q ~ U[0.5,1.5], B ~ U[-1,1]^3,
    uniform random input order), drawn on the GPU with torch's Philox generator seeded by
    cfg.seed (and x_begin), for the cell slab [x_begin, x_end) (default: the whole grid).  Same
    distribution, NOT the same sample as particles(): bench.py uses it for the large configs
    (c4: 134.7 M particles, the c5 weak-scaling slabs) whose host generation would take minutes;
    the parity tests that use it compare against the oracle run on the same drawn particles."""
    import torch
    n0, n1, n2 = cfg.n
    x_end = n0 if x_end is None else x_end
    if cfg.dist == "uniform":
        row_counts = np.full(n1, cfg.ppc, dtype=np.int64)
    else:
        row_counts = clustered_counts(n1, cfg.ppc)
    gen = torch.Generator(device=device)
    gen.manual_seed(int(cfg.seed) + 1000003 * int(x_begin))
    per_plane = int(row_counts.sum()) * n2
    total = per_plane * (x_end - x_begin)
    cnt_yz = torch.from_numpy(np.repeat(row_counts, n2)).to(device)          # per (y, z) cell
    yz = torch.repeat_interleave(torch.arange(n1 * n2, device=device), cnt_yz)  # [per_plane]
    ix = torch.arange(x_begin, x_end, device=device).repeat_interleave(per_plane)
    iyz = yz.repeat(x_end - x_begin)
    cell = torch.stack([ix, iyz // n2, iyz % n2], dim=1).to(torch.float64)
    del ix, iyz, yz
    h = torch.tensor(cfg.h, dtype=torch.float64, device=device)
    pos = (cell + torch.rand((total, 3), generator=gen, dtype=torch.float64, device=device)) * h
    bad = torch.floor(pos / h) != cell
    pos = torch.where(bad, cell * h, pos)
    del cell, bad
    q = 0.5 + torch.rand(total, generator=gen, dtype=torch.float64, device=device)
    perm = torch.randperm(total, generator=gen, device=device)
    out = {"pos": pos[perm].contiguous(), "q": q[perm].contiguous()}
    del pos, q
    if with_B:
        out["B"] = (2.0 * torch.rand((total, 3), generator=gen, dtype=torch.float64, device=device) - 1.0)[perm]
    return out


def random_particles(n, np_, seed, h=(1.0, 1.0, 1.0), bscale=1.0, qrange=(0.5, 1.5)):
    """np_ particles uniformly distributed over the whole periodic box (Poisson ppc)."""
    rng = np.random.Generator(np.random.Philox(key=int(seed)))
    L = np.asarray(n, dtype=np.float64) * np.asarray(h)
    pos = rng.random((np_, 3)) * L
    pos = np.where(pos >= L, 0.0, pos)
    q = rng.uniform(qrange[0], qrange[1], size=np_)
    B = rng.uniform(-bscale, bscale, size=(np_, 3))
    return {"pos": pos, "q": q, "B": B}


def ppc_of(cfg: Config) -> float:
    if cfg.dist == "uniform":
        return float(cfg.ppc)
    return float(clustered_counts(cfg.n[1], cfg.ppc).mean())


def num_particles(cfg: Config, x_begin=0, x_end=None) -> int:
    x_end = cfg.n[0] if x_end is None else x_end
    if cfg.dist == "uniform":
        rows = cfg.ppc * cfg.n[1]
    else:
        rows = int(clustered_counts(cfg.n[1], cfg.ppc).sum())
    return rows * cfg.n[2] * (x_end - x_begin)


__all__ = ["Config", "CONFIGS", "config", "particles", "particles_device", "random_particles", "clustered_counts",
           "num_particles", "ppc_of"]
