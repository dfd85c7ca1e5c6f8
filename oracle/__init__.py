"""ORACLE — TEST INFRASTRUCTURE ONLY.

Plain FP64 CPU oracle for the ECSIM mass-matrix assembly of arXiv 2604.19286
(eq_mass_matrix_general).  The arithmetic lives in
``oracle/oracle.c`` (plain C, single thread, input order); this module only
compiles it with gcc and marshals numpy arrays through ctypes.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  It
shares no code with ``paper_2604_19286_b200`` and never imports it.

Parity status of each function:
  phi / support_1d / alpha / locate  — pinned (SPEC/PAPER worked examples,
                                       closed forms, identities)
  keys / sort                        — pinned (numpy stable argsort, SPEC
                                       example, permutation invariants)
  assemble                           — pinned (hand-derived single-particle
                                       goldens, dense W S W^T brute force,
                                       partition of unity, symmetries)
  assemble_omp                       — timing only; equal to assemble (test)
  moments                            — pinned (hand-derived single particle,
                                       dense W^T Q, row sums of the pinned
                                       scalar mass matrix, totals)
  gather                             — pinned (dense W F, constant and linear
                                       field reproduction, adjointness with
                                       moments)
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

OR_OK, OR_ERR_INVALID_ARG, OR_ERR_DOMAIN, OR_ERR_NONFINITE = 0, 1, 2, 3


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"oracle {what} failed with code {code}")
        self.code = code


class _Grid(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32 * 3), ("h", ctypes.c_double * 3),
                ("x_begin", ctypes.c_int32), ("x_end", ctypes.c_int32)]


class _Species(ctypes.Structure):
    _fields_ = [("qom", ctypes.c_double), ("dt", ctypes.c_double),
                ("c", ctypes.c_double), ("sigma", ctypes.c_double)]


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (plain -O2, no fast-math, no FMA contraction)."""
    with _lock:
        if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-ffp-contract=off",
                                   "-fno-fast-math", "-fopenmp", "-o", tmp, _SRC, "-lm"])
            os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        lib.or_phi.restype = ctypes.c_double
        lib.or_phi.argtypes = [ctypes.c_int, ctypes.c_double]
        lib.or_support_1d.argtypes = [ctypes.c_int, ctypes.c_double, P, P]
        lib.or_alpha.argtypes = [P, P]
        lib.or_alpha.restype = None
        lib.or_locate.argtypes = [P, P, P, P]
        lib.or_keys.argtypes = [P, ctypes.c_int, ctypes.c_int64, P, P, P, P]
        lib.or_nbins.restype = ctypes.c_int64
        lib.or_nbins.argtypes = [P, ctypes.c_int]
        lib.or_sort.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int64, P, P, P, P, P, P, P, P]
        lib.or_assemble.argtypes = [P, ctypes.c_int, ctypes.c_int, P, ctypes.c_int64, P, P, P, P,
                                    ctypes.c_int]
        lib.or_apply.argtypes = [P, ctypes.c_int, ctypes.c_int, P, P, P, ctypes.c_int]
        lib.or_moments.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int64, P, P, P, P,
                                   ctypes.c_int]
        lib.or_gather.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int64, P, P, P]
        lib.or_assemble_omp.argtypes = [P, ctypes.c_int, ctypes.c_int, P, ctypes.c_int64, P, P, P, P,
                                        ctypes.c_int, P]
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _grid(n, h=(1.0, 1.0, 1.0), x_begin=0, x_end=None):
    g = _Grid()
    for i in range(3):
        g.n[i] = int(n[i])
        g.h[i] = float(h[i])
    g.x_begin = int(x_begin)
    g.x_end = int(n[0] if x_end is None else x_end)
    return g


def _f64(a, shape=None):
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


def phi(order: int, t: float) -> float:
    """1D B-spline phi^(n)(t) — PAPER.md:159-163."""
    return _load().or_phi(order, t)


def support_1d(order: int, xi: float):
    """(base, weights[order+1]) of one axis — PAPER.md:166-168."""
    base = ctypes.c_int32()
    w = np.zeros(3)
    rc = _load().or_support_1d(order, xi, ctypes.byref(base), _ptr(w))
    if rc:
        raise OracleError(rc, "support_1d")
    return base.value, w[: order + 1].copy()


def alpha(omega) -> np.ndarray:
    """3x3 rotation-response tensor — PAPER.md:91-96 (eq_alpha_matrix)."""
    om = _f64(omega, (3,))
    a = np.zeros(9)
    _load().or_alpha(_ptr(om), _ptr(a))
    return a.reshape(3, 3)


def locate(x, n=(64, 64, 64), h=(1.0, 1.0, 1.0), x_begin=0, x_end=None):
    g = _grid(n, h, x_begin, x_end)
    xx = _f64(x, (3,))
    cell = np.zeros(3, dtype=np.int32)
    xi = np.zeros(3)
    rc = _load().or_locate(ctypes.byref(g), _ptr(xx), _ptr(cell), _ptr(xi))
    if rc:
        raise OracleError(rc, "locate")
    return cell, xi


def nbins(n, order, x_begin=0, x_end=None, h=(1.0, 1.0, 1.0)):
    g = _grid(n, h, x_begin, x_end)
    return int(_load().or_nbins(ctypes.byref(g), order))


def keys(n, order, pos, q, B=None, h=(1.0, 1.0, 1.0), x_begin=0, x_end=None):
    g = _grid(n, h, x_begin, x_end)
    pos = _f64(pos, (-1, 3))
    np_ = pos.shape[0]
    q = _f64(q, (np_,))
    B = _f64(B, (np_, 3))
    key = np.zeros(max(np_, 1), dtype=np.uint32)
    rc = _load().or_keys(ctypes.byref(g), order, np_, _ptr(pos), _ptr(q), _ptr(B), _ptr(key))
    if rc:
        raise OracleError(rc, "keys")
    return key[:np_]


def sort(n, order, k_pad, pos, q, B=None, h=(1.0, 1.0, 1.0), x_begin=0, x_end=None, records=True):
    """Stable bin sort with K-padding.  Returns dict(perm, seg_begin, seg_count, np_padded, rec)."""
    g = _grid(n, h, x_begin, x_end)
    pos = _f64(pos, (-1, 3))
    np_ = pos.shape[0]
    q = _f64(q, (np_,))
    B = _f64(B, (np_, 3))
    nb = nbins(n, order, x_begin, x_end, h)
    cap = np_ + nb * (k_pad - 1)
    perm = np.full(max(cap, 1), -7, dtype=np.int32)
    seg_begin = np.zeros(nb + 1, dtype=np.int32)
    seg_count = np.zeros(nb, dtype=np.int32)
    npp = ctypes.c_int64()
    rec = np.zeros((max(cap, 1), 8)) if records else None
    rc = _load().or_sort(ctypes.byref(g), order, k_pad, np_, _ptr(pos), _ptr(q), _ptr(B), _ptr(perm),
                         _ptr(seg_begin), _ptr(seg_count), ctypes.byref(npp), _ptr(rec))
    if rc:
        raise OracleError(rc, "sort")
    m = npp.value
    return {"perm": perm[:m], "seg_begin": seg_begin, "seg_count": seg_count, "np_padded": m,
            "rec": None if rec is None else rec[:m]}


def assemble(n, order, ncomp, pos, q, B=None, h=(1.0, 1.0, 1.0), qom=1.0, dt=1.0, c=1.0, sigma=1.0,
             out=None, accumulate=False):
    """M[g][slot][comp] over the whole periodic grid — PAPER.md:101-104."""
    g = _grid(n, h)
    sp = _Species(qom, dt, c, sigma)
    pos = _f64(pos, (-1, 3))
    np_ = pos.shape[0]
    q = _f64(q, (np_,))
    B = _f64(B, (np_, 3))
    S = (2 * order + 1) ** 3
    nn = int(n[0]) * int(n[1]) * int(n[2])
    if out is None:
        out = np.zeros((nn, S, ncomp))
        accumulate = False
    assert out.dtype == np.float64 and out.flags.c_contiguous and out.size == nn * S * ncomp
    rc = _load().or_assemble(ctypes.byref(g), order, ncomp, ctypes.byref(sp), np_, _ptr(pos), _ptr(q),
                             _ptr(B), _ptr(out), int(bool(accumulate)))
    if rc:
        raise OracleError(rc, "assemble")
    return out


def assemble_omp(n, order, ncomp, pos, q, B=None, h=(1.0, 1.0, 1.0), qom=1.0, dt=1.0, c=1.0, sigma=1.0):
    """or_assemble on all host cores (x-slab colouring; timing the CPU baseline only).
    Returns (out, threads used)."""
    g = _grid(n, h)
    sp = _Species(qom, dt, c, sigma)
    pos = _f64(pos, (-1, 3))
    np_ = pos.shape[0]
    q = _f64(q, (np_,))
    B = _f64(B, (np_, 3))
    S = (2 * order + 1) ** 3
    out = np.empty((int(n[0]) * int(n[1]) * int(n[2]), S, ncomp))
    th = ctypes.c_int(1)
    rc = _load().or_assemble_omp(ctypes.byref(g), order, ncomp, ctypes.byref(sp), np_, _ptr(pos), _ptr(q), _ptr(B),
                                 _ptr(out), 0, ctypes.byref(th))
    if rc:
        raise OracleError(rc, "assemble_omp")
    return out, th.value


def moments(n, order, nq, pos, q, v, sigma=1.0, h=(1.0, 1.0, 1.0), out=None, accumulate=False):
    """Particle moments on the nodes, [nodes][nq] (nq = 4: rho, J; 10: + the second-moment
    tensor) — PAPER.md:591 (oracle.c or_moments)."""
    g = _grid(n, h)
    pos = _f64(pos, (-1, 3))
    np_ = pos.shape[0]
    q = _f64(q, (np_,))
    v = _f64(v, (np_, 3))
    nn = int(n[0]) * int(n[1]) * int(n[2])
    if out is None:
        out = np.zeros((nn, nq))
        accumulate = False
    assert out.dtype == np.float64 and out.flags.c_contiguous and out.size == nn * nq
    rc = _load().or_moments(ctypes.byref(g), order, nq, float(sigma), np_, _ptr(pos), _ptr(q), _ptr(v), _ptr(out),
                            int(bool(accumulate)))
    if rc:
        raise OracleError(rc, "moments")
    return out


def gather(n, order, pos, F, h=(1.0, 1.0, 1.0)):
    """A nodal field F [nodes][ncomp] interpolated to the particles, [np][ncomp] — PAPER.md:96
    (oracle.c or_gather)."""
    g = _grid(n, h)
    pos = _f64(pos, (-1, 3))
    np_ = pos.shape[0]
    nn = int(n[0]) * int(n[1]) * int(n[2])
    F = _f64(F).reshape(nn, -1)
    nc = F.shape[1]
    Fp = np.zeros((np_, nc))
    rc = _load().or_gather(ctypes.byref(g), order, nc, np_, _ptr(pos), _ptr(F), _ptr(Fp))
    if rc:
        raise OracleError(rc, "gather")
    return Fp


def apply(n, order, ncomp, M, E, y=None, accumulate=False):
    """y (+)= M E over the whole periodic grid — eq_field_eq, PAPER.md:77-83 (plain loops).
    M: [nodes][S][ncomp]; E, y: [nodes][3] (ncomp 9) or [nodes] (ncomp 1)."""
    g = _grid(n)
    nn = int(n[0]) * int(n[1]) * int(n[2])
    S = (2 * order + 1) ** 3
    nv = 3 if ncomp == 9 else 1
    M = _f64(M, (nn, S, ncomp))
    E = _f64(E, (nn, nv) if nv == 3 else (nn,))
    if y is None:
        y = np.zeros(E.shape)
        accumulate = False
    assert y.dtype == np.float64 and y.flags.c_contiguous and y.size == nn * nv
    rc = _load().or_apply(ctypes.byref(g), order, ncomp, _ptr(M), _ptr(E), _ptr(y), int(bool(accumulate)))
    if rc:
        raise OracleError(rc, "apply")
    return y
