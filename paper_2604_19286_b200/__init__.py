"""B200-native ECSIM mass-matrix assembly (arXiv 2604.19286) — Python binding.

A thin ctypes binding over the C ABI of ``libmm.so`` (``include/mm.h``).  It
only marshals arguments: torch tensors are passed as device pointers, the
current torch CUDA stream as the stream.  Every step of the hot path runs in
the library's CUDA kernels; there is no CPU fallback, and importing the
package on a box without the built library raises.

Entry points (same names as the C ABI):
    mm_sort_by_cell(grid, order, k_pad, pos, q, B=None, handle=None) -> Sorted
    mm_sorted_view(handle) -> dict of device tensors (perm, seg_begin, seg_count, rec)
    mm_assemble(handle, kind, prec, species, out, ghost=None, accumulate=False)
    mm_ghost_add(grid, order, kind, out, recv, first_plane, nplanes)
    mm_comm_unique_id() / mm_comm_create(nranks, rank, uid) -> Comm / mm_comm_free(comm)
    mm_ghost_exchange(comm, grid, order, kind, prec, out, ghost)
    mm_assemble_slab(handle, kind, prec, species, out, ghost, comm, accumulate=False)
    mm_free(handle)
plus helpers (Grid, Species, out_shape, ghost_shape, ...).
"""
from __future__ import annotations

import ctypes
import os

import torch

from . import _build

MM_OK, MM_ERR_INVALID_ARG, MM_ERR_DOMAIN, MM_ERR_NONFINITE, MM_ERR_INCOMPATIBLE, MM_ERR_OUT_OF_MEMORY, \
    MM_ERR_CUDA, MM_ERR_NCCL = range(8)
MM_SCALAR, MM_TENSOR = 1, 9
MM_FP64, MM_TF32, MM_TF32X3 = 0, 1, 2

_STATUS_NAMES = {0: "MM_OK", 1: "MM_ERR_INVALID_ARG", 2: "MM_ERR_DOMAIN", 3: "MM_ERR_NONFINITE",
                 4: "MM_ERR_INCOMPATIBLE", 5: "MM_ERR_OUT_OF_MEMORY", 6: "MM_ERR_CUDA", 7: "MM_ERR_NCCL"}

# Every symbol include/mm.h declares (checked by the CPU test suite).
EXPORTS = ["mm_sort_by_cell", "mm_sort_by_cell_mixed", "mm_sort_by_cell_async", "mm_sort_wait", "mm_resort_by_cell", "mm_slab_partition", "mm_sorted_view", "mm_assemble",
           "mm_assemble_slab", "mm_deposit_moments", "mm_gather_field", "mm_apply", "mm_ghost_add", "mm_ghost_exchange", "mm_ghost_planes", "mm_out_elems",
           "mm_comm_unique_id", "mm_comm_create", "mm_comm_free", "mm_free", "mm_last_error", "mm_version",
           "mm_launch_count"]


class MMError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class mm_grid(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32 * 3), ("h", ctypes.c_double * 3), ("x_begin", ctypes.c_int32),
                ("x_end", ctypes.c_int32)]


class mm_species(ctypes.Structure):
    _fields_ = [("qom", ctypes.c_double), ("dt", ctypes.c_double), ("c", ctypes.c_double),
                ("sigma", ctypes.c_double)]


class mm_sorted_info(ctypes.Structure):
    _fields_ = [("np", ctypes.c_int64), ("np_padded", ctypes.c_int64), ("nbins", ctypes.c_int64),
                ("capacity", ctypes.c_int64), ("order", ctypes.c_int32), ("k_pad", ctypes.c_int32),
                ("has_B", ctypes.c_int32), ("rec_stride", ctypes.c_int32), ("perm", ctypes.c_void_p),
                ("seg_begin", ctypes.c_void_p), ("seg_count", ctypes.c_void_p), ("rec", ctypes.c_void_p)]


_lib = None


def load_library(build_if_missing: bool = True):
    """Load libmm.so from the package directory (build it with nvcc if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_build.LIB):
        if not build_if_missing:
            raise ImportError(f"{_build.LIB} is missing; run __graft_entry__.build()")
        _build.build()
    lib = ctypes.CDLL(_build.LIB)
    P, I64, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    lib.mm_sort_by_cell.argtypes = [P, I, I, I64, P, P, P, P, P]
    lib.mm_sort_by_cell_mixed.restype = I
    lib.mm_sort_by_cell_mixed.argtypes = [P, I, I, I64, P, P, P, P, P]
    lib.mm_sort_by_cell.restype = I
    lib.mm_sort_by_cell_async.argtypes = [P, I, I, I64, P, P, P, P, P]
    lib.mm_sort_by_cell_async.restype = I
    lib.mm_resort_by_cell.argtypes = [P, I64, P, P, P, P, I]
    lib.mm_resort_by_cell.restype = I
    lib.mm_sort_wait.argtypes = [P, P]
    lib.mm_sort_wait.restype = I
    lib.mm_sorted_view.argtypes = [P, P]
    lib.mm_sorted_view.restype = I
    lib.mm_assemble.argtypes = [P, I, I, P, I, P, P, P]
    lib.mm_assemble.restype = I
    lib.mm_ghost_add.argtypes = [P, I, I, P, P, I, I, P]
    lib.mm_slab_partition.restype = I
    lib.mm_slab_partition.argtypes = [P, I64, P, P, P, P, P, P, P, P]
    lib.mm_apply.restype = I
    lib.mm_apply.argtypes = [P, I, I, P, P, P, I, P]
    lib.mm_ghost_add.restype = I
    lib.mm_ghost_planes.argtypes = [I]
    lib.mm_ghost_planes.restype = I
    lib.mm_out_elems.argtypes = [P, I, I]
    lib.mm_out_elems.restype = I64
    lib.mm_deposit_moments.argtypes = [P, I, P, P, I, P, P, P]
    lib.mm_deposit_moments.restype = I
    lib.mm_gather_field.argtypes = [P, P, P, P]
    lib.mm_gather_field.restype = I
    lib.mm_assemble_slab.argtypes = [P, I, I, P, I, P, P, P, P]
    lib.mm_assemble_slab.restype = I
    lib.mm_ghost_exchange.argtypes = [P, P, I, I, I, P, P, P]
    lib.mm_ghost_exchange.restype = I
    lib.mm_comm_unique_id.argtypes = [P]
    lib.mm_comm_unique_id.restype = I
    lib.mm_comm_create.argtypes = [I, I, P, P]
    lib.mm_comm_create.restype = I
    lib.mm_comm_free.argtypes = [P]
    lib.mm_comm_free.restype = None
    lib.mm_free.argtypes = [P]
    lib.mm_free.restype = None
    lib.mm_last_error.restype = ctypes.c_char_p
    lib.mm_version.restype = ctypes.c_char_p
    lib.mm_launch_count.restype = I64
    _lib = lib
    return lib


def _check(st: int):
    if st != MM_OK:
        raise MMError(st, load_library().mm_last_error().decode())


def Grid(n, h=(1.0, 1.0, 1.0), x_begin=0, x_end=None) -> mm_grid:
    g = mm_grid()
    for i in range(3):
        g.n[i] = int(n[i])
        g.h[i] = float(h[i])
    g.x_begin = int(x_begin)
    g.x_end = int(n[0] if x_end is None else x_end)
    return g


def Species(qom=1.0, dt=1.0, c=1.0, sigma=1.0) -> mm_species:
    return mm_species(float(qom), float(dt), float(c), float(sigma))


def _stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _dev_ptr(t, dtype=torch.float64, name="tensor"):
    if t is None:
        return None
    if not (t.is_cuda and t.dtype == dtype and t.is_contiguous()):
        raise MMError(MM_ERR_INVALID_ARG, f"{name} must be a contiguous CUDA {dtype} tensor")
    return ctypes.c_void_p(t.data_ptr())


class Sorted:
    """Owner of an ``mm_sorted*`` handle (released by mm_free / garbage collection)."""

    def __init__(self, ptr, grid: mm_grid, order: int):
        self._ptr = ptr
        self.grid = grid
        self.order = order

    @property
    def ptr(self):
        return self._ptr

    def __del__(self):
        try:
            mm_free(self)
        except Exception:
            pass


def mm_sort_by_cell(grid: mm_grid, order: int, k_pad: int, pos, q, B=None, handle: Sorted | None = None,
                    stream=None, wait: bool = True) -> Sorted:
    """Stable support-window binning with K-padding (include/mm.h).  Reuses `handle` if given.
    FP32 pos (and B) select mm_sort_by_cell_mixed (PAPER.md:572 storage; q stays FP64).
    wait=False: mm_sort_by_cell_async (no host round trip; check with mm_sort_wait)."""
    lib = load_library()
    f32 = pos is not None and pos.dtype == torch.float32
    np_ = int(pos.shape[0]) if pos is not None else 0
    if pos is not None and tuple(pos.shape) != (np_, 3):
        raise MMError(MM_ERR_INVALID_ARG, "pos must be [np, 3]")
    if B is not None and tuple(B.shape) != (np_, 3):
        raise MMError(MM_ERR_INVALID_ARG, "B must be [np, 3]")
    if handle is not None and (handle.ptr is None or not handle.ptr.value):
        raise MMError(MM_ERR_INVALID_ARG, "handle was freed")
    hp = ctypes.c_void_p(handle.ptr.value if handle is not None else None)
    pdt = torch.float32 if f32 else torch.float64
    if not wait and f32:
        raise MMError(MM_ERR_INVALID_ARG, "the asynchronous sort takes FP64 positions")
    fn = lib.mm_sort_by_cell_mixed if f32 else (lib.mm_sort_by_cell if wait else lib.mm_sort_by_cell_async)
    st = fn(ctypes.byref(grid), int(order), int(k_pad), np_,
            _dev_ptr(pos, pdt, name="pos") if np_ else None, _dev_ptr(q, name="q") if np_ else None,
            _dev_ptr(B, pdt, name="B") if (B is not None and np_) else None, _stream_ptr(stream),
            ctypes.byref(hp))
    _check(st)
    if handle is not None:
        handle._ptr = hp  # the library may only grow buffers in place; keep the pointer it returned
        return handle
    return Sorted(hp, grid, order)


def mm_resort_by_cell(handle: Sorted, pos, q, B=None, stream=None, wait: bool = True) -> Sorted:
    """Incremental re-binning of the same particles after they moved (include/mm.h); FP64 inputs."""
    np_ = int(pos.shape[0])
    if tuple(pos.shape) != (np_, 3) or (B is not None and tuple(B.shape) != (np_, 3)):
        raise MMError(MM_ERR_INVALID_ARG, "pos / B must be [np, 3]")
    _check(load_library().mm_resort_by_cell(handle.ptr, np_, _dev_ptr(pos, name="pos") if np_ else None,
                                            _dev_ptr(q, name="q") if np_ else None,
                                            _dev_ptr(B, name="B") if (B is not None and np_) else None,
                                            _stream_ptr(stream), int(bool(wait))))
    return handle


def mm_sort_wait(handle: Sorted, stream=None):
    """Deferred status of the asynchronous sorts of `handle` (include/mm.h); raises MMError."""
    _check(load_library().mm_sort_wait(handle.ptr, _stream_ptr(stream)))


class _CudaArray:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr or 0), False),
                                         "version": 3, "strides": None}


def mm_sorted_view(handle: Sorted) -> dict:
    """Device tensors aliasing the handle's arrays (valid until the next sort/free)."""
    lib = load_library()
    info = mm_sorted_info()
    _check(lib.mm_sorted_view(handle.ptr, ctypes.byref(info)))
    dev = torch.device("cuda", torch.cuda.current_device())

    def view(ptr, n, typestr, shape=None):
        if n == 0:
            return torch.empty(shape or (0,), dtype=torch.int32 if typestr == "<i4" else torch.float64, device=dev)
        return torch.as_tensor(_CudaArray(ptr, shape or (n,), typestr), device=dev)

    m = info.np_padded
    return {"np": info.np, "np_padded": m, "nbins": info.nbins, "capacity": info.capacity, "order": info.order,
            "k_pad": info.k_pad, "has_B": bool(info.has_B),
            "perm": view(info.perm, m, "<i4"), "seg_begin": view(info.seg_begin, info.nbins + 1, "<i4"),
            "seg_count": view(info.seg_count, info.nbins, "<i4"),
            "rec": view(info.rec, m * info.rec_stride, "<f8", (m, info.rec_stride))}


def out_shape(grid: mm_grid, order: int, kind: int):
    S = (2 * order + 1) ** 3
    return ((grid.x_end - grid.x_begin) * grid.n[1] * grid.n[2], S, int(kind))


def ghost_shape(grid: mm_grid, order: int, kind: int):
    S = (2 * order + 1) ** 3
    return (load_library().mm_ghost_planes(order) * grid.n[1] * grid.n[2], S, int(kind))


def is_slab(grid: mm_grid) -> bool:
    return not (grid.x_begin == 0 and grid.x_end == grid.n[0])


def mm_assemble(handle: Sorted, kind: int, prec: int, species: mm_species, out, ghost=None,
                accumulate: bool = False, stream=None):
    """Assemble the mass matrix of one species into `out` (and `ghost` for slabs).

    `out`/`ghost` are float64 for MM_FP64 and float32 for MM_TF32 / MM_TF32X3."""
    lib = load_library()
    dt = torch.float64 if int(prec) == MM_FP64 else torch.float32
    st = lib.mm_assemble(handle.ptr, int(kind), int(prec), ctypes.byref(species), int(bool(accumulate)),
                         _dev_ptr(out, dt, name="out"), _dev_ptr(ghost, dt, name="ghost") if ghost is not None else None,
                         _stream_ptr(stream))
    _check(st)
    return out


def moments_shape(grid: mm_grid, nq: int):
    return ((grid.x_end - grid.x_begin) * grid.n[1] * grid.n[2], int(nq))


def moments_ghost_shape(grid: mm_grid, order: int, nq: int):
    return (load_library().mm_ghost_planes(order) * grid.n[1] * grid.n[2], int(nq))


def mm_deposit_moments(handle: Sorted, nq: int, species: mm_species, v, out, ghost=None, accumulate: bool = False,
                       stream=None):
    """rho, J (nq = 4) or the 10 implicit-moment quantities per node (include/mm.h); v in the
    particle order given to mm_sort_by_cell."""
    _check(load_library().mm_deposit_moments(handle.ptr, int(nq), ctypes.byref(species),
                                             _dev_ptr(v, name="v") if v is not None else None,
                                             int(bool(accumulate)), _dev_ptr(out, name="out"),
                                             _dev_ptr(ghost, name="ghost") if ghost is not None else None,
                                             _stream_ptr(stream)))
    return out


def mm_gather_field(handle: Sorted, F, Fp=None, stream=None):
    """F at the sorted particles -> the handle's B fields (and Fp in the caller's order)."""
    _check(load_library().mm_gather_field(handle.ptr, _dev_ptr(F, name="F"),
                                          _dev_ptr(Fp, name="Fp") if Fp is not None else None, _stream_ptr(stream)))
    return Fp


def mm_ghost_add(grid: mm_grid, order: int, kind: int, out, recv, first_plane: int, nplanes: int, stream=None):
    lib = load_library()
    _check(lib.mm_ghost_add(ctypes.byref(grid), int(order), int(kind), _dev_ptr(out, name="out"),
                            _dev_ptr(recv, name="recv"), int(first_plane), int(nplanes), _stream_ptr(stream)))


def mm_apply(grid: mm_grid, order: int, kind: int, M, E, y, accumulate: bool = False, stream=None):
    """y (+)= M E on the device (eq_field_eq); see include/mm.h."""
    lib = load_library()
    _check(lib.mm_apply(ctypes.byref(grid), int(order), int(kind), _dev_ptr(M, name="M"), _dev_ptr(E, name="E"),
                        _dev_ptr(y, name="y"), int(bool(accumulate)), _stream_ptr(stream)))


def mm_slab_partition(grid: mm_grid, pos, q, B=None, stream=None):
    """Stable partition of a rank's particles into (stay, to r-1, to r+1) by their slab
    (include/mm.h).  Returns (pos_out, q_out, B_out, counts) with the classes concatenated."""
    lib = load_library()
    np_ = int(pos.shape[0])
    pos_o, q_o = torch.empty_like(pos), torch.empty_like(q)
    B_o = torch.empty_like(B) if B is not None else None
    counts = (ctypes.c_int64 * 3)()
    _check(lib.mm_slab_partition(ctypes.byref(grid), np_, _dev_ptr(pos, name="pos"), _dev_ptr(q, name="q"),
                                 _dev_ptr(B, name="B") if B is not None else None, _dev_ptr(pos_o, name="pos_out"),
                                 _dev_ptr(q_o, name="q_out"), _dev_ptr(B_o, name="B_out") if B is not None else None,
                                 counts, _stream_ptr(stream)))
    return pos_o, q_o, B_o, (int(counts[0]), int(counts[1]), int(counts[2]))


def mm_free(handle: Sorted):
    if handle is not None and handle._ptr is not None and handle._ptr.value:
        load_library().mm_free(handle._ptr)
        handle._ptr = None


def version() -> str:
    return load_library().mm_version().decode()


def launch_count() -> int:
    return int(load_library().mm_launch_count())


def assemble(grid: mm_grid, order: int, kind: int, pos, q, B=None, species: mm_species | None = None,
             k_pad: int = 4, out=None, handle: Sorted | None = None, stream=None):
    """Convenience: sort + assemble on the device; returns (out, handle)."""
    species = species or Species()
    h = mm_sort_by_cell(grid, order, k_pad, pos, q, B if kind == MM_TENSOR else B, handle=handle, stream=stream)
    if out is None:
        out = torch.empty(out_shape(grid, order, kind), dtype=torch.float64, device=pos.device)
    ghost = None
    if is_slab(grid):
        ghost = torch.empty(ghost_shape(grid, order, kind), dtype=torch.float64, device=pos.device)
    mm_assemble(h, kind, MM_FP64, species, out, ghost, stream=stream)
    return (out, h) if ghost is None else (out, h, ghost)


# ----------------------------------------------------------------- multi-GPU (include/mm.h)
class Comm:
    """Owner of an ``mm_comm*`` (NCCL communicator + comm stream), released by mm_comm_free."""

    def __init__(self, ptr, nranks: int, rank: int):
        self._ptr = ptr
        self.nranks = nranks
        self.rank = rank

    @property
    def ptr(self):
        return self._ptr

    def __del__(self):
        try:
            mm_comm_free(self)
        except Exception:
            pass


def mm_comm_unique_id() -> bytes:
    """ncclGetUniqueId (128 bytes): call on one rank, broadcast to the others."""
    buf = ctypes.create_string_buffer(128)
    _check(load_library().mm_comm_unique_id(buf))
    return buf.raw


def mm_comm_create(nranks: int, rank: int, uid: bytes) -> Comm:
    """ncclCommInitRank on the current CUDA device (collective over the ranks)."""
    if len(uid) != 128:
        raise MMError(MM_ERR_INVALID_ARG, "uid must be 128 bytes")
    p = ctypes.c_void_p()
    _check(load_library().mm_comm_create(int(nranks), int(rank), ctypes.create_string_buffer(uid, 128),
                                         ctypes.byref(p)))
    return Comm(p, nranks, rank)


def mm_comm_free(comm: Comm):
    if comm is not None and comm._ptr is not None and comm._ptr.value:
        load_library().mm_comm_free(comm._ptr)
        comm._ptr = None


def comm_from_group(group=None) -> Comm:
    """Bootstrap an mm_comm over a torch.distributed process group: rank 0 draws the NCCL unique
    id, broadcast_object_list sends it to every rank, each rank calls mm_comm_create."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [mm_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return mm_comm_create(world, rank, obj[0])


def mm_ghost_exchange(comm: Comm, grid: mm_grid, order: int, kind: int, prec: int, out, ghost, stream=None):
    """Ghost-plane reduction over NCCL inside libmm (include/mm.h)."""
    dt = torch.float64 if int(prec) == MM_FP64 else torch.float32
    _check(load_library().mm_ghost_exchange(comm.ptr, ctypes.byref(grid), int(order), int(kind), int(prec),
                                            _dev_ptr(out, dt, name="out"), _dev_ptr(ghost, dt, name="ghost"),
                                            _stream_ptr(stream)))


def mm_assemble_slab(handle: Sorted, kind: int, prec: int, species: mm_species, out, ghost, comm: Comm,
                     accumulate: bool = False, stream=None):
    """Slab assembly + ghost reduction with the exchange overlapped (include/mm.h).  `ghost` is
    scratch of ghost_shape(grid, order, kind)."""
    dt = torch.float64 if int(prec) == MM_FP64 else torch.float32
    _check(load_library().mm_assemble_slab(handle.ptr, int(kind), int(prec), ctypes.byref(species),
                                           int(bool(accumulate)), _dev_ptr(out, dt, name="out"),
                                           _dev_ptr(ghost, dt, name="ghost"), comm.ptr, _stream_ptr(stream)))
    return out
