"""CPU checks of the C ABI library: it builds, loads without a GPU, exports every symbol
include/mm.h declares, and rejects bad arguments before touching the device."""
import ctypes
import os
import re

import pytest

import paper_2604_19286_b200 as mm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "mm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mm_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = mm.load_library()
    syms = header_symbols()
    assert set(syms) == set(mm.EXPORTS)
    for s in syms:
        assert hasattr(lib, s), s


def test_version_and_geometry_helpers():
    lib = mm.load_library()
    assert "sm_100a" in mm.version()
    assert lib.mm_ghost_planes(1) == 1 and lib.mm_ghost_planes(2) == 3 and lib.mm_ghost_planes(3) == -1
    g = mm.Grid((4, 5, 6))
    assert lib.mm_out_elems(ctypes.byref(g), 1, 9) == 4 * 5 * 6 * 27 * 9
    assert lib.mm_out_elems(ctypes.byref(g), 2, 9) == -1           # n < 2*order+1
    g2 = mm.Grid((10, 5, 6), x_begin=2, x_end=7)
    assert lib.mm_out_elems(ctypes.byref(g2), 2, 1) == 5 * 5 * 6 * 125
    assert mm.out_shape(g2, 2, 1) == (5 * 5 * 6, 125, 1)


@pytest.mark.parametrize("n,order,xb,xe,k", [((4, 5, 5), 2, 0, 4, 4), ((5, 5, 5), 3, 0, 5, 4),
                                            ((5, 5, 5), 1, 3, 3, 4), ((5, 5, 5), 1, 0, 5, 6),
                                            ((8, 5, 5), 2, 2, 3, 4)])
def test_sort_rejects_bad_arguments_without_gpu(n, order, xb, xe, k):
    lib = mm.load_library()
    g = mm.Grid(n, x_begin=xb, x_end=xe)
    h = ctypes.c_void_p()
    st = lib.mm_sort_by_cell(ctypes.byref(g), order, k, 0, None, None, None, None, ctypes.byref(h))
    assert st == mm.MM_ERR_INVALID_ARG
    assert lib.mm_last_error()
    assert h.value is None


def test_assemble_rejects_null_handle():
    lib = mm.load_library()
    sp = mm.Species()
    st = lib.mm_assemble(None, 9, 0, ctypes.byref(sp), 0, None, None, None)
    assert st == mm.MM_ERR_INVALID_ARG
    lib.mm_free(None)


def test_sass_contains_dmma_and_red():
    """The assembly kernels are FP64 tensor-core (DMMA) kernels with FP64 global reductions."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run(["cuobjdump", "-sass", mm._build.LIB], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass
    assert "REDG.E.ADD.F64" in sass
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", mm._build.LIB], capture_output=True, text=True).stdout \
        or "sm_100" in sass
