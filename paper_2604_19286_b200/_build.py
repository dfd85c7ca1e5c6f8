"""Build libmm.so (and the probe library) in-tree with nvcc for sm_100a.

    python -m paper_2604_19286_b200._build [--force] [--verbose]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libmm.so")
PROBE_LIB = os.path.join(HERE, "libmm_probe.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "-shared", "-cudart", "static",
         "-I", os.path.join(ROOT, "include"), "-ldl"]
LIB_SOURCES = ["mm_api.cu", "mm_sort.cu", "mm_assemble_fp64.cu", "mm_assemble_o1t.cu", "mm_assemble_tf32.cu", "mm_apply.cu", "mm_halo.cu", "mm_comm.cu", "mm_moments.cu", "mm_nodesum.cu"]
PROBE_SOURCES = ["mm_probe.cu"]
_lock = threading.Lock()


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    deps = sources + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "mm.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _nvcc(target, sources, verbose=False, extra=()):
    srcs = [os.path.join(CSRC, s) for s in sources]
    if not _stale(target, srcs):
        return target
    tmp = target + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, *FLAGS, *(["-Xptxas", "-v"] if verbose else []), *extra, "-o", tmp, *srcs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    if verbose:
        sys.stderr.write(r.stdout + r.stderr)
    os.replace(tmp, target)
    return target


def build(force: bool = False, verbose: bool = False) -> str:
    with _lock:
        if force:
            for t in (LIB, PROBE_LIB):
                if os.path.exists(t):
                    os.remove(t)
        _nvcc(LIB, LIB_SOURCES, verbose)
        if all(os.path.exists(os.path.join(CSRC, s)) for s in PROBE_SOURCES):
            _nvcc(PROBE_LIB, PROBE_SOURCES, verbose)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(LIB)
