"""Per-phase cycle breakdown of the order-1 kernel (diagnostics build libmm_timers.so)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2604_19286_b200 as mm  # noqa: E402
from paper_2604_19286_b200 import _build  # noqa: E402

_build.LIB = "paper_2604_19286_b200/libmm_timers.so"
lib = mm.load_library(build_if_missing=False)
cfg = synth.config("c2")
d = synth.particles(cfg)
dd = {k: torch.from_numpy(v).cuda() for k, v in d.items()}
g = mm.Grid(cfg.n)
h = mm.mm_sort_by_cell(g, 1, 4, dd["pos"], dd["q"], dd["B"])
out = torch.empty(mm.out_shape(g, 1, 9), dtype=torch.float64, device="cuda")
buf = (ctypes.c_ulonglong * 4)()
mm.mm_assemble(h, 9, mm.MM_FP64, mm.Species(), out)
lib.mm_debug_phases(buf)
for _ in range(3):
    mm.mm_assemble(h, 9, mm.MM_FP64, mm.Species(), out)
lib.mm_debug_phases(buf)
tot = sum(buf)
print({n: round(100 * v / tot, 1) for n, v in zip(["tma_wait", "prep", "batches", "deposit+other"], buf)})
