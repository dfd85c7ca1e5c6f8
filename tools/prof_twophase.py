"""One two-phase TF32 order-2 assembly on c3 (tensor) and on c4 (scalar) for ncu captures."""
import os
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2604_19286_b200 as mm  # noqa: E402

os.environ["MM_TWO_PHASE"] = sys.argv[1] if len(sys.argv) > 1 else "1"
prec = mm.MM_TF32 if os.environ["MM_TWO_PHASE"] != "4" else mm.MM_FP64
dt = torch.float32 if prec == mm.MM_TF32 else torch.float64
cfg = synth.config("c3")
dd = {k: torch.from_numpy(v).cuda() for k, v in synth.particles(cfg).items()}
g = mm.Grid(cfg.n)
h = mm.mm_sort_by_cell(g, 2, 4, dd["pos"], dd["q"], dd["B"])
out = torch.empty(mm.out_shape(g, 2, 9), dtype=dt, device="cuda")
mm.mm_assemble(h, 9, prec, mm.Species(), out)
torch.cuda.synchronize()
del dd, h, out
cfg4 = synth.config("c4o1")
d4 = synth.particles_device(cfg4, "cuda", with_B=False)
g4 = mm.Grid(cfg4.n)
h4 = mm.mm_sort_by_cell(g4, 2, 4, d4["pos"], d4["q"], None)
out4 = torch.empty(mm.out_shape(g4, 2, 1), dtype=dt, device="cuda")
mm.mm_assemble(h4, 1, prec, mm.Species(), out4)
torch.cuda.synchronize()
print("ok")
