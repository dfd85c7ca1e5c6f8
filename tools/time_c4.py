"""c4 (128^3 clustered, scalar) sort / assembly timing per order (diagnostics).
    python tools/time_c4.py [order] [reps] [lib.so]"""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2604_19286_b200 as mm  # noqa: E402

if len(sys.argv) > 3:
    from paper_2604_19286_b200 import _build
    _build.LIB = sys.argv[3]
order = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = synth.config("c4o1")
d = synth.particles_device(cfg, "cuda", with_B=False)
g = mm.Grid(cfg.n)
h = mm.mm_sort_by_cell(g, order, 4, d["pos"], d["q"], None)
out = torch.empty(mm.out_shape(g, order, 1), dtype=torch.float64, device="cuda")
for prec, dt in ((mm.MM_FP64, torch.float64),):
    ts = []
    for i in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mm.mm_assemble(h, 1, prec, mm.Species(), out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(round(e0.elapsed_time(e1), 3))
    print("c4 order", order, prec, ts, flush=True)
