"""Per-launch timing of the assembly variants on one config (diagnostics)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2604_19286_b200 as mm  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = synth.config(name)
d = synth.particles(cfg)
dd = {k: torch.from_numpy(v).cuda() for k, v in d.items()}
g = mm.Grid(cfg.n)
h = mm.mm_sort_by_cell(g, cfg.order, 4, dd["pos"], dd["q"], dd["B"])
for prec, dt in ((mm.MM_FP64, torch.float64), (mm.MM_TF32, torch.float32), (mm.MM_TF32X3, torch.float32)):
    out = torch.empty(mm.out_shape(g, cfg.order, 9), dtype=dt, device="cuda")
    ts = []
    for i in range(12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mm.mm_assemble(h, 9, prec, mm.Species(), out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(round(e0.elapsed_time(e1), 3))
    print(name, prec, ts, flush=True)
