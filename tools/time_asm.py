"""Assembly timing (events around mm_assemble incl. its output zeroing) on a BASELINE config.
    python tools/time_asm.py [c2|c3] [reps] [lib.so] [prec 0|1|2]"""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2604_19286_b200 as mm  # noqa: E402

if len(sys.argv) > 3 and sys.argv[3] != "-":
    from paper_2604_19286_b200 import _build
    _build.LIB = sys.argv[3]
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
prec = int(sys.argv[4]) if len(sys.argv) > 4 else 0
cfg = synth.config(name)
d = synth.particles_device(cfg, "cuda")
g = mm.Grid(cfg.n)
h = mm.mm_sort_by_cell(g, cfg.order, 4, d["pos"], d["q"], d["B"])
out = torch.empty(mm.out_shape(g, cfg.order, 9), dtype=torch.float64 if prec == 0 else torch.float32, device="cuda")
ts = []
for i in range(reps + 3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    mm.mm_assemble(h, 9, prec, mm.Species(), out)
    e1.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"{name} prec {prec} assemble ms median {ts[len(ts) // 2]:.4f} min {ts[0]:.4f}", flush=True)
