"""Two-phase deposit vs the RED deposit for the TF32 order-2 assembly (diagnostics):
c3 (64^3 TSC tensor) and c4 (128^3 clustered, scalar, order 2).  Per-launch times and the
max |two-phase - RED| / max|RED| of the FP32 outputs.
    python tools/time_twophase.py [reps]"""
import os
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2604_19286_b200 as mm  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 8


def timed(fn, reps):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(round(e0.elapsed_time(e1), 3))
    return ts


cases = []
cfg = synth.config("c3")
d = synth.particles(cfg)
dd = {k: torch.from_numpy(v).cuda() for k, v in d.items()}
g3 = mm.Grid(cfg.n)
h3 = mm.mm_sort_by_cell(g3, 2, 4, dd["pos"], dd["q"], dd["B"])
cases.append(("c3", g3, h3, 2, 9))
del dd
cfg4 = synth.config("c4o1")
d4 = synth.particles_device(cfg4, "cuda", with_B=False)
g4 = mm.Grid(cfg4.n)
h4 = mm.mm_sort_by_cell(g4, 2, 4, d4["pos"], d4["q"], None)
cases.append(("c4o2", g4, h4, 2, 1))
if len(sys.argv) > 2:
    g2 = mm.Grid((64, 64, 64))
    c2 = synth.config("c2")
    d2 = {k: torch.from_numpy(v).cuda() for k, v in synth.particles(c2).items()}
    h2 = mm.mm_sort_by_cell(g2, 1, 4, d2["pos"], d2["q"], d2["B"])
    cases.append(("c2", g2, h2, 1, 9))
for name, g, h, order, kind in cases:
    for prec in (mm.MM_FP64, mm.MM_TF32, mm.MM_TF32X3):
        if prec == mm.MM_FP64 and order == 1:
            continue
        modes = ("0", "4", "12") if prec == mm.MM_FP64 else (("0", "2", "10") if order == 1 else ("0", "1", "9"))
        outs = {}
        for mode in modes:
            os.environ["MM_TWO_PHASE"] = mode
            dt = torch.float64 if prec == mm.MM_FP64 else torch.float32
            out = torch.empty(mm.out_shape(g, order, kind), dtype=dt, device="cuda")
            ts = timed(lambda: mm.mm_assemble(h, kind, prec, mm.Species(), out), reps)
            outs[mode] = out
            print(name, "prec", prec, "two_phase", mode, ts, flush=True)
        ref = outs["0"]
        for mode, o in outs.items():
            if mode in ("1", "2", "4"):
                err = ((o - ref).abs().max() / ref.abs().max()).item()
                print(name, "prec", prec, "mode", mode, "max rel diff vs RED", err, flush=True)
        del outs
os.environ["MM_TWO_PHASE"] = "1"
