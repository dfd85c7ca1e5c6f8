"""c4 sort timing (events, per order) and phases with MM_SORT_TIMERS=1.
    python tools/c4_sort_phases.py [lib.so]"""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2604_19286_b200 as mm  # noqa: E402

if len(sys.argv) > 1:
    from paper_2604_19286_b200 import _build
    _build.LIB = sys.argv[1]
cfg = synth.config("c4o1")
d = synth.particles_device(cfg, "cuda", with_B=False)
for order in (1, 2):
    g = mm.Grid(cfg.n)
    h = None
    for _ in range(2):
        h = mm.mm_sort_by_cell(g, order, 4, d["pos"], d["q"], None, handle=h)
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h = mm.mm_sort_by_cell(g, order, 4, d["pos"], d["q"], None, handle=h)
        e1.record()
        torch.cuda.synchronize()
        ts.append(round(e0.elapsed_time(e1), 3))
    print("c4 sort order", order, "ms", ts, flush=True)
    mm.mm_free(h)
