"""Sort phases on the nearly-sorted c2 input (PIC regime; MM_SORT_TIMERS=1 prints them)."""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2604_19286_b200 as mm  # noqa: E402

for mode in ("nearly", True):
    cfg = synth.config("c2")
    d = synth.particles(cfg, shuffle=mode)
    dd = {k: torch.from_numpy(v).cuda() for k, v in d.items()}
    g = mm.Grid(cfg.n)
    h = None
    for _ in range(4):
        h = mm.mm_sort_by_cell(g, 1, 4, dd["pos"], dd["q"], dd["B"], handle=h)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        h = mm.mm_sort_by_cell(g, 1, 4, dd["pos"], dd["q"], dd["B"], handle=h)
    e1.record()
    torch.cuda.synchronize()
    print("input", mode, "sort ms", e0.elapsed_time(e1) / 10, file=sys.stderr)
    mm.mm_free(h)
