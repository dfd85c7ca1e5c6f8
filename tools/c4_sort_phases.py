import sys, torch
sys.path.insert(0, ".")
import synth, paper_2604_19286_b200 as mm
cfg = synth.config("c4o1"); d = synth.particles_device(cfg, "cuda", with_B=False)
for order in (1, 2):
    g = mm.Grid(cfg.n); h = None
    for _ in range(3): h = mm.mm_sort_by_cell(g, order, 4, d["pos"], d["q"], None, handle=h)
    mm.mm_free(h)
