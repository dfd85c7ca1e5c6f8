"""Incremental re-binning vs a full sort on c2 (16.8 M particles): a PIC-like step moves a random
10% of the particles to a neighbouring cell (and jitters the rest inside their cells is NOT done:
only the movers change); shuffled and nearly-sorted caller orders.  GPU time per call."""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2604_19286_b200 as mm  # noqa: E402


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


cfg = synth.config("c2")
for order_name in ("shuffled", "nearly"):
    d = synth.particles(cfg, shuffle=True if order_name == "shuffled" else "nearly")
    dd = {k: torch.from_numpy(v).cuda() for k, v in d.items()}
    g = mm.Grid(cfg.n)
    gen = torch.Generator(device="cuda").manual_seed(5)
    L = torch.tensor(cfg.n, dtype=torch.float64, device="cuda")
    sel = torch.rand(dd["q"].shape[0], device="cuda", generator=gen) < 0.10
    step = torch.where(torch.rand(dd["pos"].shape, device="cuda", generator=gen) < 0.5, -1.0, 1.0)
    moved = dd["pos"] + sel[:, None] * step * (torch.rand(dd["pos"].shape, device="cuda", generator=gen) < 0.34)
    moved = torch.remainder(moved, L)
    moved = torch.where(moved >= L, torch.zeros_like(moved), moved)
    h = mm.mm_sort_by_cell(g, 1, 4, dd["pos"], dd["q"], dd["B"])
    st = {"h": h, "flip": 0}

    def full():
        st["h"] = mm.mm_sort_by_cell(g, 1, 4, moved, dd["q"], dd["B"], handle=st["h"], wait=False)

    def incr():
        # alternate between the two position sets: every call re-bins ~10% movers
        p = moved if st["flip"] == 0 else dd["pos"]
        st["flip"] ^= 1
        mm.mm_resort_by_cell(st["h"], p, dd["q"], dd["B"], wait=False)

    tf = timed(full)
    mm.mm_sort_wait(st["h"])
    st["h"] = mm.mm_sort_by_cell(g, 1, 4, dd["pos"], dd["q"], dd["B"], handle=st["h"])
    ti = timed(incr)
    mm.mm_sort_wait(st["h"])
    print(f"c2 {order_name}: full async sort {tf:.3f} ms, incremental {ti:.3f} ms", flush=True)
    mm.mm_free(st["h"])
