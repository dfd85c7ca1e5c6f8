"""Sort timing beyond L2: c4 (134.7 M clustered particles, scalar handle) and the weak row's
32 x 256 x 256 slab (134.2 M, with B), sync and async entry points; MM_SORT_BKT_MIN selects
the path (bucketed scatter from that many particles on).
    python tools/time_sort_big.py [reps] [lib.so|-]"""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2604_19286_b200 as mm  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
if len(sys.argv) > 2 and sys.argv[2] != "-":
    from paper_2604_19286_b200 import _build
    _build.LIB = sys.argv[2]


def timed(fn, n):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


cfg = synth.config("c4o1")
d = synth.particles_device(cfg, "cuda", with_B=False)
g = mm.Grid(cfg.n)
st = {"h": None}
for order in (1, 2):
    st["h"] = None

    def s_sync():
        st["h"] = mm.mm_sort_by_cell(g, order, 4, d["pos"], d["q"], None, handle=st["h"])
    t = timed(s_sync, reps)
    print(f"c4 order {order}: sort {t:.3f} ms", flush=True)
    mm.mm_free(st["h"])
del d
torch.cuda.empty_cache()
cw = synth.Config("weak1", (32, 256, 256), 1, "tensor", 64, seed=19290)
dw = synth.particles_device(cw, "cuda")
gw = mm.Grid(cw.n, (1.0, 1.0, 1.0), 0, 32)
st["h"] = None


def w_sync():
    st["h"] = mm.mm_sort_by_cell(gw, 1, 4, dw["pos"], dw["q"], dw["B"], handle=st["h"])


def w_async():
    st["h"] = mm.mm_sort_by_cell(gw, 1, 4, dw["pos"], dw["q"], dw["B"], handle=st["h"], wait=False)


print(f"weak 32x256x256 o1: sort {timed(w_sync, reps):.3f} ms, async {timed(w_async, reps):.3f} ms", flush=True)
mm.mm_sort_wait(st["h"])
