"""Sort timing diagnostics: GPU time (events) and wall time per mm_sort_by_cell call.
    python tools/time_sort.py [c2|c3] [reps] [lib.so]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2604_19286_b200 as mm  # noqa: E402

if len(sys.argv) > 3:
    from paper_2604_19286_b200 import _build
    _build.LIB = sys.argv[3]
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = synth.config(name)
d = synth.particles(cfg)
dd = {k: torch.from_numpy(v).cuda() for k, v in d.items()}
g = mm.Grid(cfg.n)
h = None
for _ in range(3):
    h = mm.mm_sort_by_cell(g, cfg.order, 4, dd["pos"], dd["q"], dd["B"], handle=h)
torch.cuda.synchronize()
gpu, wall = [], []
for i in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    h = mm.mm_sort_by_cell(g, cfg.order, 4, dd["pos"], dd["q"], dd["B"], handle=h)
    e1.record()
    torch.cuda.synchronize()
    wall.append((time.perf_counter() - t0) * 1e3)
    gpu.append(e0.elapsed_time(e1))
gpu.sort()
wall.sort()
print(f"{name}: sort GPU ms median {gpu[len(gpu) // 2]:.3f} min {gpu[0]:.3f}; wall ms median {wall[len(wall) // 2]:.3f}")
