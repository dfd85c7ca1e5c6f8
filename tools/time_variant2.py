"""A/B of an alternative libmm build on the c2 assembly: times and an output checksum
(bit-identical builds print the same checksum).
    python tools/time_variant2.py <lib.so> [c2|c3]"""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2604_19286_b200 as mm  # noqa: E402
from paper_2604_19286_b200 import _build  # noqa: E402

_build.LIB = sys.argv[1]
name = sys.argv[2] if len(sys.argv) > 2 else "c2"
cfg = synth.config(name)
d = synth.particles(cfg)
dd = {k: torch.from_numpy(v).cuda() for k, v in d.items()}
g = mm.Grid(cfg.n)
h = mm.mm_sort_by_cell(g, cfg.order, 4, dd["pos"], dd["q"], dd["B"])
out = torch.empty(mm.out_shape(g, cfg.order, 9), dtype=torch.float64, device="cuda")
ts = []
for i in range(30):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    mm.mm_assemble(h, 9, mm.MM_FP64, mm.Species(), out)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts = sorted(ts[5:])
bits = out.view(torch.int64)
print(sys.argv[1], name, "median ms %.4f min %.4f" % (ts[len(ts) // 2], ts[0]),
      "checksum", int((bits * 1000003 % 1000000007).sum().item()))
