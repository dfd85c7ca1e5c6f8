"""NEXT-4 timing on the c2 handle: mm_deposit_moments (nq 4, 10) and mm_gather_field.
    python tools/time_next4.py [lib.so|-]"""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2604_19286_b200 as mm  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] != "-":
    from paper_2604_19286_b200 import _build
    _build.LIB = sys.argv[1]
cfg = synth.config("c2")
d = synth.particles_device(cfg, "cuda")
g = mm.Grid(cfg.n)
h = mm.mm_sort_by_cell(g, 1, 4, d["pos"], d["q"], d["B"])
npart = d["q"].numel()
v = torch.rand(npart, 3, dtype=torch.float64, device="cuda")
F = torch.rand(64 ** 3, 3, dtype=torch.float64, device="cuda")
Fp = torch.empty(npart, 3, dtype=torch.float64, device="cuda")


def t(fn, n=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for nq in (4, 10):
    mo = torch.empty(mm.moments_shape(g, nq), dtype=torch.float64, device="cuda")
    print(f"moments nq {nq}: {t(lambda: mm.mm_deposit_moments(h, nq, mm.Species(), v, mo)):.4f} ms", flush=True)
print(f"gather: {t(lambda: mm.mm_gather_field(h, F, Fp)):.4f} ms", flush=True)
