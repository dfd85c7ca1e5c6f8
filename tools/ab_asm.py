"""A/B timing of the FP64 assembly kernels (diagnostics):
    python tools/ab_asm.py c2 c3          # default kernels
    MM_ASM_LEGACY=1 python tools/ab_asm.py c2 c3
Prints per-config median ms of mm_assemble (zero-fill included) and a checksum."""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2604_19286_b200 as mm  # noqa: E402

for name in sys.argv[1:] or ["c2"]:
    cfg = synth.config(name)
    d = synth.particles(cfg)
    dd = {k: torch.from_numpy(v).cuda() for k, v in d.items()}
    g = mm.Grid(cfg.n)
    h = mm.mm_sort_by_cell(g, cfg.order, 4, dd["pos"], dd["q"], dd["B"])
    out = torch.empty(mm.out_shape(g, cfg.order, cfg.ncomp), dtype=torch.float64, device="cuda")
    ts = []
    for i in range(12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mm.mm_assemble(h, cfg.ncomp, mm.MM_FP64, mm.Species(), out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts = sorted(ts[2:])
    o = out.view(-1, cfg.ncomp)
    print(f"{name}: median {ts[len(ts)//2]:.4f} ms min {ts[0]:.4f} ms  sum/comp {o.sum(0)[:3].tolist()} "
          f"abs {out.abs().sum().item():.12e}", flush=True)
    mm.mm_free(h)
    del out, dd
