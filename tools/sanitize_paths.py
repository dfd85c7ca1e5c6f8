"""One small invocation of every libmm kernel path, for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck).  No oracle, no timing: the sanitizer reports are the product.

    compute-sanitizer --tool racecheck python tools/sanitize_paths.py [c1|small]

c1: BASELINE.json configs[0] (4^3, 16 ppc); small: 12 x 10 x 9 grid, 40 ppc (several chunks per
bin, several bins per CTA / warp, slab grids with ghost planes).
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2604_19286_b200 as mm  # noqa: E402


def main(which="small"):
    torch.cuda.set_device(0)
    if which == "c1":
        n, ppc = (4, 4, 4), 16
    else:
        n, ppc = (12, 10, 9), 40
    sp = mm.Species()
    for order in ((1,) if which == "c1" else (1, 2)):  # c1 (4^3) admits order 1 only (n >= 2 order + 1)
        for slab in (False, True):
            xb, xe = (0, n[0]) if not slab else ((1, 3) if which == "c1" else (3, 3 + 2 * order + 2))
            cfg = synth.Config("san", n, order, "tensor", ppc, seed=7 + order)
            d = synth.particles(cfg, x_begin=xb, x_end=xe)
            dd = {k: torch.from_numpy(v).cuda() for k, v in d.items()}
            g = mm.Grid(n, (1.0, 1.0, 1.0), xb, xe)
            h = mm.mm_sort_by_cell(g, order, 4, dd["pos"], dd["q"], dd["B"])
            hs = mm.mm_sort_by_cell(g, order, 4, dd["pos"], dd["q"], None)
            ghost = None
            for kind, hh in ((mm.MM_TENSOR, h), (mm.MM_SCALAR, hs)):
                for prec in (mm.MM_FP64, mm.MM_TF32, mm.MM_TF32X3):
                    dt = torch.float64 if prec == mm.MM_FP64 else torch.float32
                    out = torch.empty(mm.out_shape(g, order, kind), dtype=dt, device="cuda")
                    if slab:
                        ghost = torch.empty(mm.ghost_shape(g, order, kind), dtype=dt, device="cuda")
                    try:
                        mm.mm_assemble(hh, kind, prec, sp, out, ghost)
                        mm.mm_assemble(hh, kind, prec, sp, out, ghost, accumulate=True)
                    except mm.MMError as e:  # documented incompatibilities (e.g. k_pad vs K tile)
                        print("skip", order, slab, kind, prec, e)
                    torch.cuda.synchronize()
            if not slab:
                M = torch.empty(mm.out_shape(g, order, 9), dtype=torch.float64, device="cuda")
                mm.mm_assemble(h, mm.MM_TENSOR, mm.MM_FP64, sp, M)
                E = torch.randn(n[0] * n[1] * n[2], 3, dtype=torch.float64, device="cuda")
                y = torch.empty_like(E)
                mm.mm_apply(g, order, 9, M, E, y)
            for nq in (4, 10):
                mo = torch.empty(mm.moments_shape(g, nq), dtype=torch.float64, device="cuda")
                mg = (torch.empty(mm.moments_ghost_shape(g, order, nq), dtype=torch.float64, device="cuda")
                      if slab else None)
                v = torch.randn(dd["pos"].shape[0], 3, dtype=torch.float64, device="cuda")
                mm.mm_deposit_moments(h, nq, sp, v, mo, mg)
            if not slab:
                F = torch.randn(n[0] * n[1] * n[2], 3, dtype=torch.float64, device="cuda")
                Fp = torch.empty(dd["pos"].shape[0], 3, dtype=torch.float64, device="cuda")
                mm.mm_gather_field(h, F, Fp)
            else:
                mm.mm_slab_partition(g, dd["pos"], dd["q"], dd["B"])
            torch.cuda.synchronize()
            # record-first sort (k_scatter0 / k_fixrec_*) and the two-phase deposit (k_nodesum)
            os.environ["MM_SORT_RECFIRST_MIN"] = "1"
            hr = mm.mm_sort_by_cell(g, order, 4, dd["pos"], dd["q"], dd["B"])
            hrs = mm.mm_sort_by_cell(g, order, 4, dd["pos"], dd["q"], None)
            os.environ["MM_TWO_PHASE"] = "7"
            for kind, hh in ((mm.MM_TENSOR, hr), (mm.MM_SCALAR, hrs)):
                for prec in (mm.MM_FP64, mm.MM_TF32):
                    dt = torch.float64 if prec == mm.MM_FP64 else torch.float32
                    out = torch.empty(mm.out_shape(g, order, kind), dtype=dt, device="cuda")
                    ghost = torch.empty(mm.ghost_shape(g, order, kind), dtype=dt, device="cuda") if slab else None
                    mm.mm_assemble(hh, kind, prec, sp, out, ghost)
                    torch.cuda.synchronize()
            os.environ.pop("MM_TWO_PHASE")
            if not slab:
                mm.mm_resort_by_cell(hr, dd["pos"], dd["q"], dd["B"])  # rebuilds the inverse permutation
            torch.cuda.synchronize()
            os.environ.pop("MM_SORT_RECFIRST_MIN")
            for x in (h, hs, hr, hrs):
                mm.mm_free(x)
    # record-first fix-up of a bin beyond the warp path (k_fixrec_cta) and beyond CTA_BIN_MAX
    # (k_fixrec_huge)
    os.environ["MM_SORT_RECFIRST_MIN"] = "1"
    for npart in (700, 17000):
        rng = np.random.default_rng(npart)
        pos = torch.from_numpy(np.array([2.0, 3.0, 1.0]) + rng.random((npart, 3)) * 0.999).cuda()
        q = torch.from_numpy(rng.uniform(0.5, 1.5, npart)).cuda()
        hb = mm.mm_sort_by_cell(mm.Grid((5, 5, 5)), 1, 4, pos, q, None)
        torch.cuda.synchronize()
        mm.mm_free(hb)
    os.environ.pop("MM_SORT_RECFIRST_MIN")
    print("sanitize paths done", which)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "small")
