timeout 900 python -m pytest tests -m gpu -x -q -k "tf32 or TF32" 2>&1 | tail -2
for lib in paper_2604_19286_b200/libmm_prev.so paper_2604_19286_b200/libmm.so; do
for c in c2 c3; do
timeout 300 python - $lib $c <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2604_19286_b200 import _build
_build.LIB = sys.argv[1]
import synth, paper_2604_19286_b200 as mm
cfg = synth.config(sys.argv[2]); d = synth.particles_device(cfg, "cuda")
g = mm.Grid(cfg.n); h = mm.mm_sort_by_cell(g, cfg.order, 4, d["pos"], d["q"], d["B"])
for prec in (mm.MM_TF32, mm.MM_TF32X3):
    out = torch.empty(mm.out_shape(g, cfg.order, 9), dtype=torch.float32, device="cuda")
    for _ in range(3): mm.mm_assemble(h, 9, prec, mm.Species(), out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): mm.mm_assemble(h, 9, prec, mm.Species(), out)
    e1.record(); torch.cuda.synchronize()
    print(sys.argv[1].split('/')[-1], sys.argv[2], prec, round(e0.elapsed_time(e1)/20, 4), flush=True)
mm.mm_free(h); del d
cfg = synth.config("c4o1"); d = synth.particles_device(cfg, "cuda", with_B=False)
if sys.argv[2] == "c3":
    g = mm.Grid(cfg.n); h = mm.mm_sort_by_cell(g, 2, 4, d["pos"], d["q"], None)
    out = torch.empty(mm.out_shape(g, 2, 1), dtype=torch.float32, device="cuda")
    for _ in range(2): mm.mm_assemble(h, 1, mm.MM_TF32, mm.Species(), out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): mm.mm_assemble(h, 1, mm.MM_TF32, mm.Species(), out)
    e1.record(); torch.cuda.synchronize()
    print(sys.argv[1].split('/')[-1], "c4o2 tf32", round(e0.elapsed_time(e1)/5, 4), flush=True)
PY
done; done
