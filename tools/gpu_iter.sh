timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -4 gpurun_out/pytest_gpu.log
timeout 300 python tools/time_sort.py c2 30
MM_SORT_TIMERS=1 timeout 300 python tools/time_sort.py c2 3 2>&1 | tail -2
timeout 300 python tools/time_sort.py c3 30
python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
import synth, paper_2604_19286_b200 as mm
cfg = synth.config("c4o1"); d = synth.particles_device(cfg, "cuda", with_B=False)
for order in (1, 2):
    g = mm.Grid(cfg.n); h = None
    for _ in range(3): h = mm.mm_sort_by_cell(g, order, 4, d["pos"], d["q"], None, handle=h)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): h = mm.mm_sort_by_cell(g, order, 4, d["pos"], d["q"], None, handle=h)
    e1.record(); torch.cuda.synchronize(); print("c4 sort order", order, e0.elapsed_time(e1) / 5)
    out = torch.empty(mm.out_shape(g, order, 1), dtype=torch.float32, device="cuda")
    for _ in range(2): mm.mm_assemble(h, 1, mm.MM_TF32, mm.Species(), out)
    e0.record()
    for _ in range(5): mm.mm_assemble(h, 1, mm.MM_TF32, mm.Species(), out)
    e1.record(); torch.cuda.synchronize(); print("c4 tf32 order", order, e0.elapsed_time(e1) / 5)
    mm.mm_free(h)
PY
