#!/usr/bin/env python
"""Benchmark of the ECSIM mass-matrix assembly hot path on B200 (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (weak scaling over x-slabs)

A step = one pass of the whole hot path over one batch of synthetic particles
already resident in HBM: mm_sort_by_cell (locate, key, histogram, padded scan,
stable placement, record scatter) + mm_assemble (fused W/alpha, DMMA
contraction, node-stencil scatter) [at N>1: mm_assemble_slab, the ghost exchange
over libmm's NCCL communicator overlapped with the interior bins].
Workload at N=1: BASELINE config[1] "c2" (64^3, CIC, 64 ppc, random B, FP64
tensor); N>1: weak scaling, one 64^3 x-slab per GPU of a (64N)x64x64 grid.
The order-2 config c3 is measured the same way and reported under "order2";
the survey's weak row (32N)x256x256 (c5 at N=8, orders 1 and 2) under "weak_c5".

`--impl reference` times the oracle (plain FP64 CPU loop, oracle/) on the host
cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "assembly Mparticles/s, B-spline order 1&2, 1/2/4/8 B200; % tensor/HBM roofline"
UNIT = "Mparticles/s"
HBM_BYTES_PER_PARTICLE_IN = 56.0   # x,y,z,q,Bx,By,Bz (FP64) read once


def flops_per_particle(order, ncomp, kind="unique"):
    """FP64 FLOPs per particle:
    unique   F_unique = 2 x N(N+1)/2 x C, N = 8 | 27 support nodes (the stricter
             floor): the `roofline` figure
    plan     F_method = 2 x (MMA entries per component of the paper's tile plan: 64 | 640) x C
    pair     this build's pair-product contraction: 2 x (9 x 27 | 36 x 54) (tensor)
    executed DMMA FLOPs issued by the pair-product kernels incl. tile padding: 5 | 35 DMMA.8x8x4
             per batch of 4 particles (tensor; the order-1 kernel adds 3 SIMT FMAs per particle)"""
    n = 8 if order == 1 else 27
    if kind == "unique":
        return 2 * (n * (n + 1) // 2) * ncomp
    if kind == "plan":
        return 2 * (64 if order == 1 else 640) * ncomp
    if kind == "pair":
        return 2 * (9 * 27 if order == 1 else 36 * 54) * ncomp // 9
    if kind == "executed":
        if ncomp == 1:  # scalar kernels k_asm_pps: 2 | 5 DMMA per batch of 4
            return (2 if order == 1 else 5) * 512 // 4
        return (5 if order == 1 else 35) * 512 // 4
    raise ValueError(kind)


def alg_bytes_per_particle(order, ncomp, ppc):
    S = (2 * order + 1) ** 3
    return (HBM_BYTES_PER_PARTICLE_IN if ncomp == 9 else 32.0) + S * ncomp * 8.0 / ppc


def sort_path(np_):
    """Which sort pipeline libmm takes for np_ particles (include/mm.h)."""
    thr = int(os.environ.get("MM_SORT_RECFIRST_MIN", 48_000_000))
    return ("record-first (k_key, scan, k_scatter0, k_fixrec)" if np_ >= thr
            else "classic (k_key, scan, k_place, k_fix, k_scatter)")


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "MEASURED_PEAKS.json"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "B200_PROFILING.md fallback"


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: an NVML polling thread
    (every 2 ms, so that even a region of a few tens of ms gets samples), nvidia-smi -lms 50 as
    the fallback when NVML is unavailable."""

    # NVML clocks-event reason bits (nvml.h): 0x8 hw_slowdown, 0x20 sw_thermal, 0x40 hw_thermal,
    # 0x4 sw_power_cap
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, index):
        self.index = index
        self.sm, self.reasons, self.mx = [], set(), None
        self.stop = threading.Event()
        self.nvml = None
        self.smi = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.hnd = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(self.hnd, pynvml.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception:
            self.nvml = None
            self._start_smi()
        return self

    def _poll(self):
        p = self.nvml
        while not self.stop.is_set():
            try:
                self.sm.append(float(p.nvmlDeviceGetClockInfo(self.hnd, p.NVML_CLOCK_SM)))
                r = p.nvmlDeviceGetCurrentClocksEventReasons(self.hnd)
                for bit, nm in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(nm)
            except Exception:
                pass
            time.sleep(0.002)

    def _start_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.smi = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                         "--format=csv,noheader,nounits", "-lms", "50"],
                                        stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            first = threading.Event()

            def rd():
                names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
                for ln in self.smi.stdout:
                    f = [x.strip() for x in ln.split(",")]
                    first.set()
                    if len(f) < 6 or self.stop.is_set():
                        continue
                    try:
                        self.sm.append(float(f[0]))
                        self.mx = float(f[1])
                    except ValueError:
                        continue
                    for nm, v in zip(names, f[2:6]):
                        if v.lower() == "active":
                            self.reasons.add(nm)

            threading.Thread(target=rd, daemon=True).start()
            first.wait(timeout=10.0)  # nvidia-smi starts slowly: the region begins once it reports
            self.sm.clear()
        except Exception:
            self.smi = None

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(timeout=1)
        if self.smi:
            self.smi.terminate()
            try:
                self.smi.wait(timeout=2)
            except Exception:
                self.smi.kill()

    def summary(self):
        src = "nvml" if self.nvml is not None else "nvidia-smi"
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.mx, "reasons": [], "samples": 0, "source": src}
        return {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": self.mx, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": src}


def _oracle_cost(cfg, d, omp=False):
    """(fixed seconds per call, seconds per particle) of the oracle on this workload: two short
    calls of 20k and 100k particles (the fixed part is the whole-grid output zeroing)."""
    import oracle
    kind = cfg.ncomp
    ts = []
    for m in (20000, 100000) if not omp else (100000, 500000):
        m = min(m, len(d["q"]))
        t0 = time.perf_counter()
        _oracle_call(cfg, d, slice(0, m), omp)
        ts.append((m, time.perf_counter() - t0))
    (m1, t1), (m2, t2) = ts
    b = max((t2 - t1) / max(m2 - m1, 1), 1e-10)
    return max(t1 - b * m1, 0.0), b


def _oracle_call(cfg, d, sl, omp):
    """One oracle assembly of the particles d[sl] into the whole grid; returns the threads used."""
    import oracle
    kind = cfg.ncomp
    B = d["B"][sl] if kind == 9 else None
    if omp:
        return oracle.assemble_omp(cfg.n, cfg.order, kind, d["pos"][sl], d["q"][sl], B)[1]
    oracle.assemble(cfg.n, cfg.order, kind, d["pos"][sl], d["q"][sl], B)
    return 1


def oracle_rate(cfg, d, budget_s=10.0):
    """The oracle (plain FP64 C loop, oracle/) on a bounded sample (~budget_s each) of the workload:
    on all host cores (or_assemble_omp, x-slab colouring) and single-threaded (or_assemble)."""
    res = {}
    for omp in (True, False):
        a, b = _oracle_cost(cfg, d, omp)
        m = int(min(len(d["q"]), max(20000, (budget_s - a) / b)))
        t0 = time.perf_counter()
        th = _oracle_call(cfg, d, slice(0, m), omp)
        t = time.perf_counter() - t0
        res[omp] = (m / t / 1e6, th, m, t)
    v, th, m, t = res[True]
    v1, _, m1, t1 = res[False]
    return {"value": v, "unit": UNIT, "cores": th, "kind": "oracle",
            "sample": f"first {m} of {len(d['q'])} particles of {cfg.name} (input order) into the whole "
                      f"{'x'.join(map(str, cfg.n))} grid, {t:.1f} s on {th} threads (or_assemble_omp: the oracle's "
                      f"loop over x-slabs of one colour in parallel; host has {os.cpu_count()} cores)",
            "single_core": {"value": v1, "unit": UNIT, "cores": 1,
                            "sample": f"first {m1} particles, {t1:.1f} s, or_assemble"}}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = synth.config("c2")
    d = synth.particles(cfg)
    # bounded sample per step so that the whole --steps/--warmup run takes ~150 s of host time,
    # the oracle on all host cores (or_assemble_omp)
    a, b = _oracle_cost(cfg, d, omp=True)
    per_step = 150.0 / max(args.steps + args.warmup, 1)
    m = int(min(len(d["q"]) // 2, max(2000, (per_step - a) / b)))
    steps = []
    th = 1
    for _ in range(args.warmup):
        _oracle_call(cfg, d, slice(0, m), True)
    for k in range(args.steps):
        t0 = time.perf_counter()
        off = (k * m) % (len(d["q"]) - m)
        th = _oracle_call(cfg, d, slice(off, off + m), True)
        steps.append(time.perf_counter() - t0)
    t = float(np.sum(steps))
    val = m * args.steps / t / 1e6
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": "c2: 64^3 periodic grid, CIC (order 1), 64 ppc, random B, FP64 tensor mass matrix",
                       "sample_particles_per_step": m},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": th, "kind": "oracle",
                             "sample": f"{m} particles per step of c2 (consecutive slices of the shuffled input), "
                                       f"whole-grid output, or_assemble_omp on {th} threads "
                                       f"(host has {os.cpu_count()} cores)"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-order2", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-tf32", action="store_true")
    ap.add_argument("--pipeline", action="store_true")
    ap.add_argument("--no-c4", action="store_true")
    ap.add_argument("--no-weak", action="store_true")
    ap.add_argument("--sync-sort", action="store_true",
                    help="step with the synchronous mm_sort_by_cell (host round trip) instead of the async sort")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_2604_19286_b200 as mm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    mm.load_library(build_if_missing=False)
    peaks, peak_src = load_peaks()
    # libmm's own NCCL communicator (ghost exchange inside mm_assemble_slab), bootstrapped over the
    # torch process group; one rank: the self ring (used by the c5 weak-scaling row at N = 1)
    # (NCCL prints its version banner on stdout at communicator creation: fd 1 -> fd 2 meanwhile,
    # so that stdout carries only the JSON line)
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        comm = mm.comm_from_group() if world > 1 else mm.mm_comm_create(1, 0, mm.mm_comm_unique_id())
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    cache = {}

    def setup(name, order_kind=True):
        key = (name, order_kind)
        if key in cache:
            return cache[key]
        base = synth.config(name)
        if world == 1:
            cfg, xb, xe = base, 0, base.n[0]
        else:
            cfg = synth.Config(base.name + f"-weak{world}", (base.n[0] * world, base.n[1], base.n[2]), base.order,
                               base.kind, base.ppc, seed=base.seed)
            xb, xe = rank * base.n[0], (rank + 1) * base.n[0]
        d = synth.particles(cfg, xb, xe, shuffle=order_kind)
        grid = mm.Grid(cfg.n, cfg.h, xb, xe)
        dd = {k: torch.from_numpy(v).to(dev) for k, v in d.items()}
        cache.clear()  # keep one workload resident at a time (device memory)
        cache[key] = (cfg, grid, d, dd)
        return cache[key]

    def measure(name, with_extras, prec=None):
        prec = mm.MM_FP64 if prec is None else prec
        odt = torch.float64 if prec == mm.MM_FP64 else torch.float32
        cfg, grid, d, dd = setup(name)
        order, kind = cfg.order, cfg.ncomp
        sp = mm.Species(cfg.qom, cfg.dt, cfg.c, cfg.sigma)
        out = torch.empty(mm.out_shape(grid, order, kind), dtype=odt, device=dev)
        ghost = torch.empty(mm.ghost_shape(grid, order, kind), dtype=odt, device=dev) \
            if mm.is_slab(grid) else None
        state = {"h": None}
        ev = []

        def step(record=False):
            # mm_sort_by_cell_async: no host round trip between the sort and the assembly; the
            # deferred domain/finiteness status is checked with mm_sort_wait after the timed loop
            # (sticky over all steps)
            state["h"] = mm.mm_sort_by_cell(grid, order, 4, dd["pos"], dd["q"], dd["B"], handle=state["h"],
                                            wait=args.sync_sort)
            if record:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
            if world > 1:  # slab assembly with the ghost exchange overlapped, inside libmm
                mm.mm_assemble_slab(state["h"], kind, prec, sp, out, ghost, comm)
            else:
                mm.mm_assemble(state["h"], kind, prec, sp, out, ghost)
            if record:
                e1.record()
                ev.append((e0, e1))

        # Optional pipelined schedule (--pipeline, single GPU): the sort of batch k+1 runs on the
        # main stream while the assembly of batch k runs on a second stream (two handles).
        # Measured: no gain (the kernels contend for LSU/issue), so the default
        # step is the serial sort -> assemble.
        pipeline = world == 1 and args.pipeline
        s_main = torch.cuda.current_stream()
        s_asm = torch.cuda.Stream() if pipeline else s_main
        hs = [None, None]

        def run_pipelined(k_steps, record):
            hs[0] = mm.mm_sort_by_cell(grid, order, 4, dd["pos"], dd["q"], dd["B"], handle=hs[0], stream=s_main)
            ev_asm = []
            for k in range(k_steps):
                ev_sorted = torch.cuda.Event()
                ev_sorted.record(s_main)
                s_asm.wait_event(ev_sorted)
                if record:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(s_asm)
                mm.mm_assemble(hs[k % 2], kind, prec, sp, out, ghost, stream=s_asm)
                if record:
                    e1.record(s_asm)
                    ev.append((e0, e1))
                ea = torch.cuda.Event()
                ea.record(s_asm)
                ev_asm.append(ea)
                if k + 1 < k_steps:
                    if k >= 1:
                        s_main.wait_event(ev_asm[k - 1])  # the handle about to be re-sorted is free
                    hs[(k + 1) % 2] = mm.mm_sort_by_cell(grid, order, 4, dd["pos"], dd["q"], dd["B"],
                                                         handle=hs[(k + 1) % 2], stream=s_main)
            s_main.wait_event(ev_asm[-1])

        if pipeline:
            run_pipelined(args.warmup, False)
        else:
            for _ in range(args.warmup):
                step()
        barrier()
        l0 = mm.launch_count()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            barrier()
            t0.record()
            if pipeline:
                run_pipelined(args.steps, True)
            else:
                for _ in range(args.steps):
                    step(record=True)
            t1.record()
            barrier()
        state["h"] = hs[0] if pipeline else state["h"]
        launches = mm.launch_count() - l0
        mm.mm_sort_wait(state["h"])  # raises if any step met an invalid particle
        ms = t0.elapsed_time(t1)
        if world > 1:
            tt = torch.tensor([ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        asm_ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
        npart = len(d["q"])
        total = npart * world
        res = {"cfg": cfg, "ms_per_step": ms / args.steps, "assemble_ms": asm_ms, "np": npart, "pipelined": pipeline,
               "value": total * args.steps / (ms / 1e3) / 1e6, "launches": launches, "clocks": clk.summary()}
        # sort-only timing (same handle, same inputs)
        if with_extras:
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier()
            s0.record()
            for _ in range(max(5, args.steps // 10)):
                state["h"] = mm.mm_sort_by_cell(grid, order, 4, dd["pos"], dd["q"], dd["B"], handle=state["h"])
            s1.record()
            barrier()
            res["sort_ms"] = s0.elapsed_time(s1) / max(5, args.steps // 10)
            s0.record()
            for _ in range(max(5, args.steps // 10)):
                state["h"] = mm.mm_sort_by_cell(grid, order, 4, dd["pos"], dd["q"], dd["B"], handle=state["h"],
                                                wait=False)
            s1.record()
            barrier()
            mm.mm_sort_wait(state["h"])
            res["sort_async_ms"] = s0.elapsed_time(s1) / max(5, args.steps // 10)
            # assembly alone (no concurrent sort)
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier()
            a0.record()
            for _ in range(max(5, args.steps // 10)):
                if world > 1:
                    mm.mm_assemble_slab(state["h"], kind, prec, sp, out, ghost, comm)
                else:
                    mm.mm_assemble(state["h"], kind, prec, sp, out, ghost)
            a1.record()
            barrier()
            res["assemble_alone_ms"] = a0.elapsed_time(a1) / max(5, args.steps // 10)
            # the assembly kernel alone: accumulate=1 launches the same kernel into the filled
            # output without the zero-fill memset of accumulate=0 (same work, same REDs)
            if world == 1:
                barrier()
                a0.record()
                for _ in range(max(5, args.steps // 10)):
                    mm.mm_assemble(state["h"], kind, prec, sp, out, ghost, accumulate=True)
                a1.record()
                barrier()
                res["kernel_ms"] = a0.elapsed_time(a1) / max(5, args.steps // 10)
            # operator apply y = M E on the assembled matrix (NEXT-3, eq_field_eq), whole domain only
            if not mm.is_slab(grid):
                nrows = out.shape[0]
                Ef = torch.rand((nrows, 3), dtype=torch.float64, device=dev, generator=None)
                yf = torch.empty_like(Ef)
                for _ in range(3):
                    mm.mm_apply(grid, order, kind, out, Ef, yf)
                p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                nap = max(10, args.steps // 5)
                barrier()
                p0.record()
                for _ in range(nap):
                    mm.mm_apply(grid, order, kind, out, Ef, yf)
                p1.record()
                barrier()
                t_ap = p0.elapsed_time(p1) / nap
                byts = nrows * (out[0].numel() * 8 + 48)
                res["apply"] = {"ms": t_ap, "bytes_per_node": out[0].numel() * 8 + 48,
                                "roofline": {"bound": "hbm", "achieved": byts / (t_ap / 1e3) / 1e9,
                                             "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                                             "frac": byts / (t_ap / 1e3) / 1e9 / peaks.get("hbm_gbs", 6535.1)}}
                del Ef, yf
        res["d"] = d
        res["grid"], res["out"], res["ghost"], res["sp"], res["state"] = grid, out, ghost, sp, state
        return res

    # sort cost when the input is nearly sorted (the PIC-step regime; a random 10% of the particles permuted)
    sort_nearly_ms = None
    if world == 1:
        cfgn, gridn, dn, ddn = setup("c2", "nearly")
        hn = None
        for _ in range(3):
            hn = mm.mm_sort_by_cell(gridn, 1, 4, ddn["pos"], ddn["q"], ddn["B"], handle=hn)
        barrier()
        n0, n1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n0.record()
        for _ in range(20):
            hn = mm.mm_sort_by_cell(gridn, 1, 4, ddn["pos"], ddn["q"], ddn["B"], handle=hn)
        n1.record()
        barrier()
        sort_nearly_ms = n0.elapsed_time(n1) / 20
        mm.mm_free(hn)
        del hn, dn, ddn
    # NEXT-1: incremental re-binning (mm_resort_by_cell) of the c2 particles when a random 7% of
    # them move to a neighbouring cell per step (two position sets alternated), vs the full sort
    resort = None
    if world == 1:
        cfgr, gridr, dr, ddr = setup("c2")
        gen = torch.Generator(device=dev).manual_seed(5)
        Lr = torch.tensor(cfgr.n, dtype=torch.float64, device=dev)
        npr = ddr["q"].shape[0]
        sel = (torch.rand(npr, device=dev, generator=gen) < 0.10)[:, None]
        hop = torch.where(torch.rand(npr, 3, device=dev, generator=gen) < 0.5, -1.0, 1.0)
        hop = hop * (torch.rand(npr, 3, device=dev, generator=gen) < 0.34)
        moved = torch.remainder(ddr["pos"] + sel * hop, Lr)
        moved = torch.where(moved >= Lr, torch.zeros_like(moved), moved)
        nmov = int(((torch.floor(moved) != torch.floor(ddr["pos"])).any(dim=1)).sum().item())
        hr = mm.mm_sort_by_cell(gridr, 1, 4, ddr["pos"], ddr["q"], ddr["B"])
        sets = [moved, ddr["pos"]]
        for k in range(4):
            mm.mm_resort_by_cell(hr, sets[k % 2], ddr["q"], ddr["B"], wait=False)
        nrs = max(10, args.steps // 10)
        barrier()
        n0.record()
        for k in range(nrs):
            mm.mm_resort_by_cell(hr, sets[k % 2], ddr["q"], ddr["B"], wait=False)
        n1.record()
        barrier()
        mm.mm_sort_wait(hr)
        t_inc = n0.elapsed_time(n1) / nrs
        n0.record()
        for k in range(nrs):
            hr = mm.mm_sort_by_cell(gridr, 1, 4, sets[k % 2], ddr["q"], ddr["B"], handle=hr, wait=False)
        n1.record()
        barrier()
        mm.mm_sort_wait(hr)
        t_full = n0.elapsed_time(n1) / nrs
        resort = {"workload": "c2, a random 7% of the particles moved to a neighbouring cell per step",
                  "moved_particles": nmov, "incremental_ms": t_inc, "full_async_sort_ms": t_full}
        mm.mm_free(hr)
        del moved, sets, hop, sel
    r1 = measure("c2", True)
    cfg = r1["cfg"]
    ppc = synth.ppc_of(cfg)
    F = flops_per_particle(1, 9)
    # dominant kernel: mm_assemble (zero-fill + DMMA assembly kernel), events on the launch stream
    fp64_peak, fp64_src = None, None
    probe = os.path.join(ROOT, "profiles", "peaks_fp64.json")
    if os.path.exists(probe):
        with open(probe) as f:
            pk = json.load(f)
        fp64_peak, fp64_src = pk.get("dmma_tflops"), "profiles/peaks_fp64.json (DMMA.8x8x4 probe, measured)"
    if fp64_peak is None:
        fp64_peak = peaks.get("bf16_tflops", 1590.0) * 40.0 / 2250.0
        fp64_src = f"{peak_src} bf16 x nominal FP64/bf16 ratio 40/2250"
    achieved_zf = r1["np"] * F / (r1["assemble_ms"] / 1e3) / 1e12
    k1_ms = r1.get("kernel_ms") or r1["assemble_ms"]
    achieved = r1["np"] * F / (k1_ms / 1e3) / 1e12

    def flop_views(r, order):
        t = (r.get("kernel_ms") or r["assemble_ms"]) / 1e3
        v = {}
        for k in ("plan", "pair", "executed"):
            f = flops_per_particle(order, 9, k)
            v[k] = {"flops_per_particle": f, "tflops": r["np"] * f / t / 1e12, "frac": r["np"] * f / t / 1e12 / fp64_peak}
        return v

    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("assemble_o1_bytes_per_launch")
    roof = {"bound": "tensor", "kernel": "k_asm_o1t (pair-product FP64 DMMA; mm_assemble accumulate=1, CUDA "
                                         "events on the launch stream)",
            "kernel_ms": k1_ms,
            "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak,
            "incl_zero_fill": {"note": "mm_assemble(accumulate=0): memset of the 510 MB output + the kernel, "
                                       "as timed in the step", "ms": r1["assemble_ms"], "achieved": achieved_zf,
                               "frac": achieved_zf / fp64_peak},
            "traffic": traffic, "peak_source": fp64_src, "alg_flops_per_particle": F,
            "alg_flops_definition": "F_unique = 2 x 36 node pairs x 9 comps (SURVEY.md 8(d) stricter floor)",
            "other_flop_counts": flop_views(r1, 1),
            "alg_bytes_per_particle": alg_bytes_per_particle(1, 9, ppc),
            "hbm_achieved_gbs": r1["np"] * alg_bytes_per_particle(1, 9, ppc) / (k1_ms / 1e3) / 1e9,
            "hbm_peak_gbs": peaks.get("hbm_gbs")}

    line = {"metric": METRIC, "value": r1["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r1["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": ("c2: 64^3 periodic grid, CIC (order 1), 64 ppc, random B, FP64 tensor mass matrix"
                                    if world == 1 else
                                    f"weak scaling: ({64 * world})x64x64 grid, one 64^3 x-slab per GPU, CIC, 64 ppc"),
                       "grid": list(cfg.n), "order": 1, "kind": "tensor", "ppc": ppc, "particles": r1["np"] * world,
                       "parallelism": f"x-slab x{world}" if world > 1 else "single GPU",
                       "l2": "inputs (940 MB) and output (510 MB) larger than the 126 MB L2; no flush",
                       "k_pad": 4},
            "roofline": roof, "gpu_launches": r1["launches"], "clocks": r1["clocks"],
            "breakdown": {"pipelined": r1["pipelined"], "sort_alone_ms": r1.get("sort_ms"),
                          "assemble_alone_ms": r1.get("assemble_alone_ms"),
                          "serial_step_ms": (r1.get("sort_ms") or 0) + (r1.get("assemble_alone_ms") or 0),
                          "sort_ms": r1.get("sort_ms"), "sort_async_ms": r1.get("sort_async_ms"),
                          "sort_path": sort_path(r1["np"]),
                          "step_sort": "mm_sort_by_cell" if args.sync_sort else "mm_sort_by_cell_async + mm_sort_wait",
                          "assemble_ms": r1["assemble_ms"],
                          "sort_nearly_sorted_input_ms": sort_nearly_ms,
                          "resort": resort,
                          "sort_mps": r1["np"] / (r1["sort_ms"] / 1e3) / 1e6 if r1.get("sort_ms") else None,
                          # sort against the HBM roofline: algorithmic bytes = 24 B (positions, key
                          # pass) + 56 B (pos, q, B, record pass) read + 64 B record written
                          "sort_roofline": {"bound": "hbm", "alg_bytes_per_particle": 144.0,
                                            "achieved": r1["np"] * 144.0 / (r1["sort_ms"] / 1e3) / 1e9,
                                            "unit": "GB/s", "peak": peaks.get("hbm_gbs"),
                                            "frac": r1["np"] * 144.0 / (r1["sort_ms"] / 1e3) / 1e9 /
                                            peaks.get("hbm_gbs", 6535.1)} if r1.get("sort_ms") else None,
                          "assemble_mps": r1["np"] / (r1["assemble_ms"] / 1e3) / 1e6},
            "apply": r1.get("apply")}

    # ---- NEXT-4 on the c2 handle: moment deposition (rho, J: nq = 4; implicit-moment quantities:
    #      nq = 10) on FP64 DMMA tiles and the B-field gather, each against the HBM roofline on its
    #      algorithmic bytes: 32 B (xi, q of the record) + 4 B (perm) + 24 B (v, caller order) read
    #      + nq x 8 B per node written once (moments); 32 + 4 B read + 24 B written (B in the record)
    #      + 24 B (F_p, caller order) per particle (gather)
    if world == 1:
        h1, g1 = r1["state"]["h"], r1["grid"]
        npart = r1["np"]
        nnodes = cfg.n[0] * cfg.n[1] * cfg.n[2]
        vdev = torch.rand(npart, 3, dtype=torch.float64, device=dev) - 0.5
        nx4 = {}
        reps4 = max(10, args.steps // 10)

        def timed4(fn):
            for _ in range(3):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier()
            e0.record()
            for _ in range(reps4):
                fn()
            e1.record()
            barrier()
            return e0.elapsed_time(e1) / reps4

        for nq in (4, 10):
            mo = torch.empty(mm.moments_shape(g1, nq), dtype=torch.float64, device=dev)
            t = timed4(lambda: mm.mm_deposit_moments(h1, nq, mm.Species(), vdev, mo))
            byts = npart * 60.0 + nnodes * nq * 8.0
            nx4[f"moments_nq{nq}"] = {"ms": t, "mps": npart / (t / 1e3) / 1e6,
                                      "roofline": {"bound": "hbm", "achieved": byts / (t / 1e3) / 1e9,
                                                   "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                                                   "frac": byts / (t / 1e3) / 1e9 / peaks.get("hbm_gbs", 6535.1),
                                                   "alg_bytes_per_particle": 60.0 + nq * 8.0 / ppc}}
            del mo
        Fn = torch.rand(nnodes, 3, dtype=torch.float64, device=dev)
        Fp = torch.empty(npart, 3, dtype=torch.float64, device=dev)
        t = timed4(lambda: mm.mm_gather_field(h1, Fn, Fp))
        byts = npart * 84.0 + nnodes * 24.0
        nx4["gather"] = {"ms": t, "mps": npart / (t / 1e3) / 1e6,
                         "roofline": {"bound": "hbm", "achieved": byts / (t / 1e3) / 1e9,
                                      "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                                      "frac": byts / (t / 1e3) / 1e9 / peaks.get("hbm_gbs", 6535.1),
                                      "alg_bytes_per_particle": 84.0 + 24.0 / ppc}}
        del Fn, Fp, vdev
        line["next4"] = dict(workload="c2 handle (16.8 M particles, 64^3 CIC)", **nx4)

    if not args.no_order2:
        r2 = measure("c3", True)
        F2 = flops_per_particle(2, 9)
        a2z = r2["np"] * F2 / (r2["assemble_ms"] / 1e3) / 1e12
        k2_ms = r2.get("kernel_ms") or r2["assemble_ms"]
        a2 = r2["np"] * F2 / (k2_ms / 1e3) / 1e12
        line["order2"] = {"workload": "c3: 64^3, TSC (order 2), 64 ppc, random B, FP64 tensor" if world == 1 else
                          "c3 weak-scaled slabs", "value": r2["value"], "unit": UNIT, "ms_per_step": r2["ms_per_step"],
                          "sort_ms": r2.get("sort_ms"), "assemble_ms": r2["assemble_ms"],
                          "assemble_alone_ms": r2.get("assemble_alone_ms"), "pipelined": r2["pipelined"],
                          "apply": r2.get("apply"),
                          "roofline": {"bound": "tensor", "kernel": "k_asm_o2t (mm_assemble accumulate=1)",
                                       "kernel_ms": k2_ms,
                                       "achieved": a2, "peak": fp64_peak, "unit": "TFLOP/s",
                                       "frac": a2 / fp64_peak, "alg_flops_per_particle": F2,
                                       "incl_zero_fill": {"ms": r2["assemble_ms"], "achieved": a2z,
                                                          "frac": a2z / fp64_peak},
                                       "alg_flops_definition": "F_unique = 2 x 378 node pairs x 9 comps",
                                       "other_flop_counts": flop_views(r2, 2)}}
        del r2
    if world == 1 and not args.no_tf32:
        # TF32 / 3xTF32 variant on tcgen05 (FP32 output), reported separately (north_star)
        tf = {}
        for name, order in (("c2", 1), ("c3", 2)):
            for pname, prec in (("tf32", mm.MM_TF32), ("tf32x3", mm.MM_TF32X3)):
                r = measure(name, False, prec)
                tf[f"{name}_{pname}"] = {"value": r["value"], "unit": UNIT, "ms_per_step": r["ms_per_step"],
                                         "assemble_ms": r["assemble_ms"],
                                         "assemble_mps": r["np"] / (r["assemble_ms"] / 1e3) / 1e6,
                                         "hbm_achieved_gbs": r["np"] * (64 + (27 if order == 1 else 125) * 9 * 4 /
                                                                        synth.ppc_of(r["cfg"])) /
                                         (r["assemble_ms"] / 1e3) / 1e9}
                # HBM-bound variant: 64-B record read + FP32 output per particle
                tf[f"{name}_{pname}"]["roofline"] = {
                    "bound": "hbm", "achieved": tf[f"{name}_{pname}"]["hbm_achieved_gbs"],
                    "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                    "frac": tf[f"{name}_{pname}"]["hbm_achieved_gbs"] / peaks.get("hbm_gbs", 6535.1)}
                del r
        line["tf32"] = tf

    # ---- c2 with the production storage of PAPER.md:572 (NEXT-2): FP32 positions and B, FP64
    #      charges and mass matrix; sort + FP64 assembly per step
    if world == 1:
        cfg2 = synth.config("c2")
        d2 = synth.particles(cfg2)
        p32 = d2["pos"].astype(np.float32)
        L32 = np.array(cfg2.n, dtype=np.float32)
        p32 = np.where(p32 >= L32, p32 - L32, p32)  # FP32 rounding up to the box edge: periodic image
        dm = {"pos": torch.from_numpy(p32).to(dev),
              "q": torch.from_numpy(d2["q"]).to(dev),
              "B": torch.from_numpy(d2["B"].astype(np.float32)).to(dev)}
        gm = mm.Grid(cfg2.n)
        outm = torch.empty(mm.out_shape(gm, 1, 9), dtype=torch.float64, device=dev)
        stm = {"h": None}

        def step_m():
            stm["h"] = mm.mm_sort_by_cell(gm, 1, 4, dm["pos"], dm["q"], dm["B"], handle=stm["h"])
            mm.mm_assemble(stm["h"], 9, mm.MM_FP64, mm.Species(), outm)

        for _ in range(3):
            step_m()
        nm = max(10, args.steps // 10)
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        q0.record()
        for _ in range(nm):
            step_m()
        q1.record()
        barrier()
        tm = q0.elapsed_time(q1) / nm
        q0.record()
        for _ in range(nm):
            stm["h"] = mm.mm_sort_by_cell(gm, 1, 4, dm["pos"], dm["q"], dm["B"], handle=stm["h"])
        q1.record()
        barrier()
        line["mixed_inputs"] = {"workload": "c2 with FP32 positions and B, FP64 q and mass matrix (PAPER.md:572)",
                                "value": len(d2["q"]) / (tm / 1e3) / 1e6, "unit": UNIT, "ms_per_step": tm,
                                "sort_ms": q0.elapsed_time(q1) / nm, "input_bytes_per_particle": 32}
        mm.mm_free(stm["h"])
        del dm, outm, d2

    # ---- c4: 128^3 clustered (double-Harris-like) plasma, scalar (MPM-style) mass matrix, orders 1
    #      and 2 (+ TF32 for order 2); particles drawn on the device (same recipe)
    if world == 1 and not args.no_c4:
        cache.clear()
        torch.cuda.empty_cache()
        c4 = {}
        cfg4 = synth.config("c4o1")
        d4 = synth.particles_device(cfg4, dev, with_B=False)
        np4 = int(d4["q"].numel())
        ppc4 = synth.ppc_of(cfg4)
        sp4 = mm.Species()
        reps = max(5, min(20, args.steps // 10))

        def timed(fn, n):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier()
            e0.record()
            for _ in range(n):
                fn()
            e1.record()
            barrier()
            return e0.elapsed_time(e1) / n

        for name, order in (("c4o1", 1), ("c4o2", 2)):
            grid4 = mm.Grid(cfg4.n)
            st4 = {"h": None}
            out4 = torch.empty(mm.out_shape(grid4, order, 1), dtype=torch.float64, device=dev)

            def sort4():
                st4["h"] = mm.mm_sort_by_cell(grid4, order, 4, d4["pos"], d4["q"], None, handle=st4["h"],
                                              wait=args.sync_sort)

            def asm4(prec=mm.MM_FP64, o=out4):
                mm.mm_assemble(st4["h"], mm.MM_SCALAR, prec, sp4, o)

            for _ in range(3):
                sort4()
                asm4()
            with ClockSampler(local) as clk4:
                t_sort = timed(sort4, reps)
                t_asm = timed(asm4, reps)
            S = (2 * order + 1) ** 3
            F = flops_per_particle(order, 1)
            B = alg_bytes_per_particle(order, 1, ppc4)
            ent = {"workload": f"{name}: 128^3, clustered double-Harris-like ppc (mean {ppc4:.2f}), "
                               f"{'CIC' if order == 1 else 'TSC'}, scalar FP64 mass matrix",
                   "particles": np4, "value": np4 / ((t_sort + t_asm) / 1e3) / 1e6, "unit": UNIT,
                   "ms_per_step": t_sort + t_asm, "sort_ms": t_sort, "sort_path": sort_path(np4),
                   "assemble_ms": t_asm,
                   "assemble_mps": np4 / (t_asm / 1e3) / 1e6, "clocks": clk4.summary()}
            hbm = np4 * B / (t_asm / 1e3) / 1e9
            tfl = np4 * F / (t_asm / 1e3) / 1e12
            if order == 1:  # HBM-bound (35.4 B vs 128 FLOP per particle)
                ent["roofline"] = {"bound": "hbm", "achieved": hbm, "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                                   "frac": hbm / peaks.get("hbm_gbs", 6535.1), "alg_bytes_per_particle": B,
                                   "alg_bytes_definition": f"32 B (x, q) read + {S}x8 B output per node / ppc",
                                   "tensor_view": {"tflops": tfl, "frac": tfl / fp64_peak}}
            else:
                ent["roofline"] = {"bound": "tensor", "achieved": tfl, "peak": fp64_peak, "unit": "TFLOP/s",
                                   "frac": tfl / fp64_peak, "alg_flops_per_particle": F,
                                   "alg_flops_definition": "F_unique = 2 x 378 node pairs x 1 comp",
                                   "hbm_view": {"gbs": hbm, "frac": hbm / peaks.get("hbm_gbs", 6535.1)}}
                out4f = torch.empty(mm.out_shape(grid4, order, 1), dtype=torch.float32, device=dev)
                asm4(mm.MM_TF32, out4f)
                t_tf = timed(lambda: asm4(mm.MM_TF32, out4f), reps)
                Bf = 32.0 + S * 4.0 / ppc4
                ent["tf32"] = {"assemble_ms": t_tf, "assemble_mps": np4 / (t_tf / 1e3) / 1e6,
                               "roofline": {"bound": "hbm", "achieved": np4 * Bf / (t_tf / 1e3) / 1e9,
                                            "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                                            "frac": np4 * Bf / (t_tf / 1e3) / 1e9 / peaks.get("hbm_gbs", 6535.1),
                                            "alg_bytes_per_particle": Bf}}
                del out4f
            c4[name] = ent
            mm.mm_sort_wait(st4["h"])  # the deferred status of every timed sort
            mm.mm_free(st4["h"])
            del out4
            torch.cuda.empty_cache()
        line["c4"] = c4
        del d4
        torch.cuda.empty_cache()

    # ---- the survey's weak-scaling row: (32N) x 256 x 256, one 32 x 256 x 256
    #      x-slab (134.2 M particles, 64 ppc, random B) per GPU, FP64 tensor, orders 1 and 2; a step
    #      = mm_sort_by_cell + mm_assemble_slab (boundary bins, ghost exchange over libmm's NCCL
    #      communicator overlapped with the interior bins, ghost add).  N = 8 is config c5 (256^3).
    #      At N = 1 the communicator is the self ring (same code path, the slab is the whole grid).
    if not args.no_weak:
        cache.clear()
        torch.cuda.empty_cache()
        weak = {}
        per = 32
        cfgw = synth.Config(f"weak{world}", (per * world, 256, 256), 1, "tensor", 64, seed=synth.SEED0 + 4)
        xb, xe = rank * per, (rank + 1) * per
        dw = synth.particles_device(cfgw, dev, with_B=True, x_begin=xb, x_end=xe)
        npw = int(dw["q"].numel())
        for order in (1, 2):
            gw = mm.Grid(cfgw.n, x_begin=xb, x_end=xe)
            outw = torch.empty(mm.out_shape(gw, order, 9), dtype=torch.float64, device=dev)
            ghw = torch.empty(mm.ghost_shape(gw, order, 9), dtype=torch.float64, device=dev)
            stw = {"h": None}

            def sortw():
                stw["h"] = mm.mm_sort_by_cell(gw, order, 4, dw["pos"], dw["q"], dw["B"], handle=stw["h"],
                                              wait=args.sync_sort)

            def asmw():
                mm.mm_assemble_slab(stw["h"], 9, mm.MM_FP64, mm.Species(), outw, ghw, comm)

            kw = max(3, min(10, args.steps))
            for _ in range(3):
                sortw()
                asmw()
            barrier()
            ev_a = []
            w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with ClockSampler(local) as clkw:
                barrier()
                w0.record()
                for _ in range(kw):
                    sortw()
                    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a0.record()
                    asmw()
                    a1.record()
                    ev_a.append((a0, a1))
                w1.record()
                barrier()
            msw = w0.elapsed_time(w1) / kw
            asm_w = float(np.mean([a.elapsed_time(b) for a, b in ev_a]))
            if world > 1:
                tt = torch.tensor([msw, asm_w], device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                msw, asm_w = (float(x) for x in tt.tolist())
            Fw = flops_per_particle(order, 9)
            aw = npw * Fw / (asm_w / 1e3) / 1e12
            S = (2 * order + 1) ** 3
            weak[f"order{order}"] = {
                "value": npw * world / (msw / 1e3) / 1e6, "unit": UNIT, "ms_per_step": msw,
                "assemble_slab_ms": asm_w, "particles_per_gpu": npw, "particles": npw * world, "steps": kw,
                "exchanged_bytes_per_rank": (1 if order == 1 else 3) * 256 * 256 * S * 9 * 8,
                "output_bytes_per_gpu": outw.numel() * 8, "clocks": clkw.summary(),
                "roofline": {"bound": "tensor", "achieved": aw, "peak": fp64_peak, "unit": "TFLOP/s",
                             "frac": aw / fp64_peak, "alg_flops_per_particle": Fw,
                             "note": "mm_assemble_slab (zero-fill, boundary + interior bins, ghost exchange and "
                                     "add), max over ranks"}}
            mm.mm_sort_wait(stw["h"])
            mm.mm_free(stw["h"])
            del outw, ghw
            torch.cuda.empty_cache()
        line["weak_c5"] = {"workload": f"({per * world})x256x256 grid, one {per}x256x256 x-slab per GPU, 64 ppc, "
                                       "random B, FP64 tensor; particles drawn on the device (synth.particles_device)",
                           "n_gpus": world, "grid": list(cfgw.n), "scaling": "weak",
                           "exchange": "NCCL send/recv inside libmm (mm_assemble_slab), self ring at N = 1",
                           "sort_path": sort_path(int(np.prod(cfgw.n[1:])) * per * 64),
                           **weak}
        del dw
        torch.cuda.empty_cache()

    # ---- end to end through the public API with host buffers (pinned), H2D + D2H in the timed region
    if not args.no_e2e:
        import torch as T
        d = r1["d"]
        hp = {k: T.from_numpy(v).pin_memory() for k, v in d.items()}
        dd = {k: T.empty(v.shape, dtype=v.dtype, device=dev) for k, v in hp.items()}
        host_out = T.empty(r1["out"].shape, dtype=T.float64).pin_memory()
        grid, out, ghost, sp, state = r1["grid"], r1["out"], r1["ghost"], r1["sp"], r1["state"]
        ke = max(3, min(20, args.steps // 10))
        # Pipelined across steps (double-buffered device inputs, outputs and sort handles): the
        # H2D copy of step k+1 and the D2H copy of step k-1 run on their own streams (the two
        # copy engines, full duplex) while step k sorts and assembles.  Every step still moves
        # its whole input in and its whole matrix out.
        s_h2d, s_comp, s_d2h = T.cuda.Stream(), T.cuda.Stream(), T.cuda.Stream()
        dds = [dd, {k: T.empty_like(v) for k, v in dd.items()}]
        outs = [out, T.empty_like(out)]
        ghosts = [ghost, None if ghost is None else T.empty_like(ghost)]
        hs = [state["h"], None]
        ev_d2h = [None, None]

        def h2d(k):
            with T.cuda.stream(s_h2d):
                for key in ("pos", "q", "B"):
                    dds[k % 2][key].copy_(hp[key], non_blocking=True)
            ev = T.cuda.Event()
            ev.record(s_h2d)
            return ev

        def run_e2e(n):
            ev_in = h2d(0)
            for k in range(n):
                b = k % 2
                # dds[(k+1) % 2] is free: sort(k-1) has returned (it synchronises its stream)
                ev_next = h2d(k + 1) if k + 1 < n else None
                s_comp.wait_event(ev_in)
                if ev_d2h[b] is not None:
                    s_comp.wait_event(ev_d2h[b])  # outs[b] has been copied out (step k-2)
                with T.cuda.stream(s_comp):
                    hs[b] = mm.mm_sort_by_cell(grid, 1, 4, dds[b]["pos"], dds[b]["q"], dds[b]["B"], handle=hs[b],
                                               stream=s_comp)
                    if world > 1:
                        mm.mm_assemble_slab(hs[b], 9, mm.MM_FP64, sp, outs[b], ghosts[b], comm, stream=s_comp)
                    else:
                        mm.mm_assemble(hs[b], 9, mm.MM_FP64, sp, outs[b], ghosts[b], stream=s_comp)
                ev_c = T.cuda.Event()
                ev_c.record(s_comp)
                s_d2h.wait_event(ev_c)
                with T.cuda.stream(s_d2h):
                    host_out.copy_(outs[b], non_blocking=True)
                ev = T.cuda.Event()
                ev.record(s_d2h)
                ev_d2h[b] = ev
                ev_in = ev_next

        run_e2e(2)
        T.cuda.synchronize()
        barrier()
        e0, e1 = T.cuda.Event(enable_timing=True), T.cuda.Event(enable_timing=True)
        e0.record(s_h2d)
        run_e2e(ke)
        e1.record(s_d2h)
        T.cuda.synchronize()
        barrier()
        ems = e0.elapsed_time(e1)
        if world > 1:
            tt = T.tensor([ems], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        # the last step's matrix as read back on the host equals the device result (pipeline check)
        e2e_ok = bool(T.equal(host_out, outs[(ke - 1) % 2].cpu()))
        h2d_bytes = sum(v.numel() * v.element_size() for v in hp.values())
        line["e2e"] = {"value": r1["np"] * world * ke / (ems / 1e3) / 1e6, "unit": UNIT,
                       "h2d_bytes_per_step": h2d_bytes,
                       "d2h_bytes_per_step": host_out.numel() * 8, "steps": ke, "host_copy_matches_device": e2e_ok,
                       "note": "pinned host pos/q/B -> device, sort + assemble, full mass matrix -> pinned host; "
                               "pipelined across steps (H2D of k+1 and D2H of k-1 overlap step k)"}
        # the same end-to-end pipeline with the production storage of PAPER.md:572 (FP32 positions
        # and B, mm_sort_by_cell_mixed): half the H2D bytes of the inputs
        if world == 1 and "mixed_inputs" in line:
            p32 = d["pos"].astype(np.float32)
            L32 = np.array(cfg.n, dtype=np.float32)
            p32 = np.where(p32 >= L32, p32 - L32, p32)
            hp = {"pos": T.from_numpy(p32).pin_memory(), "q": hp["q"],
                  "B": T.from_numpy(d["B"].astype(np.float32)).pin_memory()}
            dds[0] = {k: T.empty(v.shape, dtype=v.dtype, device=dev) for k, v in hp.items()}
            dds[1] = {k: T.empty_like(v) for k, v in dds[0].items()}
            hs[0], hs[1] = None, None
            ev_d2h[0] = ev_d2h[1] = None
            run_e2e(2)
            T.cuda.synchronize()
            e0.record(s_h2d)
            run_e2e(ke)
            e1.record(s_d2h)
            T.cuda.synchronize()
            ems_m = e0.elapsed_time(e1)
            line["mixed_inputs"]["e2e"] = {"value": r1["np"] * ke / (ems_m / 1e3) / 1e6, "unit": UNIT,
                                           "h2d_bytes_per_step": sum(v.numel() * v.element_size() for v in hp.values()),
                                           "d2h_bytes_per_step": host_out.numel() * 8, "steps": ke}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = oracle_rate(cfg, r1["d"])
    if rank == 0:
        print(json.dumps(line), flush=True)
    mm.mm_comm_free(comm)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
