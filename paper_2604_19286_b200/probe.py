"""Microbenchmarks for the roofline denominators (run on the B200):

    python -m paper_2604_19286_b200.probe [--out profiles/peaks_fp64.json]

FP64 DMMA 8x8x4 and DFMA peaks (and whether they share a pipe), global FP64
RED throughput (random lines / random elements) and HBM copy bandwidth.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess

import torch

from . import _build


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(os.path.dirname(_build.HERE), "profiles", "peaks_fp64.json"))
    args = ap.parse_args()
    lib = ctypes.CDLL(_build.PROBE_LIB)
    F, P, I, I64 = ctypes.c_float, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    for nm, at in (("probe_batch", [I, I, P]), ("probe_dmma", [I, I, I, P]), ("probe_dfma", [I, I, I, P]), ("probe_mixed", [I, I, I, P]),
                   ("probe_red", [P, I64, I, I, I, I]), ("probe_copy", [P, P, I64]), ("probe_tf32", [I, I, P])):
        getattr(lib, nm).argtypes = at
        getattr(lib, nm).restype = F
    sink = torch.zeros(1024, dtype=torch.float64, device="cuda")
    sp = P(sink.data_ptr())
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    res = {"gpu": torch.cuda.get_device_name(0), "sms": sms}
    best = {}
    for blocks_per_sm, threads in ((4, 256), (8, 256), (2, 512), (16, 128)):
        b = sms * blocks_per_sm
        it = 2000
        ms = lib.probe_dmma(b, threads, it, sp)
        fl = b * threads / 32 * it * 8 * 512
        best["dmma"] = max(best.get("dmma", 0), fl / ms / 1e9)
        ms = lib.probe_dfma(b, threads, it, sp)
        fl = b * threads * it * 8 * 2
        best["dfma"] = max(best.get("dfma", 0), fl / ms / 1e9)
        ms = lib.probe_mixed(b, threads, it, sp)
        fl = b * threads / 32 * it * 8 * 512 + b * threads * it * 8 * 2
        best["mixed"] = max(best.get("mixed", 0), fl / ms / 1e9)
        best.setdefault("mixed_ms_vs_sum", [])
        ms_d = lib.probe_dmma(b, threads, it, sp)
        ms_f = lib.probe_dfma(b, threads, it, sp)
        best["mixed_ms_vs_sum"].append({"cfg": [blocks_per_sm, threads], "mixed_ms": ms, "dmma_ms": ms_d,
                                        "dfma_ms": ms_f})
    res["batch_loop"] = []
    for bps in (1, 2, 3, 4):
        b = sms * bps
        ms = lib.probe_batch(b, 500, sp)
        fl = b * 8 * 500 * 8 * 9 * 512
        res["batch_loop"].append({"ctas_per_sm": bps, "dmma_tflops": fl / ms / 1e9})
    # tcgen05 kind::tf32 (M 128, N 256, K 8) issued back to back by one thread per SM
    tf = []
    for iters in (2000, 8000):
        ms = lib.probe_tf32(sms, iters, sp)
        tf.append(sms * iters * 4 * 2 * 128 * 256 * 8 / ms / 1e9 if ms > 0 else None)
    res["tf32_tcgen05_tflops"] = max(t for t in tf if t) if any(tf) else None
    res["dmma_tflops"] = best["dmma"]
    res["dfma_tflops"] = best["dfma"]
    res["mixed_tflops"] = best["mixed"]
    res["mixed_detail"] = best["mixed_ms_vs_sum"]
    n = 510 * 1024 * 1024 // 8
    buf = torch.zeros(n, dtype=torch.float64, device="cuda")
    for contig in (1, 0):
        for blocks in (sms * 8, sms * 32):
            per = 64
            ms = lib.probe_red(P(buf.data_ptr()), n, blocks, 256, per, contig)
            reds = blocks * 256 * per
            res[f"red_{'line' if contig else 'rand'}_b{blocks}_gops"] = reds / ms / 1e6
    nb = 2 * 1024 ** 3 // 32
    a = torch.empty(nb * 4, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    ms = lib.probe_copy(P(a.data_ptr()), P(c.data_ptr()), nb)
    res["copy_gbs"] = 2 * nb * 32 / ms / 1e6
    try:
        res["clocks"] = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw",
                                        "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    except Exception:
        pass
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
