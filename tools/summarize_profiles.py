"""Summarise ncu captures brought back in gpurun_out/ into profiles/ (tracked).

    python tools/summarize_profiles.py --round r01 [--src gpurun_out]

Writes profiles/<round>_ncu_summary.md (per-kernel metrics and stall breakdown of the
full captures), profiles/<round>_launches.csv (+ a per-kernel share table from the
`--metrics gpu__time_duration.sum` launch list) and profiles/traffic.json (DRAM bytes
per launch of the assembly kernels, read by bench.py for roofline.traffic).
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import shutil
import subprocess

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe % active"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.sum", "DMMA instructions"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe % active"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("lts__t_requests_op_red.sum", "L2 RED requests"),
    ("lts__t_sectors_op_red.sum", "L2 RED sectors"),
    ("lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed", "L2 atomic input % active"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % active (tcgen05)"),
    ("sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.sum", "UTCHMMA TF32 ops"),
    ("sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
     "UTCHMMA TF32 % of peak"),
    ("smsp__sass_inst_executed_op_utcmma.sum", "tcgen05.mma instructions"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for i, h in enumerate(hdr):
            d[h] = (r[i], units[i])
        d["Kernel Name"] = r[hdr.index("Kernel Name")]
        res.append((d, hdr, r))
    return res


def stalls(hdr, r):
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                v = float(r[i])
            except ValueError:
                continue
            if v > 0.3:
                st.append((h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], v))
    return sorted(st, key=lambda x: -x[1])[:8]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--src", default="gpurun_out")
    ap.add_argument("--reps", nargs="*", default=["prof_c2", "prof_c3", "prof_tf32", "prof_c4o2", "prof_apply", "prof_sort", "prof_next4", "prof_recfirst", "prof_tp"])
    a = ap.parse_args()
    os.makedirs("profiles", exist_ok=True)
    lines = [f"# ncu summary ({a.round})", "",
             "Captured with `ncu --set full --clock-control none --import-source on` on one B200 "
             "(gpurun), kernels of `tools/gpu_round.sh` (bench.py / tools timing scripts on c2, c3, c4).  Values per launch.", ""]
    traffic = {}
    for rep in a.reps:
        path = os.path.join(a.src, rep + ".ncu-rep")
        if not os.path.exists(path):
            continue
        for d, hdr, r in raw(path):
            name = d["Kernel Name"]
            lines.append(f"## `{name[:110]}`")
            lines.append("")
            lines.append("| metric | value |")
            lines.append("|---|---|")
            for key, label in METRICS:
                if key in d:
                    v, u = d[key]
                    lines.append(f"| {label} (`{key}`) | {v} {u} |")
            lines.append(f"| top stalls (warps per issue) | {', '.join(f'{k} {v:.2f}' for k, v in stalls(hdr, r))} |")
            lines.append("")

            def to_bytes(key):
                v, u = d[key]
                v = float(v.replace(",", ""))
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            nm = name.replace("(int)", "").replace(" ", "")
            if ("k_asm_o1t" in nm or "k_asm_o1<9>" in nm) and "dram__bytes_read.sum" in d:
                traffic["assemble_o1_bytes_per_launch"] = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
            if ("k_asm_o2t" in nm or "k_asm_o2<9>" in nm) and "dram__bytes_read.sum" in d:
                traffic["assemble_o2_bytes_per_launch"] = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
    lc = os.path.join(a.src, "launches.csv")
    if os.path.exists(lc):
        shutil.copy(lc, os.path.join("profiles", f"{a.round}_launches.csv"))
        rows = list(csv.reader(open(lc)))
        hdr, data = None, []
        for r in rows:
            if r and r[0] == "ID":
                hdr = r
                continue
            if hdr and len(r) == len(hdr):
                data.append(dict(zip(hdr, r)))
        agg = collections.OrderedDict()
        for d in data:
            k = d["Kernel Name"].split("(")[0].replace("void ", "")[:60]
            agg.setdefault(k, []).append(float(d["Metric Value"].replace(",", "")))
        tot = sum(sum(v) for v in agg.values())
        lines += ["## Launch list (`--metrics gpu__time_duration.sum`, cold-cache, serialised)", "",
                  "| kernel | launches | mean us | share of listed time |", "|---|---|---|---|"]
        for k, v in agg.items():
            lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {100 * sum(v) / tot:.1f}% |")
        lines.append("")
    with open(os.path.join("profiles", f"{a.round}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if traffic:
        with open(os.path.join("profiles", "traffic.json"), "w") as f:
            json.dump(traffic, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
