"""Per-instruction hot spots of one kernel in an ncu report (diagnostics):
    python tools/ncu_hot.py <report.ncu-rep> [kernel-regex] [launch-index] [--top N] [--range lo hi]
Prints instructions executed / warp-stall samples per opcode and the top SASS lines."""
import argparse
import collections
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("kernel", nargs="?", default=None)
ap.add_argument("--launch", type=int, default=None)
ap.add_argument("--top", type=int, default=25)
ap.add_argument("--range", nargs=2, default=None)
a = ap.parse_args()
cmd = ["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"]
if a.kernel:
    cmd += ["-k", "regex:" + a.kernel]
if a.launch is not None:
    cmd += ["--launch-skip", str(a.launch), "--launch-count", "1"]
txt = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = next(r for r in rows if "Address" in r)
ia, isrc = h.index("Address"), h.index("Source")
ie, iss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")


def num(x):
    try:
        return int(x)
    except ValueError:
        return None


data, seen = [], set()
for r in rows[rows.index(h) + 1:]:
    if len(r) > ie and num(r[ie]) is not None and r[ia] not in seen:
        seen.add(r[ia])
        data.append((int(r[ia], 16), r[isrc].strip(), num(r[ie]), num(r[iss])))
base = data[0][0]
tot, ts = sum(d[2] for d in data), sum(d[3] for d in data)
print(f"instructions {tot}  stall samples {ts}")
agg, cnt = collections.Counter(), collections.Counter()
for _, s, e, ss in data:
    op = (s.split()[1] if s.startswith("@") else s.split()[0]).split(".")[0]
    agg[op] += ss
    cnt[op] += e
for op, v in agg.most_common(18):
    print(f"  {op:12s} samples {v:8d} ({100 * v / ts:5.1f}%)  executed {cnt[op]}")
if a.range:
    lo, hi = int(a.range[0], 16), int(a.range[1], 16)
    for ad, s, e, ss in data:
        if lo <= ad - base < hi:
            print(f"{ad - base:#07x} {e:12d} {ss:7d} {s[:80]}")
else:
    for ad, s, e, ss in sorted(data, key=lambda d: -d[3])[:a.top]:
        print(f"{ad - base:#07x} {e:12d} {ss:7d} {s[:80]}")
