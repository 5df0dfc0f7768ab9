"""Aggregate an ncu --csv launch list (gpu__time_duration.sum per launch) by
kernel: launches, total ms, share. Usage: python tools/launch_table.py launches.csv [skip_first_n]"""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
ids = hdr.index("ID")
per = []
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    unit = r[ui]
    ms = v / 1e6 if unit in ("nsecond", "ns") else (v / 1e3 if unit in ("usecond", "us") else v)
    per.append((int(r[ids]), re.sub(r"\(.*", "", r[ki]), ms))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
per = [p for p in per if p[0] >= skip]
agg = defaultdict(lambda: [0, 0.0])
for _, k, ms in per:
    agg[k][0] += 1
    agg[k][1] += ms
tot = sum(v[1] for v in agg.values())
print(f"{len(per)} launches, {tot:.3f} ms device time")
for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{ms:9.3f} ms {100 * ms / tot:5.1f}% {n:6d}  {k[:110]}")
