"""Per-source-line stall samples / instructions of one kernel in an ncu report.

usage: python tools/ncu_lines.py <report.ncu-rep> <kernel-regex> [top]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, rx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + rx,
                               "--print-source", "cuda,sass"], text=True)
agg = defaultdict(lambda: [0, 0, ""])
cur = "?"
for r in csv.reader(io.StringIO(raw)):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) < 8 or not r[0].isdigit():
        continue
    try:
        s, ie = int(r[4] or 0), int(r[7] or 0)
    except ValueError:
        continue
    a = agg[(cur, int(r[0]))]
    a[0] += s
    a[1] += ie
    a[2] = r[1][:100]
tot = sum(v[0] for v in agg.values()) or 1
for (f, ln), (s, ie, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100.0 * s / tot:5.1f}% {s:6d} {ie:9d}  {f}:{ln:<5d} {src.strip()}")
