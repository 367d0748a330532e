"""Summarise ncu reports / launch lists from gpurun_out/ into profiles/ (committed).

usage: python tools/summarize_ncu.py <report.ncu-rep> <out.txt> [kernel-regex]
       python tools/summarize_ncu.py --launches <launches.csv> <out.txt>
Also updates profiles/ncu_traffic.json (DRAM read+write bytes per launch of the
dominant kernels, read by bench.py for roofline.traffic).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes_read.sum.per_second", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
        "l1tex__m_xbar2l1tex_read_bytes.sum"]
UNIT_MB = {"dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "l1tex__m_xbar2l1tex_read_bytes.sum"}


def report(rep, out, rx=None):
    raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = []
    traffic = {}
    for row in rows[2:]:
        name = row[hdr.index("Kernel Name")]
        if rx and not re.search(rx, name):
            continue
        lines.append(f"== {name[:100]}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"   {k:70s} {row[i]:>16s} {units[i]}")
        st = [(hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", ""), row[i]) for i in range(len(hdr))
              if "pcsamp_warps_issue_stalled" in hdr[i] and not hdr[i].endswith("not_issued")]
        st = sorted([(a, float(b)) for a, b in st if b and float(b) > 0], key=lambda x: -x[1])[:8]
        lines.append("   top stall samples: " + ", ".join(f"{a}={int(b)}" for a, b in st))
        try:
            sc = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}
            rd = float(row[hdr.index("dram__bytes_read.sum")]) * sc.get(units[hdr.index("dram__bytes_read.sum")], 1e6)
            wr = float(row[hdr.index("dram__bytes_write.sum")]) * sc.get(units[hdr.index("dram__bytes_write.sum")], 1e6)
            key = "lmh" if "lmh_tc" in name else ("scan" if "sem_scan" in name else None)
            if key:
                traffic[key] = rd + wr   # bytes per launch (read + write)
        except (ValueError, IndexError):
            pass
    open(out, "w").write("\n".join(lines) + "\n")
    if traffic:
        tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        cur = json.load(open(tf)) if os.path.exists(tf) else {}
        cur.update(traffic)
        json.dump(cur, open(tf, "w"), indent=1)


def launches(csv_path, out):
    rows = list(csv.reader(open(csv_path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    idx = {h: j for j, h in enumerate(hdr)}
    agg = defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        agg[r[idx["Kernel Name"]][:70]].append(float(r[idx["Metric Value"]]) / 1e3)
    setup = [k for k in agg if "rownorm_max" in k]       # once per weight tensor, not per step
    steps = max(len(v) for k, v in agg.items() if k not in setup)
    tot = sum(sum(v) for k, v in agg.items() if k not in setup) / steps
    lines = ["kernel launches (ncu gpu__time_duration.sum, cold-cache, serialised): launches captured, mean us per",
             "launch, share of one step (setup kernels listed, excluded from the shares)",
             f"{'n':>4s} {'mean_us':>9s} {'share':>6s}  kernel"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        m = sum(v) / len(v)
        share = "setup" if k in setup else f"{sum(v) / steps / tot:6.1%}"
        lines.append(f"{len(v):4d} {m:9.1f} {share:>6s}  {k}")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        report(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
