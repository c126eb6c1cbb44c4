"""Summarise ncu captures for profiles/ (dev tool, runs here without a GPU).

python tools/ncu_summary.py launches gpurun_out/launches.csv            # per-kernel launch list summary
python tools/ncu_summary.py full gpurun_out/prof.ncu-rep [label]         # key --set full metrics + top stalls
"""

from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpc__cycles_elapsed.max",
    "sm__cycles_active.avg", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_issued.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__cycles_active.avg",
    "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__memory_throughput.avg.pct_of_peak_sustained_elapsed",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    d = collections.defaultdict(list)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            x = dict(zip(hdr, r))
            if x.get("Metric Name") == "gpu__time_duration.sum":
                name = x["Kernel Name"]
                short = name.split("(")[0][:80]
                d[short].append(float(x["Metric Value"]) / (1e3 if x["Metric Unit"] == "ns" else 1.0))
    tot = sum(sum(v) for v in d.values())
    out = []
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        out.append({"kernel": k, "launches": len(v), "mean_us": round(sum(v) / len(v), 3),
                    "total_us": round(sum(v), 2), "share": round(sum(v) / tot, 4)})
    return out


def full(path, label=""):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, units, vals = r[0], r[1], r[2:]
    res = []
    for v in vals:
        m = {}
        for i, n in enumerate(h):
            if n in KEYS or n == "Kernel Name":
                m[n] = (v[i] + (" " + units[i] if units[i] else "")).strip()
        res.append(m)
    # stall reasons (sass page)
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    stalls = collections.Counter()
    top = []
    if len(rows) > 2:
        hh = rows[1]
        ix = {n: i for i, n in enumerate(hh)}
        cols = [n for n in hh if n.startswith("stall_") and "Not Issued" not in n]
        for row in rows[2:]:
            if len(row) != len(hh):
                continue
            try:
                s = int(row[ix["Warp Stall Sampling (All Samples)"]] or 0)
            except ValueError:
                continue
            for c in cols:
                try:
                    stalls[c] += int(row[ix[c]] or 0)
                except ValueError:
                    pass
            top.append((s, row[ix["Source"]].strip()))
    top.sort(reverse=True)
    return {"label": label, "kernels": res, "stall_totals": dict(stalls.most_common(10)),
            "top_stall_instructions": [f"{s} {t}" for s, t in top[:12]]}


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(json.dumps(launches(sys.argv[2]), indent=1))
    else:
        print(json.dumps(full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""), indent=1))
