"""Summarise ncu output for profiles/.

    python scripts/ncu_summary.py launches <launches.csv>            # per-kernel shares
    python scripts/ncu_summary.py report <file.ncu-rep> [workload]    # key metrics of a --set full capture
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum.per_second",
    "dram__bytes_write.sum.per_second", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_barrier",
    "smsp__pcsamp_sample_count", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
]


def launches(path: str) -> dict:
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    per = defaultdict(lambda: defaultdict(list))
    for r in rows[hdr + 1:]:
        if len(r) > vi and r[vi]:
            name = r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "")
            per[name][r[mi]].append(float(r[vi].replace(",", "")))
    t = "gpu__time_duration.sum"
    total = sum(sum(m[t]) for m in per.values())
    out = {}
    for k, m in sorted(per.items(), key=lambda kv: -sum(kv[1][t])):
        v = m[t]
        out[k] = {"launches": len(v), "total_ns": sum(v), "mean_ns": sum(v) / len(v), "share": sum(v) / total}
        for metric, vals in m.items():  # any other metric captured with the launch list: mean per launch
            if metric != t:
                out[k][f"mean_{metric}"] = sum(vals) / len(vals)
    return out


def report(path: str) -> dict:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")][:80]}
        for i, n in enumerate(h):
            if n in KEYS:
                d[n] = f"{v[i]} {units[i]}".strip()
        res.append(d)
    return {"launches": res}


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(json.dumps(launches(path) if mode == "launches" else report(path), indent=1))
