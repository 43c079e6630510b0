#!/usr/bin/env python
"""Summarise an `ncu --set full` report of k_simulate into the JSON bench.py
reads for its roofline (profiles/ncu_simulate_summary.json): per-launch warp
instructions, DRAM bytes, cycles, issue / occupancy and the warp-stall mix,
keyed by the sha of the library sources it was captured from.

usage: tools/ncu_capture.py REPORT.ncu-rep OUT.json "what was captured"
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

KEEP = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "sm__cycles_active.avg", "gpc__cycles_elapsed.max",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__shared_mem_per_block_dynamic"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ms": 1e-3,
         "ns": 1e-9, "s": 1.0}


def main():
    rep, out, what = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}

    def num(r, name):
        v = r[col[name]].replace(",", "")
        return float(v) * SCALE.get(units[col[name]], 1.0)

    n = len(data)
    mean = lambda name: sum(num(r, name) for r in data) / n
    stall = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): sum(num(r, h) for r in data)
             for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_")
             and not h.endswith("_not_issued")}
    tot = sum(stall.values()) or 1.0
    from bench import source_sha
    res = {
        "kernel": data[0][col["Kernel Name"]] if "Kernel Name" in col else "k_simulate",
        "workload": what,
        "source_sha": source_sha(),
        "launches": n,
        "inst_executed_per_launch": mean("smsp__inst_executed.sum"),
        "dram_bytes_per_launch": mean("dram__bytes_read.sum") + mean("dram__bytes_write.sum"),
        "duration_us": mean("gpu__time_duration.sum") * 1e6,
        "sm_cycles_active_avg": mean("sm__cycles_active.avg"),
        "cycles_elapsed_max": mean("gpc__cycles_elapsed.max"),
        "metrics": {k: [r[col[k]] + " " + units[col[k]] for r in data] for k in KEEP if k in col},
        "warp_stall_pct": {k: round(100.0 * v / tot, 1)
                           for k, v in sorted(stall.items(), key=lambda kv: -kv[1]) if v > 0},
        "note": "cold-cache, serialised, --clock-control none; per-launch means over the "
                "captured launches",
    }
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: res[k] for k in ("kernel", "inst_executed_per_launch",
                                           "dram_bytes_per_launch", "duration_us")}))


if __name__ == "__main__":
    main()
