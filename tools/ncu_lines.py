#!/usr/bin/env python
"""Per-source-line totals from `ncu -i rep --page source --csv --print-source
cuda,sass`: instructions executed and warp-stall samples, top N lines.
usage: tools/ncu_lines.py src.csv [N]"""
import csv
import sys
from collections import defaultdict


def main():
    path, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows = list(csv.reader(open(path)))
    fname = None
    hdr = None
    tot = defaultdict(lambda: [0, 0, ""])
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            ii = hdr.index("Instructions Executed")
            iss = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
            continue
        if r[1] == "" and r[2] == "":
            continue
        key = (fname, int(r[0]))
        try:
            tot[key][0] += int(float(r[ii] or 0))
            tot[key][1] += int(float(r[iss] or 0))
        except ValueError:
            continue
        if r[1]:
            tot[key][2] = r[1].strip()[:70]
    S = sum(v[1] for v in tot.values()) or 1
    I = sum(v[0] for v in tot.values()) or 1
    print("total instr %d  samples %d" % (I, S))
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1][1])[:n]:
        print("%-16s %5d  instr %9d (%4.1f%%)  stall %6d (%4.1f%%)  %s" % (
            k[0], k[1], v[0], 100.0 * v[0] / I, v[1], 100.0 * v[1] / S, v[2]))


if __name__ == "__main__":
    main()
