#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per
kernel: launches, mean us, share of the library's own kernel time.
usage: tools/ncu_summary.py launches.csv [title] > profiles/rNN_launches_summary.csv"""
import csv
import re
import sys
from collections import OrderedDict


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    with open(path) as f:
        lines = [x for x in f if x.startswith('"')]
    rows = list(csv.DictReader(lines))
    agg = OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        name = re.sub(r"\(.*\)$", "", name).replace("void ", "").replace("(int)", "")
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(
            r["Metric Unit"], 1e-3)
        v = float(r["Metric Value"].replace(",", "")) * scale
        n, s = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, s + v)
    own = {k: v for k, v in agg.items() if not k.startswith("at::")}
    tot = sum(s for _, s in own.values()) or 1.0
    print("# ncu launch list, %s, gpu__time_duration.sum, --clock-control none" % title)
    print("# cold-cache and serialised: compare shares, not absolute values")
    print("kernel, launches, mean_us, share_of_distir_step")
    for k, (n, s) in agg.items():
        share = "%.3f" % (s / tot) if k in own else "-"
        print("%s, %d, %.2f, %s" % (k.replace(",", ";"), n, s / n, share))


if __name__ == "__main__":
    main()
