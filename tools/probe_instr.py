"""Instrumented probe (build with -DDISTIR_INSTR): per grid, counts of
add_task calls / fast-path hits / cache refreshes / crossing passes / warp
steps, and warp cycles per work item.  Not part of the product."""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import workloads as W
import paper_2111_05426_b200 as pkg
from paper_2111_05426_b200 import Simulator

NAMES = ["tasks", "fast", "refresh", "plain", "steps", "item_cycles", "-", "items", "max_item_cycles",
         "slow_cycles", "slow_entries", "max_item_tag", "refresh_cyc", "cross_cyc", "-", "addtask_cyc",
         "quick_try", "quick_ok", "setup_cycles", "wave_cycles", "fill_cycles", "q_range", "q_tieE", "q_range1", "q_tieE1",
         "q_twice", "q_rest", "cost_cycles", "mem_cycles", "-", "-", "-", "fstep_cyc", "fstep_n",
         "sstep_cyc", "sstep_n", "-", "-", "-", "-"]


def counters():
    buf = (ctypes.c_ulonglong * 40)()
    pkg.lib.distir_debug_counters(buf, 40)
    return list(buf)


def main():
    sim = Simulator(W.MODELS, W.TOPOLOGIES)
    names = list(W.MODELS)
    mi = {n: i for i, n in enumerate(names)}
    tb = list(W.TOPOLOGIES).index("TB200")
    cases = [("xl P2 K128", None, [(mi["gpt2_xl"], tb, 8, 1, 2, 128, 1 << 20)]),
             ("xl P16 K128", None, [(mi["gpt2_xl"], tb, 1, 1, 16, 128, 1 << 20)]),
             ("mlp1b P2 K128", None, [(mi["mlp_1b"], tb, 8, 1, 2, 128, 1 << 18)]),
             ("16x xl P2 K128", None, [(mi["gpt2_xl"], tb, 8, 1, 2, 128, 1 << e) for e in range(7, 21)])]
    # one warp each when DISTIR_PLAN_BUDGET_X=0 (no splitting): do the binade
    # crossings of configurations that differ only in batch size line up?
    cases += [("8x xl P2 K128 Bsweep", None, [(mi["gpt2_xl"], tb, 1, 1, 2, 128, 1 << e) for e in range(13, 21)]),
              ("8x xl P2 K128 DTmix", None, [(mi["gpt2_xl"], tb, D, T, 2, 128, 1 << 20)
                                             for D, T in [(1, 1), (2, 1), (1, 2), (4, 1), (2, 2), (1, 4), (8, 1), (4, 2)]])]
    if os.environ.get("PROBE_GRIDS", "1") == "1":
        cases += [(g, W.GRIDS[g], None) for g in ["W3", "W2", "W5"]]
    for name, grid, cfgs in cases:
        n = sim.upload(grid=grid, configs=cfgs)
        outs = sim.device_outputs(n, k=10)
        sim.launch(outs, k=10)
        torch.cuda.synchronize()
        counters()
        sim.profile(True)
        sim.launch(outs, k=10)
        p = sim.profile(False)
        c = counters()
        d = dict(zip(NAMES, c))
        print("%-16s sim %.3f ms  tasks %d fast %.3f refresh/task %.3f plain/task %.3f steps %d "
              "items %d avg_item_cyc %.0f max_item_cyc %d slow_cyc/item %.0f slow_entries/item %.1f" % (
                  name, p["ms_simulate"], d["tasks"], d["fast"] / max(d["tasks"], 1),
                  d["refresh"] / max(d["tasks"], 1), d["plain"] / max(d["tasks"], 1), d["steps"],
                  d["items"], d["item_cycles"] / max(d["items"], 1), d["max_item_cycles"],
                  d["slow_cycles"] / max(d["items"], 1), d["slow_entries"] / max(d["items"], 1)))
        print("   lane-cycles in add_task %d: refresh %d, crossing passes %d (per add_task call: %.0f / %.0f / %.0f)" % (
            d["addtask_cyc"], d["refresh_cyc"], d["cross_cyc"], d["addtask_cyc"] / max(d["tasks"], 1),
            d["refresh_cyc"] / max(d["tasks"], 1), d["cross_cyc"] / max(d["tasks"], 1)))
        print("   quick path: %d tries, %d ok; wavefront cycles (lane 0, summed over items) %d = %.0f%% of item cycles" % (
            d["quick_try"], d["quick_ok"], d["wave_cycles"], 100.0 * d["wave_cycles"] / max(d["item_cycles"], 1)))
        print("   setup (costs, memory) %d cycles/item [costs %d, memory profiles %d], table fill %d cycles/item" % (
            d["setup_cycles"] / max(d["items"], 1), d["cost_cycles"] / max(d["items"], 1),
            d["mem_cycles"] / max(d["items"], 1), d["fill_cycles"] / max(d["items"], 1)))
        print("   quick-path misses: x outside table %d, ties in E %d, E+1 outside table %d, ties in E+1 %d, "
              "crossing pass beyond E+1 %d, rest overflows E+1 %d" % tuple(d[k] for k in (
                  "q_range", "q_tieE", "q_range1", "q_tieE1", "q_twice", "q_rest")))
        print("   GPT-2 wavefront steps without a slow lane: %d, %.0f cycles each; with: %d, %.0f cycles each" % (
            d["fstep_n"], d["fstep_cyc"] / max(d["fstep_n"], 1), d["sstep_n"], d["sstep_cyc"] / max(d["sstep_n"], 1)))
        tag = d["max_item_tag"]
        key = (tag >> 5) & 0x7FFFF
        print("   slowest item: %d cycles, kind %d P %d L %d, %d configs" % (
            tag >> 24, key & 1, ((key >> 1) & 63) + 1, ((key >> 7) & 1023) + 1, tag & 31))


if __name__ == "__main__":
    main()
