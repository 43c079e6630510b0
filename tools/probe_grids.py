"""Per-grid k_simulate time and work counters (tasks, slow-path entries,
warp steps).  usage: python tools/probe_grids.py [GRID|GRID:MODEL ...]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from paper_2111_05426_b200 import Simulator


def main():
    names = sys.argv[1:] or ["W2:mlp_1b_1f1b", "W4:mlp_w4_1f1b", "W2", "W4", "W3"]
    sim = Simulator(W.MODELS, W.TOPOLOGIES)
    for nm in names:
        g, _, m = nm.partition(":")
        grid = W.grid_with(g, models=[m]) if m else W.GRIDS[g]
        n = sim.upload(grid)
        outs = sim.device_outputs(n, k=10)
        for _ in range(3):
            sim.launch(outs, k=10)
        torch.cuda.synchronize()
        st = sim.last_stats()
        sim.profile(True)
        reps = 5 if n > 100000 else 20
        for _ in range(reps):
            sim.launch(outs, k=10)
        p = sim.profile(False)
        print("%-18s n=%-7d simulate %.4f ms  tasks %d slow %d steps %d items %d" % (
            nm, n, p["ms_simulate"] / p["launches"], st["tasks"], st["slow_tasks"],
            st["wave_steps"], st["n_items"]))


if __name__ == "__main__":
    main()
