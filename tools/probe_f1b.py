"""Probe: 1F1B grids (k_simulate mode 5) -- device time per launch."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
from paper_2111_05426_b200 import Simulator
from probe_longpole import time_launch

sim = Simulator(W.MODELS, W.TOPOLOGIES)
for name, g in [("W1-1F1B", W.grid_with("W1", models=["mlp_w1_1f1b"])),
                ("W2-1F1B", W.grid_with("W2", models=["mlp_1b_1f1b"])),
                ("W4-1F1B", W.grid_with("W4", models=["mlp_w4_1f1b"]))]:
    n, t = time_launch(sim, grid=g)
    print("%-16s n=%-6d simulate %.4f ms  prepare %.4f  topk %.4f" % (name, n, t["ms_simulate"], t["ms_prepare"], t["ms_topk"]))
