"""Debug probe (instrumented build, -DDISTIR_INSTR): steady-state jump
checks per grid -- attempts with an interior window, and live lanes failing
the binade / uniform-shift / even-ulps / memory tests -- plus warp steps."""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
import paper_2111_05426_b200 as pkg
from paper_2111_05426_b200 import Simulator


def main():
    sim = Simulator(W.MODELS, W.TOPOLOGIES)
    buf = (ctypes.c_ulonglong * 40)()
    for nm in sys.argv[1:] or ["W2:mlp_1b_1f1b", "W3", "W2"]:
        g, _, m = nm.partition(":")
        grid = W.grid_with(g, models=[m]) if m else W.GRIDS[g]
        n = sim.upload(grid)
        outs = sim.device_outputs(n, k=10)
        sim.launch(outs, k=10)
        torch.cuda.synchronize()
        pkg.lib.distir_debug_counters(buf, 40)
        sim.launch(outs, k=10)
        torch.cuda.synchronize()
        pkg.lib.distir_debug_counters(buf, 40)
        c = list(buf)
        print("%-18s steps %d  jump attempts %d  lanes failing: binade %d  shift %d  odd-ulps %d  memory %d" % (
            nm, c[4], c[36], c[37], c[38], c[39], c[31]))


if __name__ == "__main__":
    main()
