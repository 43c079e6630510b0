"""Probe: k_simulate time of single configurations launched alone (the
long-pole latency of one config), and of whole grids.  Prints one line per
probe: name, configs, kernel ms (CUDA events via distir_profile)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from paper_2111_05426_b200 import Simulator


def time_launch(sim, grid=None, configs=None, reps=20):
    n = sim.upload(grid=grid, configs=configs)
    outs = sim.device_outputs(n, k=10)
    for _ in range(3):
        sim.launch(outs, k=10)
    torch.cuda.synchronize()
    sim.profile(True)
    for _ in range(reps):
        sim.launch(outs, k=10)
    p = sim.profile(False)
    return n, {k: p[k] / p["launches"] for k in ("ms_prepare", "ms_simulate", "ms_topk")}


def main():
    only = sys.argv[1] if len(sys.argv) > 1 else None
    sim = Simulator(W.MODELS, W.TOPOLOGIES)
    names = list(W.MODELS)
    mi = {n: i for i, n in enumerate(names)}
    tb = list(W.TOPOLOGIES).index("TB200")
    probes = [
        ("xl P2 K128 D8", [(mi["gpt2_xl"], tb, 8, 1, 2, 128, 1 << 20)]),
        ("xl P2 K128 D1", [(mi["gpt2_xl"], tb, 1, 1, 2, 128, 1 << 20)]),
        ("xl P16 K128", [(mi["gpt2_xl"], tb, 1, 1, 16, 128, 1 << 20)]),
        ("xl P1 K1", [(mi["gpt2_xl"], tb, 16, 1, 1, 1, 1 << 20)]),
        ("small P2 K128", [(mi["gpt2_small"], tb, 8, 1, 2, 128, 1 << 20)]),
        ("xl P2 K2", [(mi["gpt2_xl"], tb, 8, 1, 2, 2, 1 << 20)]),
        ("mlp1b P2 K128", [(mi["mlp_1b"], tb, 8, 1, 2, 128, 1 << 18)]),
        ("mlpw4 P64 K128", [(mi["mlp_w4"], tb, 1, 1, 64, 128, 1024)]),
        ("mlpw4 P1 K128", [(mi["mlp_w4"], tb, 1, 1, 1, 128, 1024)]),
        ("16x xl P2 K128", [(mi["gpt2_xl"], tb, 8, 1, 2, 128, 1 << e) for e in range(7, 21)] * 1),
    ]
    for name, cf in probes:
        if only and name != only:
            continue
        n, t = time_launch(sim, configs=cf)
        print("%-18s n=%-6d simulate %.4f ms  prepare %.4f  topk %.4f" % (
            name, n, t["ms_simulate"], t["ms_prepare"], t["ms_topk"]))
    for g in ([] if only else ["W1", "W2", "W3", "W4", "W5"]):
        n, t = time_launch(sim, grid=W.GRIDS[g], reps=5 if g == "W5" else 20)
        print("%-18s n=%-8d simulate %.4f ms  prepare %.4f  topk %.4f" % (
            g, n, t["ms_simulate"], t["ms_prepare"], t["ms_topk"]))


if __name__ == "__main__":
    main()
