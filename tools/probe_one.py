"""Launch one explicit configuration repeatedly (for ncu / compute-sanitizer
of a single long pole).  usage: python tools/probe_one.py MODEL P K [D T B REPS]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from paper_2111_05426_b200 import Simulator


def main():
    a = sys.argv[1:]
    model, P, K = a[0], int(a[1]), int(a[2])
    D = int(a[3]) if len(a) > 3 else 1
    T = int(a[4]) if len(a) > 4 else 1
    B = int(a[5]) if len(a) > 5 else (1 << 20)
    reps = int(a[6]) if len(a) > 6 else 6
    sim = Simulator(W.MODELS, W.TOPOLOGIES)
    mi = list(W.MODELS).index(model)
    tb = list(W.TOPOLOGIES).index("TB200")
    n = sim.upload(configs=[(mi, tb, D, T, P, K, B)])
    outs = sim.device_outputs(n, k=10)
    sim.profile(True)
    for _ in range(reps):
        sim.launch(outs, k=10)
    torch.cuda.synchronize()
    p = sim.profile(False)
    print("%s P%d K%d D%d T%d: simulate %.4f ms/launch, makespan %r" % (
        model, P, K, D, T, p["ms_simulate"] / p["launches"], outs["makespan"][0].item()))


if __name__ == "__main__":
    main()
