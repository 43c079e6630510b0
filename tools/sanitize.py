"""One evaluation of a named grid through the C ABI (for compute-sanitizer
runs, tools/sanitize.sh): W1, W4 (two stages per lane, shuffles across the
lane-31/32 wrap), W4 under 1F1B (the co-simulation), W2 under ZeRO (lane =
(stage, replica)), W3 (GPT-2 and its steady-state jumps), W2 under 1F1B (its
jumps), a 3,000-configuration synthetic sweep (concurrent simulate kernels,
the plain MLP kernel) -- plus the device merge of 3 virtual shards.
usage: python tools/sanitize.py NAME"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from paper_2111_05426_b200 import Simulator

GRIDS = {
    "W1": W.GRIDS["W1"],
    "W3": W.GRIDS["W3"],
    "W4": W.GRIDS["W4"],
    "W4_1F1B": W.grid_with("W4", models=["mlp_w4_1f1b"]),
    "W2_ZERO": W.grid_with("W2", models=["mlp_1b_zero"]),
    # the 1F1B steady-state jumps (K up to 128)
    "W2_1F1B": W.grid_with("W2", models=["mlp_1b_1f1b"]),
    # the synthetic sweep: five simulate kernels at once (side streams), the
    # plain MLP kernel (mode 8)
    "SYN": dict(W.GRIDS["W5"], synth_count=3000),
}


def main():
    name = sys.argv[1]
    sim = Simulator(W.MODELS, W.TOPOLOGIES, device=0)
    res = sim.eval(GRIDS[name], k=10)
    lists = torch.full((3, 10, 4), -1, dtype=torch.int64, device="cuda")
    for g in range(3):
        n = sim.upload(GRIDS[name], rank=g, n_ranks=3)
        outs = sim.device_outputs(n, k=10)
        sim.launch(outs, k=10)
        lists[g].copy_(outs["topk"])
    out, nn = sim.merge_topk(lists, None, k=10)
    torch.cuda.synchronize()
    assert out[:int(nn.item()), 0].cpu().tolist() == res["topk"]["index"].tolist()
    print("%s: %d configs, top-1 %d, merge ok" % (name, res["n"], res["topk"]["index"][0]))
    sim.close()


if __name__ == "__main__":
    main()
