"""GPU parity of the raw-program mode (f3, distir_raw_eval) against the CPU
oracle's explicit-program walk: the Fig. 3 traces (88 / 94),
random programs (P7), and the oracle's own generated MLP / GPT-2 programs --
makespans, per-op start/end, final clocks and per-device peaks bit-exact."""
import json
import os

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def sim():
    from paper_2111_05426_b200 import Simulator
    s = Simulator(W.MODELS, W.TOPOLOGIES, device=0)
    yield s
    s.close()


def test_fig3_on_gpu(sim):
    with open(os.path.join(GOLDEN, "fig3_trace.json")) as f:
        g = json.load(f)
    top = [(e[1], float(e[2])) for e in g["events_top"]]
    names = [e[0] for e in g["events_top"]]
    i, j = names.index(g["swap"][0]), names.index(g["swap"][1])
    sw = list(top)
    sw[i], sw[j] = sw[j], sw[i]
    a, b = sim.eval_raw([(2, top, []), (2, sw, [])])
    assert a["makespan"] == 88 and b["makespan"] == 94


def test_random_programs_match_oracle(sim):
    progs = [W.random_program(seed) for seed in range(300)]
    res = sim.eval_raw([(n, ops, []) for n, ops in progs])
    for (n, ops), r in zip(progs, res):
        ref = oracle.simulate_raw(n, ops)
        assert r["makespan"] == ref["makespan"]
        assert (r["start"] == ref["start"]).all() and (r["end"] == ref["end"]).all()
        assert (r["clocks"] == ref["clocks"]).all()


def test_generated_programs_match_oracle(sim):
    t = W.TOPOLOGIES["TB200"]
    cases = [(W.MODELS["mlp_w1"], D, T, P, K, 64) for (D, T, P, K) in
             [(1, 1, 1, 1), (2, 1, 1, 2), (1, 2, 2, 2), (2, 2, 1, 1), (1, 1, 2, 2)]]
    g = dict(W.MODELS["gpt2_small"], n_layer=3, d_model=64, n_head=4, vocab_pad=128, n_ctx=16)
    cases += [(g, D, T, P, K, D * K * 2) for (D, T, P, K) in [(1, 2, 2, 2), (2, 1, 3, 3)]]
    progs, refs = [], []
    for (m, D, T, P, K, B) in cases:
        vals, ops = oracle.export_program(m, t, D, T, P, K, B)
        progs.append((D * T * P, [o[:4] for o in ops], vals))
        refs.append(oracle.eval_config(m, t, D, T, P, K, B))
    res = sim.eval_raw(progs)
    for r, ref in zip(res, refs):
        assert r["makespan"] == ref["makespan"]
        assert r["peak"].tolist() == ref["peaks"].tolist()


def test_invalid_program_rejected(sim):
    from paper_2111_05426_b200 import DistirError
    with pytest.raises(DistirError):
        sim.eval_raw([(2, [([0, 5], 1.0)], [])])       # device 5 of 2
