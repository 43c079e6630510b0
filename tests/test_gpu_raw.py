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


def test_program_rules_rejected(sim):
    """distir_raw_eval checks the program rules the kernel relies on (P:301-306,
    P:506): inputs defined before use, each value defined once, outputs on one
    of the op's devices, non-overlapping per-program ranges."""
    import ctypes
    import paper_2111_05426_b200 as pkg
    from paper_2111_05426_b200 import DistirError
    p = (1, 16, True, False)                     # a parameter on device 1
    # input used before it is defined (value 1 is produced by the second op)
    with pytest.raises(DistirError, match="before"):
        sim.eval_raw([(2, [([0], 1.0, [1], []), ([0], 1.0, [], [1])], [p, (0, 8, False, False)])])
    # defined twice
    with pytest.raises(DistirError, match="twice"):
        sim.eval_raw([(2, [([1], 1.0, [], [0])], [p])])
    # output off the op's devices
    with pytest.raises(DistirError, match="devices"):
        sim.eval_raw([(2, [([0], 1.0, [0], [1])], [p, (1, 8, False, False)])])
    # the accepted form of the same program
    r = sim.eval_raw([(2, [([0, 1], 1.0, [0], [1])], [p, (0, 8, False, True)])])[0]
    assert r["makespan"] == 1.0 and r["peak"].tolist() == [8, 16]
    # two programs sharing a value range
    progs = (pkg.distir_raw_program * 2)(pkg.distir_raw_program(1, 0, 0, 1, 0, 0),
                                         pkg.distir_raw_program(1, 0, 0, 1, 0, 1))
    vals = (pkg.distir_raw_value * 1)(pkg.distir_raw_value(0, 1, 8))
    ms = (ctypes.c_double * 2)()
    b = ctypes.c_size_t()
    pkg.lib.distir_raw_workspace_size(2, 0, 0, 1, 2, ctypes.byref(b))
    ws = sim.torch.empty(b.value, dtype=sim.torch.uint8, device=sim.device)
    st = pkg.lib.distir_raw_eval(sim.handle, progs, 2, None, 0, None, 0, vals, 1, 2,
                                 ctypes.c_void_p(ws.data_ptr()), ws.numel(), ms, None, None,
                                 None, None)
    assert st == 1 and b"overlap" in pkg.lib.distir_last_error()
