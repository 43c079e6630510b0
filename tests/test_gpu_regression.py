"""GPU parity of the regression cost model (
DESIGN reading R7): the CUDA path's closed-form per-op FLOPs and tensor
bytes against the oracle's explicit programs, with the bars of
test_gpu_parity.py."""
import numpy as np
import pytest

import oracle
import workloads as W
from test_gpu_parity import assert_parity, full_grid_check

pytestmark = pytest.mark.gpu

REG = [t for t in ("TRD", "TB200R") if t in W.TOPOLOGIES]


@pytest.fixture(scope="module")
def sim():
    import torch
    assert torch.cuda.is_available()
    from paper_2111_05426_b200 import Simulator
    s = Simulator(W.MODELS, W.TOPOLOGIES, device=0)
    yield s
    s.close()


def test_w1_w2_regression(sim):
    for t in REG:
        assert full_grid_check(sim, W.grid_with("W1", topos=[t])) == 1.0
        assert full_grid_check(sim, W.grid_with("W2", topos=[t])) == 1.0


def test_w3_regression(sim):
    """GPT-2 inference grid with both regression topologies and an analytic
    one in the same spec."""
    assert full_grid_check(sim, W.grid_with("W3", topos=REG + ["TB200"])) == 1.0


def test_1f1b_regression(sim):
    g = W.grid_with("W2", models=["mlp_1b_1f1b", "mlp_1b"], topos=REG)
    assert full_grid_check(sim, g) == 1.0


def test_single_feature_topologies(sim):
    """One coefficient at a time (unit value): per-op FLOPs / bytes / op
    counts of every kind, summed by the timeline, on small explicit configs
    with T, P > 1."""
    from paper_2111_05426_b200 import Simulator
    topos = {}
    for k in W.REGRESSION_KEYS:
        t = dict(W.TOPOLOGIES["TB200"], cost_model=1)
        for kk in W.REGRESSION_KEYS:
            t[kk] = 1.0 if kk == k else 0.0
        topos[k] = t
    models = {"m": W.mlp(6, 64), "g": dict(W.MODELS["gpt2_small"], n_layer=3, d_model=64,
                                             n_head=8, vocab_pad=256, n_ctx=32)}
    s = Simulator(models, topos, device=0)
    cfgs = []
    for mi in range(2):
        for ti in range(len(topos)):
            for (D, T, P, K) in [(1, 1, 1, 1), (1, 2, 3, 2), (2, 2, 2, 3), (1, 4, 1, 2)]:
                cfgs.append((mi, ti, D, T, P, K, 4 * D * K))
    res = s.eval(configs=cfgs, k=4)
    ref = {"makespan": [], "peak": [], "reason": []}
    for (mi, ti, D, T, P, K, B) in cfgs:
        r = oracle.eval_config(models[list(models)[mi]], topos[list(topos)[ti]], D, T, P, K, B)
        for k in ref:
            ref[k].append(r[k])
    ref = {k: np.array(v) for k, v in ref.items()}
    ref["reason"] = ref["reason"].astype(np.uint32)
    assert assert_parity(res, ref, "features") == 1.0
    s.close()


def test_invalid_regression_topology_rejected():
    from paper_2111_05426_b200 import DistirError, Simulator
    t = dict(W.TOPOLOGIES["TRD"], mm_s_per_byte=-1.0)
    with pytest.raises(DistirError, match="regression"):
        Simulator({"m": W.mlp(2, 64)}, {"t": t}, device=0)
    t = dict(W.TOPOLOGIES["TB200"], cost_model=7)
    with pytest.raises(DistirError, match="cost_model"):
        Simulator({"m": W.mlp(2, 64)}, {"t": t}, device=0)
