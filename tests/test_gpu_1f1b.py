"""GPU parity of the synchronous 1F1B schedule (
DESIGN reading R6) -- the CUDA co-simulation (k_simulate mode 5) against the
CPU oracle on the same seeded inputs, with the bars of test_gpu_parity.py
(reason bits, peaks, top-k bit-exact; makespans within 1e-12 relative)."""
import numpy as np
import pytest

import oracle
import workloads as W
from test_gpu_parity import THREADS, assert_parity, full_grid_check

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sim():
    import torch
    assert torch.cuda.is_available()
    from paper_2111_05426_b200 import Simulator
    s = Simulator(W.MODELS, W.TOPOLOGIES, device=0)
    yield s
    s.close()


def test_w1_1f1b(sim):
    for topo in ["TB200", "TV100", "TM0", "TM5"]:
        g = W.grid_with("W1", models=["mlp_w1_1f1b"], topos=[topo])
        assert full_grid_check(sim, g) == 1.0


def test_w2_1f1b(sim):
    """The paper's MLP-1B grid under 1F1B."""
    assert full_grid_check(sim, W.grid_with("W2", models=["mlp_1b_1f1b"])) == 1.0


def test_w4_1f1b(sim):
    """Deep pipelines: 64-layer MLP, P up to 64 (two stages per lane beyond
    32), K up to 128."""
    g = W.grid_with("W4", models=["mlp_w4_1f1b"])
    assert full_grid_check(sim, g) == 1.0


def test_mixed_schedules_one_grid(sim):
    """GPipe and 1F1B models in one spec: buckets never mix schedules."""
    g = W.grid_with("W2", models=["mlp_1b", "mlp_1b_1f1b"], topos=["TB200", "TM2"])
    assert full_grid_check(sim, g, k=32) == 1.0


def test_explicit_1f1b_all_shapes(sim):
    """Every P in 1..32 (not only powers of two) with K in 1..200: more
    distinct warp shapes than hash buckets, so the 1F1B catch-all bucket runs
    too."""
    from paper_2111_05426_b200 import Simulator
    models = {"a": W.mlp(32, 64, schedule=1), "b": W.mlp(5, 32, schedule=1)}
    topos = {"TM1": W.TOPOLOGIES["TM1"], "TB200": W.TOPOLOGIES["TB200"]}
    s = Simulator(models, topos, device=0)
    rng = np.random.default_rng(524)
    cfgs = []
    for P in range(1, 33):
        for K in range(1, 201):
            D = 1 << int(rng.integers(0, 2))
            T = 1 << int(rng.integers(0, 2)) if P <= 16 else 1
            cfgs.append((0, int(rng.integers(2)), D, T, P, K, D * K * 4))
    for P in range(1, 8):
        for K in [1, 2, 3, 7]:
            cfgs.append((1, 1, 1, 2, P, K, 2 * K))       # P > L: invalid
    res = s.eval(configs=cfgs, k=16)
    ref = {"makespan": [], "peak": [], "reason": []}
    for (mi, ti, D, T, P, K, B) in cfgs:
        r = oracle.eval_config(models[list(models)[mi]], topos[list(topos)[ti]],
                               D, T, P, K, B)
        for k in ref:
            ref[k].append(r[k])
    ref = {k: np.array(v) for k, v in ref.items()}
    ref["reason"] = ref["reason"].astype(np.uint32)
    assert assert_parity(res, ref, "1f1b explicit") == 1.0
    bt = np.array([c[6] for c in cfgs])
    pos, _ = oracle.topk(np.arange(len(cfgs)), bt, ref["makespan"], ref["peak"],
                         ref["reason"], 16)
    assert res["topk"]["index"].tolist() == pos.tolist()
    s.close()


def test_1f1b_beyond_32_stages(sim):
    """32 < P <= 64 runs two stages per lane (k_simulate mode 7): explicit
    configurations (non-power-of-two P too) against the oracle."""
    mi = list(W.MODELS).index("mlp_w4_1f1b")
    cfgs = [(mi, 0, 1, 1, P, K, 64 * K) for P in (33, 40, 47, 64) for K in (1, 2, 5, 16)]
    res = sim.eval(configs=cfgs, k=4)
    ref = {"makespan": [], "peak": [], "reason": []}
    for (m_, ti, D, T, P, K, B) in cfgs:
        r = oracle.eval_config(W.MODELS["mlp_w4_1f1b"], W.TOPOLOGIES[list(W.TOPOLOGIES)[ti]],
                               D, T, P, K, B)
        for k in ref:
            ref[k].append(r[k])
    ref = {k: np.array(v) for k, v in ref.items()}
    ref["reason"] = ref["reason"].astype(np.uint32)
    assert assert_parity(res, ref, "1f1b P > 32") == 1.0
