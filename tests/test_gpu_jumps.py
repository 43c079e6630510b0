"""GPU parity of the steady-state jumps (DESIGN §5 "Steady-state jumps"):
long pipelines (K = 64, 128) where k_simulate adds whole 8-step (GPipe) or
24-step (1F1B) windows in closed form, against the CPU oracle's op-by-op
walk, element by element -- including the dyadic regression topology TRD,
whose costs put round-to-nearest ties in the higher binades (the even-ulps
condition of the jump is what keeps those exact).  Each case also checks,
on configurations launched alone (one per warp), that the jumps really
fired: fewer warp wavefront steps than the schedule has."""
import numpy as np
import pytest

import oracle
import workloads as W
from test_gpu_parity import assert_parity

pytestmark = pytest.mark.gpu

MODELS = list(W.MODELS)
TOPOS = list(W.TOPOLOGIES)


@pytest.fixture(scope="module")
def sim():
    import torch
    assert torch.cuda.is_available()
    from paper_2111_05426_b200 import Simulator
    s = Simulator(W.MODELS, W.TOPOLOGIES, device=0)
    yield s
    s.close()


def _check_list(sim, cfgs):
    res = sim.eval(configs=cfgs, k=10)
    ref = {"makespan": [], "peak": [], "reason": []}
    for (mi, ti, D, T, P, K, B) in cfgs:
        r = oracle.eval_config(W.MODELS[MODELS[mi]], W.TOPOLOGIES[TOPOS[ti]], D, T, P, K, B)
        for key in ref:
            ref[key].append(r[key])
    ref = {key: np.array(v) for key, v in ref.items()}
    ref["reason"] = ref["reason"].astype(np.uint32)
    assert assert_parity(res, ref, "jumps") == 1.0      # bit-exact makespans
    return res


def _steps_alone(sim, cfg):
    return sim.eval(configs=[cfg], k=1)["stats"]["wave_steps"]


@pytest.mark.parametrize("topo", ["TB200", "TM3", "TRD"])
def test_gpt2_gpipe_jumps(sim, topo):
    ti = TOPOS.index(topo)
    cfgs = []
    for model in ["gpt2_small", "gpt2_xl"]:
        mi = MODELS.index(model)
        for (D, T) in [(1, 1), (4, 1), (1, 2)]:
            for P in [1, 2, 8, 16]:
                for K in [64, 128]:
                    cfgs.append((mi, ti, D, T, P, K, D * K * 4))
    _check_list(sim, cfgs)
    # the jumps fired: a configuration alone walks fewer than 2(K-1)+P steps
    xl = MODELS.index("gpt2_xl")
    fired = [_steps_alone(sim, (xl, ti, 1, 1, P, 128, 512)) < 2 * 127 + P for P in (2, 8, 16)]
    assert any(fired), fired


@pytest.mark.parametrize("topo", ["TB200", "TRD"])
def test_mlp_1f1b_jumps(sim, topo):
    ti = TOPOS.index(topo)
    mi = MODELS.index("mlp_1b_1f1b")
    cfgs = []
    for (D, T) in [(1, 1), (2, 1), (1, 2)]:
        for P in [2, 4, 8, 16]:
            for K in [64, 128]:
                cfgs.append((mi, ti, D, T, P, K, D * K * 2))
    _check_list(sim, cfgs)
    fired = [_steps_alone(sim, (mi, ti, 1, 1, P, 128, 256)) < 3 * (2 * P + 2 * 128 - 3) + 3
             for P in (2, 4, 8)]
    assert any(fired), fired


@pytest.mark.parametrize("topo", ["TB200", "TRD"])
def test_mlp_gpipe_two_stages_per_lane_jumps(sim, topo):
    """32 < P <= 64: lanes hold two stages (k_simulate mode 4) and the jump
    tests both (wave_jump2)."""
    ti = TOPOS.index(topo)
    mi = MODELS.index("mlp_w4")
    cfgs = [(mi, ti, 1, 1, P, K, 1024) for P in (33, 48, 64) for K in (64, 128)]
    _check_list(sim, cfgs)
    fired = [_steps_alone(sim, (mi, ti, 1, 1, P, 128, 1024)) < 2 * (2 * 127 + P) for P in (48, 64)]
    assert any(fired), fired


@pytest.mark.parametrize("topo", ["TB200", "TRD"])
def test_mlp_1f1b_two_stages_per_lane_jumps(sim, topo):
    """1F1B with 32 < P <= 64 (k_simulate mode 7): the jump tests both stages
    of a lane; bit-exact against the oracle."""
    ti = TOPOS.index(topo)
    mi = MODELS.index("mlp_w4_1f1b")
    cfgs = [(mi, ti, 1, 1, P, K, 1024) for P in (33, 48, 64) for K in (64, 128)]
    _check_list(sim, cfgs)
    fired = [_steps_alone(sim, (mi, ti, 1, 1, P, 128, 1024)) < 3 * (2 * P + 2 * 128 - 3) + 3 for P in (48, 64)]
    assert any(fired), fired
