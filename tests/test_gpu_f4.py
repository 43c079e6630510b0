"""GPU parity of the memory-saving variants (DESIGN
readings R8 / R9): gradient checkpointing (run_mlp, all schedules) and ZeRO
(k_simulate mode 6: one lane per (stage, replica)) against the CPU oracle on
the same seeded inputs, with the bars of test_gpu_parity.py (reason bits,
peaks, top-k and op counts bit-exact; makespans within 1e-12 relative)."""
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


@pytest.mark.parametrize("name", ["mlp_w1_ckpt", "mlp_w1_zero"])
def test_w1_variants(sim, name):
    for topo in ["TB200", "TV100", "TM0", "TM5"]:
        g = W.grid_with("W1", models=[name], topos=[topo])
        assert full_grid_check(sim, g) == 1.0


@pytest.mark.parametrize("name", ["mlp_1b_ckpt", "mlp_1b_zero", "mlp_1b_zero_ckpt"])
def test_w2_variants(sim, name):
    """The paper's MLP-1B grid (W <= 16, K up to 128, 12 batch sizes)."""
    assert full_grid_check(sim, W.grid_with("W2", models=[name], topos=["TB200", "TM1"])) == 1.0


def test_variants_and_baseline_in_one_grid(sim):
    """Baseline, checkpointed, ZeRO and 1F1B models in one spec: warps
    never mix a ZeRO configuration (D lanes per stage) with others."""
    g = W.grid_with("W2", models=["mlp_1b", "mlp_1b_ckpt", "mlp_1b_zero", "mlp_1b_1f1b"],
                    world=[1, 2, 4, 8])
    assert full_grid_check(sim, g, k=32) == 1.0


def test_small_models_all_shapes(sim):
    """Odd layer counts, non-power-of-two P (balanced stage split), T up to
    4, D up to 8, node size 4, checkpointing under GPipe and 1F1B, ZeRO with
    and without checkpointing; explicit configurations one by one."""
    from paper_2111_05426_b200 import Simulator
    models = {}
    for L in (2, 3, 5, 8):
        models["c%d" % L] = W.mlp(L, 64, recompute=1)
        models["c1f%d" % L] = W.mlp(L, 64, recompute=1, schedule=1)
        models["z%d" % L] = W.mlp(L, 64, zero=1)
        models["zc%d" % L] = W.mlp(L, 64, zero=1, recompute=1)
    topos = {k: W.TOPOLOGIES[k] for k in ("TB200", "TM0", "TM6", "TRD")}
    s = Simulator(models, topos, device=0)
    names, tn = list(models), list(topos)
    rng = np.random.default_rng(974)
    cfgs = []
    for _ in range(400):
        mi = int(rng.integers(len(names)))
        L = models[names[mi]]["n_layer"]
        D = 1 << int(rng.integers(0, 4))
        T = 1 << int(rng.integers(0, 3))
        P = min(int(rng.integers(1, L + 2)), 64 // (D * T))   # P > L: invalid (bit 1)
        p2 = 1 << (P - 1).bit_length()
        if models[names[mi]]["zero"] and p2 * D > 32:
            D = max(1, 32 // p2)
        K = int(rng.integers(1, 9))
        cfgs.append((mi, int(rng.integers(len(tn))), D, T, P, K, D * K * int(rng.integers(1, 5))))
    res = s.eval(configs=cfgs, k=16)
    ref = {"makespan": [], "peak": [], "reason": []}
    for (mi, ti, D, T, P, K, B) in cfgs:
        r = oracle.eval_config(models[names[mi]], topos[tn[ti]], D, T, P, K, B)
        ref["makespan"].append(r["makespan"]); ref["peak"].append(r["peak"])
        ref["reason"].append(r["reason"])
    ref = {k: np.array(v) for k, v in ref.items()}
    ref["reason"] = ref["reason"].astype(np.uint32)
    assert assert_parity(res, ref, "f4 explicit") == 1.0
    bt = np.array([c[6] for c in cfgs])
    pos, _ = oracle.topk(np.arange(len(cfgs)), bt, ref["makespan"], ref["peak"], ref["reason"], 16)
    assert res["topk"]["index"].tolist() == pos.tolist()
    s.close()


def test_checkpointing_lowers_gpu_peaks(sim):
    """The property the variant exists for, on the GPU results of
    the W2 grid: never a higher peak, and lower for deep stages."""
    a = sim.eval(W.grid_with("W2", models=["mlp_1b"]), k=1)
    b = sim.eval(W.grid_with("W2", models=["mlp_1b_ckpt"]), k=1)
    ok = (a["reason"] & 0x1F) == 0
    assert (b["peak"][ok] <= a["peak"][ok]).all()
    assert (b["peak"][ok] < a["peak"][ok]).any()
    assert (b["makespan"][ok] >= a["makespan"][ok]).all()


def test_zero_unsupported_shapes():
    """ZeRO configurations needing more than 32 lanes (next_pow2(P) * D > 32
    with D > 1) are rejected with DISTIR_E_UNSUPPORTED (include/distir.h)."""
    from paper_2111_05426_b200 import DistirError, Simulator
    s = Simulator({"z": W.mlp(64, 64, zero=1)}, {"t": W.TOPOLOGIES["TB200"]}, device=0)
    with pytest.raises(DistirError) as e:
        s.eval(configs=[(0, 0, 4, 1, 16, 2, 64)], k=1)
    assert e.value.status == 2
    # a grid is rejected only when one of its (D, T, P) needs > 32 lanes
    with pytest.raises(DistirError) as e:
        s.eval(W.grid_with("W4", models=["z"], topos=["t"], dp_mask=W.ALL), k=1)
    assert e.value.status == 2
    s.close()


def test_w4_zero_model_runs(sim):
    """The W4 grid (P up to 64, D = 1) of a ZeRO model: D = 1 configurations
    run on the plain kernels (ZeRO partitions over replicas only), against
    the oracle on the whole grid."""
    assert full_grid_check(sim, W.grid_with("W4", models=["mlp_w4_zero"])) == 1.0


@pytest.mark.parametrize("name", ["mlp_w1_zero_1f1b"])
def test_w1_zero_under_1f1b(sim, name):
    """ZeRO under the paper's 1F1B schedule (oracle: the same ZeRO tasks in
    the unit-time order of reading R6)."""
    for topo in ["TB200", "TV100", "TM0", "TM5"]:
        assert full_grid_check(sim, W.grid_with("W1", models=[name], topos=[topo])) == 1.0


def test_w2_zero_under_1f1b(sim):
    """The paper's MLP-1B grid under ZeRO + 1F1B, plain and with checkpointing
    in one spec with the GPipe variant."""
    g = W.grid_with("W2", models=["mlp_1b_zero_1f1b", "mlp_1b_zero"], topos=["TB200", "TM1"])
    assert full_grid_check(sim, g) == 1.0