"""Pins of the oracle's synchronous 1F1B schedule (
DESIGN reading R6).

* Fig. 2/3 is the paper's own 1F1B program for a 2-layer MLP on
  2 devices with 2 microbatches.  Its per-device op order (Splits dropped,
  WU = SGD) must be exactly the oracle's: device 1 runs as_1, ar_1, as_2,
  ar_2, dar_1, dw1_1, dar_2, dw1_2, WU; device 2 runs ar_1, p_1, ar_2, dp_1,
  dw2_1, dar_1, p_2, dp_2, dw2_2, dar_2, WU.
* With zero-cost communication 1F1B has the same makespan as GPipe (both
  (P-1+K)(F+B) + K*g + tail for uniform stages), exactly with
  dyadic costs.
* 1F1B never needs more memory than GPipe (fewer microbatches in flight).
* Its global order is deadlock-free: the per-device co-simulation of the
  projected per-rank programs completes and equals the walk.
"""
import math

import pytest

import oracle
from oracle import bruteforce as bf
import workloads as W


def dyadic_topo():
    t = dict(W.TOPOLOGIES["TB200"])
    t.update(flops_per_s=2.0 ** 30, op_overhead_s=2.0 ** -20, alpha_intra_s=0.0,
             bw_intra_Bps=math.inf, alpha_inter_s=0.0, bw_inter_Bps=math.inf)
    return t


def device_pattern(ops, dev):
    return "".join("S" if o[4] == 1 else "C" for o in ops if dev in o[0])


def test_fig3_program_order():
    """Our MLP ops per task: forward = MatMul, Relu (CC); backward on the last
    stage = LossGrad, ReluGrad, MatMulGrad, Add (CCCC), elsewhere CCC; the
    weight update = SGD (C).  Reading Fig. 3's event order with these sizes
    gives the two patterns below."""
    _, ops = oracle.export_program(W.mlp(2, 64, schedule=1), W.TOPOLOGIES["TB200"],
                                   1, 1, 2, 2, 64)
    # device 1: as_1 ar_1 as_2 ar_2 dar_1 dw1_1 dar_2 dw1_2 WU
    assert device_pattern(ops, 0) == "CC" "S" "CC" "S" "S" "CCC" "S" "CCC" "C"
    # device 2: ar_1 p_1 ar_2 dp_1+dw2_1 dar_1 p_2 dp_2+dw2_2 dar_2 WU
    assert device_pattern(ops, 1) == "S" "CC" "S" "CCCC" "S" "CC" "CCCC" "S" "C"


@pytest.mark.parametrize("D,T,P,K,L", [
    (1, 1, 2, 2, 4), (1, 1, 4, 8, 8), (2, 1, 2, 3, 4), (1, 2, 2, 5, 4),
    (2, 2, 4, 4, 8), (1, 1, 8, 16, 8), (1, 1, 4, 2, 8), (1, 1, 2, 1, 2),
    (1, 1, 16, 32, 16)])
def test_zero_comm_makespan_equals_gpipe(D, T, P, K, L):
    t = dyadic_topo()
    g = oracle.eval_config(W.mlp(L, 64), t, D, T, P, K, 16 * D * K)
    f = oracle.eval_config(W.mlp(L, 64, schedule=1), t, D, T, P, K, 16 * D * K)
    assert f["makespan"] == g["makespan"]


@pytest.mark.parametrize("D,T,P,K", [(1, 1, 2, 8), (1, 2, 4, 16), (2, 1, 8, 32),
                                     (1, 1, 4, 3), (2, 2, 2, 1)])
def test_peak_not_above_gpipe(D, T, P, K):
    for t in [W.TOPOLOGIES["TB200"], W.TOPOLOGIES["TV100"]]:
        g = oracle.eval_config(W.MODELS["mlp_1b"], t, D, T, P, K, 64 * D * K)
        f = oracle.eval_config(W.MODELS["mlp_1b_1f1b"], t, D, T, P, K, 64 * D * K)
        assert f["peak"] <= g["peak"]
        if K > P:
            assert f["peak"] < g["peak"]


@pytest.mark.parametrize("P,K", [(2, 3), (3, 5), (4, 4), (4, 9), (5, 2), (6, 7)])
def test_deadlock_free_and_cosimulation(P, K):
    m = W.mlp(max(P, 6), 32, schedule=1)
    t = W.TOPOLOGIES["TM0"]
    vals, ops = oracle.export_program(m, t, 1, 2, P, K, 4 * K)
    r = oracle.eval_config(m, t, 1, 2, P, K, 4 * K)
    n = 2 * P
    assert bf.cosimulate(n, ops)[2] == r["makespan"]
    assert bf.interval_peaks(n, ops, vals) == r["peaks"].tolist()


def test_op_count_unchanged():
    """1F1B reorders the GPipe program; it has the same ops."""
    for (D, T, P, K) in [(1, 1, 2, 2), (2, 2, 4, 8), (1, 4, 2, 3)]:
        g = oracle.eval_config(W.mlp(8, 64), W.TOPOLOGIES["TB200"], D, T, P, K, 8 * D * K)
        f = oracle.eval_config(W.mlp(8, 64, schedule=1), W.TOPOLOGIES["TB200"], D, T, P, K,
                               8 * D * K)
        assert f["n_ops"] == g["n_ops"]
