"""Pins of the oracle's regression cost model (
DESIGN reading R7) and of the calibration fit.

* With the bytes coefficients at zero, c0 = o and c_flop = 1/F for a
  power-of-two F, the regression model IS the analytic model (flops/F + o is
  then exact and commutes), so every makespan and peak is bit-identical.
* On one device the makespan is the plain sum of op costs, so selecting one
  feature at a time with a unit coefficient turns the makespan into a count
  that is derived here BY HAND from the C.3 / C.4 programs (number of
  MatMul-type / other ops, their FLOPs, the bytes of the tensors they touch).
  A dropped tensor, a tensor counted on the wrong op class or a wrong shape
  changes one of these integers.
* `fit_cost` recovers known coefficients from exact synthetic samples
  (SPEC S:378-380 calibration check) and stays close under noise.
"""
import math

import numpy as np
import pytest

import oracle
import workloads as W


def reg_topo(**coef):
    t = dict(W.TOPOLOGIES["TB200"])
    t["cost_model"] = 1
    for k in W.REGRESSION_KEYS:
        t[k] = float(coef.get(k, 0.0))
    return t


def one_feature(name):
    return reg_topo(**{name: 1.0})


@pytest.mark.parametrize("model", ["mlp_w1", "mlp_1b", "gpt2_small", "gpt2_1_6b", "mlp_1b_1f1b"])
@pytest.mark.parametrize("D,T,P,K", [(1, 1, 1, 1), (2, 2, 2, 4), (1, 4, 4, 8), (4, 1, 2, 2)])
def test_regression_reduces_to_analytic(model, D, T, P, K):
    F = 2.0 ** 50
    an = dict(W.TOPOLOGIES["TB200"], flops_per_s=F)
    rg = reg_topo(mm_c0_s=an["op_overhead_s"], mm_s_per_flop=1.0 / F,
                  ew_c0_s=an["op_overhead_s"], ew_s_per_flop=1.0 / F)
    rg["flops_per_s"] = F
    m = W.MODELS[model]
    B = 64 * D * K
    a = oracle.eval_config(m, an, D, T, P, K, B)
    r = oracle.eval_config(m, rg, D, T, P, K, B)
    assert a["reason"] == r["reason"]
    if a["reason"] & 0x1F == 0:
        assert r["makespan"] == a["makespan"]
        assert r["peak"] == a["peak"]


MLP_CASES = [(2, 64, 64), (3, 128, 32), (8, 256, 16), (5, 8, 3)]


@pytest.mark.parametrize("L,d,m", MLP_CASES)
def test_mlp_feature_counts(L, d, m):
    """One device, one microbatch: C.3 forward MatMul + Relu per layer,
    LossGrad, per layer ReluGrad + MatMulGrad + Add, then SGD per layer.
    MatMul (m,d)x(d,d): 2md^2 FLOPs, tensors act + W + Z = 2md + d^2;
    MatMulGrad: 4md^2 FLOPs, act + W + dZ + dA + dW = 3md + 2d^2;
    Relu md / 2md; ReluGrad md / 3md; Add d^2 / 3d^2; SGD 2d^2 / 3d^2;
    LossGrad 3md / 3md (values of e = 2 bytes)."""
    e = 2
    model = W.mlp(L, d)
    ev = lambda name: oracle.eval_config(model, one_feature(name), 1, 1, 1, 1, m)["makespan"]
    assert ev("mm_c0_s") == 2 * L
    assert ev("ew_c0_s") == 4 * L + 1
    assert ev("mm_s_per_flop") == 6 * L * m * d * d
    assert ev("ew_s_per_flop") == L * (2 * m * d + 3 * d * d) + 3 * m * d
    assert ev("mm_s_per_byte") == L * e * (5 * m * d + 3 * d * d)
    assert ev("ew_s_per_byte") == L * e * (5 * m * d + 6 * d * d) + 3 * m * d * e


GPT_CASES = [(1, 64, 4, 4, 2, 256, 32), (2, 128, 8, 8, 3, 512, 64), (3, 96, 6, 2, 5, 384, 16)]


@pytest.mark.parametrize("L,d,h,S,m,V,nctx", GPT_CASES)
def test_gpt2_feature_counts(L, d, h, S, m, V, nctx):
    """One device, one microbatch of m sequences of S tokens (n = mS).
    Per block (C.4): ln_1, QKV, scores, softmax, context, proj, residual,
    ln_2, FC1, GeLU, FC2, residual; prologue Embed; epilogue ln_f, LM head.
    MatMul-type tensors per block: QKV nd+3d^2+3d+3nd, scores 3nd+mhS^2,
    context mhS^2+3nd+nd, proj nd+d^2+d+nd, FC1 nd+4d^2+4d+4nd, FC2
    4nd+4d^2+d+nd = 23nd + 12d^2 + 9d + 2mhS^2; LM head nd + Vd + nV.
    Others per block: 2x LayerNorm 2nd+2d, softmax 2mhS^2, 2x residual 3nd,
    GeLU 8nd = 18nd + 4d + 2mhS^2; Embed n*8 + Vd + nctx*d + nd; ln_f 2nd+2d."""
    e, ide = 2, 8
    n = m * S
    model = W.gpt2(L, d, h, seq_len=S, vocab_pad=V, n_ctx=nctx)
    ev = lambda name: oracle.eval_config(model, one_feature(name), 1, 1, 1, 1, m)["makespan"]
    assert ev("mm_c0_s") == 6 * L + 1
    assert ev("ew_c0_s") == 6 * L + 2
    mm_flops = L * (2 * n * d * 3 * d + n * 3 * d + 2 * m * S * S * d + 2 * m * S * S * d +
                    2 * n * d * d + n * d + 2 * n * d * 4 * d + n * 4 * d +
                    2 * n * 4 * d * d + n * d) + 2 * n * d * V
    assert ev("mm_s_per_flop") == mm_flops
    ew_flops = L * (5 * n * d + 5 * m * h * S * S + n * d + 5 * n * d + 8 * n * 4 * d + n * d) + \
        2 * n * d + 5 * n * d
    assert ev("ew_s_per_flop") == ew_flops
    mhs = m * h * S * S
    assert ev("mm_s_per_byte") == e * (L * (23 * n * d + 12 * d * d + 9 * d + 2 * mhs) +
                                       n * d + V * d + n * V)
    assert ev("ew_s_per_byte") == (L * e * (18 * n * d + 4 * d + 2 * mhs) +
                                   n * ide + e * (V * d + nctx * d + n * d) + e * (2 * n * d + 2 * d))


def test_gpt2_no_lm_head_drops_one_matmul():
    m = W.gpt2(2, 64, 4, seq_len=4, vocab_pad=256, n_ctx=32, lm_head=0)
    r = oracle.eval_config(m, one_feature("mm_c0_s"), 1, 1, 1, 1, 2)
    assert r["makespan"] == 6 * 2


def test_tensor_parallel_shards_matmul_bytes():
    """T = 2 on an MLP: the per-rank MatMul touches act (m x k_in), the W
    shard and Z (m x n_out); column layers (even) have k_in = d, n_out = d/2,
    row layers (odd) k_in = d/2, n_out = d.  On ranks of stage 0 (P = 1) the
    makespan is the per-rank sum (the TP AllReduces cost 0 here)."""
    L, d, m, e = 2, 64, 8, 2
    t = one_feature("mm_s_per_byte")
    t.update(alpha_intra_s=0.0, bw_intra_Bps=math.inf, alpha_inter_s=0.0, bw_inter_Bps=math.inf)
    r = oracle.eval_config(W.mlp(L, d), t, 1, 2, 1, 1, m)
    col_f = m * d + d * d // 2 + m * d // 2
    row_f = m * d // 2 + d * d // 2 + m * d
    col_b = 2 * m * d + 2 * (d * d // 2) + m * d // 2
    row_b = 2 * m * d // 2 + 2 * (d * d // 2) + m * d
    assert r["makespan"] == e * (col_f + row_f + col_b + row_b)


# ------------------------------------------------------------- the fit -----

def test_fit_recovers_exact_coefficients():
    from paper_2111_05426_b200.calibrate import fit_cost, predict
    rng = np.random.default_rng(518)
    true = (4.5e-6, 1.0 / 1.2e15, 1.0 / 6.5e12)
    f = rng.uniform(1e6, 1e13, 60)
    b = rng.uniform(1e4, 1e10, 60)
    t = predict(true, f, b)
    got = fit_cost(f, b, t)
    for g, w in zip(got, true):
        assert abs(g - w) <= 1e-6 * w


def test_fit_under_noise_and_nonnegative():
    from paper_2111_05426_b200.calibrate import fit_cost, predict
    rng = np.random.default_rng(519)
    true = (8e-6, 1.0 / 9e14, 0.0)
    f = 10.0 ** rng.uniform(6, 13, 200)          # log-uniform: the intercept matters
    b = 10.0 ** rng.uniform(4, 9, 200)
    t = predict(true, f, b) * (1 + 0.01 * rng.standard_normal(200))
    got = fit_cost(f, b, t)
    assert all(c >= 0 for c in got)
    assert abs(got[0] - true[0]) < 0.05 * true[0]
    assert abs(got[1] - true[1]) < 0.05 * true[1]
    p = predict(got, f, b)
    assert np.median(np.abs(p - t) / t) < 0.02
