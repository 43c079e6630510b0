"""Pins of the oracle's memory-saving variants: gradient
checkpointing (Appendix Fig. 8) and ZeRO-2/3 parameter and
gradient partitioning (Fig. 9).  DESIGN readings R8 / R9.

The listings of Figs. 8/9 are stripped from PAPER.md; what survives is each
listing's per-device value list in listing order (the `emph` lists, stored
with their citation in tests/golden/fig8_fig9_values.json) and the prose.
The expected values below come from those lists, the prose, hand traces
(written out in the docstrings), closed forms and the independent
brute-force formulations of oracle.bruteforce -- never from the oracle's
own formulas.
"""
import json
import math
import os

import pytest

import oracle
from oracle import bruteforce as bf
import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden():
    with open(os.path.join(GOLDEN, "fig8_fig9_values.json")) as f:
        return json.load(f)


def dyadic_topo(**over):
    """Dyadic costs (exact sums): F = 2^30, o = 0, alpha = 2^-19,
    bandwidth 2^33 B/s."""
    t = dict(W.TOPOLOGIES["TB200"])
    t.update(flops_per_s=2.0 ** 30, op_overhead_s=0.0, alpha_intra_s=2.0 ** -19,
             bw_intra_Bps=2.0 ** 33, alpha_inter_s=2.0 ** -19, bw_inter_Bps=2.0 ** 33)
    t.update(over)
    return t


COMPUTE, SEND, ALLREDUCE, ALLGATHER, BCAST, REDUCE = range(6)


def _figure_names(model, D, B, L=2, d=64):
    """Per-device lists of the figure-named values the program creates, in
    program order, for a 2-layer MLP with T = P = K = 1 (Figs. 8/9 shapes).
    Ops are classified by their class, arity and FLOPs (F = 2^30, o = 0, so
    cost * 2^30 = FLOPs exactly); names follow the figures: as / p (forward
    Relu outputs of layers 1 / 2), dp (LossGrad), as_b (recomputed), dw<l> /
    das (MatMulGrad), w<l>_<dev>_f / _b (weight copies received), dw<l>
    (reduced gradient), w<l>_new (weight update)."""
    t = dyadic_topo()
    vals, ops = oracle.export_program(model, t, D, 1, 1, 1, B)
    m = B // D
    n = D
    names = [[] for _ in range(n)]
    bwd = [False] * n
    relu_f = [0] * n
    mmg = [0] * n
    sgd = [0] * n
    for devs, cost, ins, outs, cls in ops:
        flops = round(cost * 2.0 ** 30)
        if cls == BCAST:
            src = vals[ins[0]][0]
            layer = src % D          # the owner of layer l is replica l mod D
            for v in outs:
                dv = vals[v][0]
                tag = "b" if bwd[dv] else "f"
                names[dv].append("w%d_%d_%s" % (layer + 1, dv + 1, tag))
            continue
        if cls == REDUCE:
            dv = vals[outs[0]][0]
            names[dv].append("dw%d" % (dv % D + 1))
            continue
        if cls != COMPUTE:
            continue
        dv = devs[0]
        suf = "_%d" % (dv + 1) if D > 1 else ""
        if len(outs) == 2:                                   # MatMulGrad
            layer = L - 1 - mmg[dv]
            mmg[dv] += 1
            names[dv].append("dw%d%s" % (layer + 1, suf))
            if layer > 0:
                names[dv].append("das%s" % suf)
        elif len(ins) == 1:                                  # Relu
            if bwd[dv]:
                names[dv].append("as_b")
            else:
                names[dv].append(("as" if relu_f[dv] == 0 else "p") +
                                 ("_f" if D == 1 and relu_f[dv] == 0 else suf))
                relu_f[dv] += 1
        elif flops == 3 * m * d:                             # LossGrad
            names[dv].append("dp%s" % suf)
            bwd[dv] = True
        elif vals[outs[0]][3]:                               # SGD (returned)
            layer = dv % D if D > 1 else sgd[dv]
            sgd[dv] += 1
            names[dv].append("w%d_new" % (layer + 1))
    return names


def test_fig8_checkpointing_value_order():
    """Fig. 8 (P:858 value list, P:974 prose): sequential training of a
    2-layer MLP with gradient checkpointing creates, in order, as_f, p, dp,
    as_b, dw2, das, dw1, w1_new, w2_new -- the recompute (as_b) follows the
    loss gradient and precedes the second layer's gradients."""
    g = _golden()
    model = W.mlp(2, 64, recompute=1)
    names = _figure_names(model, 1, 32)
    expect = [v for v in g["fig8_values_device1"] if v not in g["fig8_params"]]
    assert names[0] == expect


def test_fig8_as_f_discarded_after_p():
    """"the first activation (as_f) is discarded after line p": its
    last use is the forward MatMul of layer 2, so it is freed before the
    loss gradient; the recomputed as_b is a different value."""
    t = dyadic_topo()
    vals, ops = oracle.export_program(W.mlp(2, 64, recompute=1), t, 1, 1, 1, 1, 32)
    relus = [i for i, o in enumerate(ops) if o[4] == COMPUTE and len(o[2]) == 1]
    as_f, as_b = ops[relus[0]][3][0], ops[relus[2]][3][0]
    users = [i for i, o in enumerate(ops) if as_f in o[2]]
    loss = [i for i, o in enumerate(ops) if o[4] == COMPUTE and round(o[1] * 2 ** 30) == 3 * 32 * 64]
    assert len(users) == 1 and users[0] < relus[1] < loss[0]
    assert as_b != as_f and all(i > loss[0] for i, o in enumerate(ops) if as_b in o[2])


def test_fig9_zero_value_order_and_ownership():
    """Fig. 9 (P:894-897 value lists, P:976 prose), data parallelism over 2
    devices with ZeRO: per device, the program creates exactly the figure's
    values in the figure's order -- weight copies received before their
    forward (w2_1_f) and backward (w2_1_b, w1_2_b) use, gradients reduced to
    the owner (dw1 on device 1, dw2 on device 2) -- and each device holds
    only its own layer's weight as a parameter."""
    g = _golden()
    model = W.mlp(2, 64, zero=1)
    names = _figure_names(model, 2, 64)
    for dv, key in enumerate(["fig9_values_device1", "fig9_values_device2"]):
        expect = [v for v in g[key] if v not in g["fig9_params"]]
        assert names[dv] == expect, (dv, names[dv])
    vals, ops = oracle.export_program(model, dyadic_topo(), 2, 1, 1, 1, 64)
    w_bytes = 64 * 64 * 2
    for dv in range(2):
        params = [b for (dev, b, p, r) in vals if p and dev == dv]
        # X_k, Y_k (32 x 64 x 2 each) + W_l and its gradient buffer (C.9 A20)
        assert sorted(params) == sorted([32 * 64 * 2] * 2 + [w_bytes] * 2)


def test_fig9_timeline_hand_derivation():
    """Fig. 9 timeline with dyadic costs (exact).  Both devices run the same
    ops up to the reduce of dw1 (X, below); the Bcast / Reduce collectives
    synchronise them; the owner-only Add / SGD then differ:
      X = 4 c_B + 2 c_MM + 2 c_R + c_LG + 2 c_RG + 2 c_MMG + c_Red
      dev 1: X + c_Add(dw1) + c_Red(dw2 waits for dev 1's Add) + c_SGD
      dev 2: X + c_Add + c_Red + c_Add(dw2) + c_SGD  (the makespan).
    Op costs are the C.5 values (FLOPs / F for compute, g = 2 collectives are
    a Send: alpha + bytes / bw)."""
    t = dyadic_topo()
    m, d, e = 32, 64, 2
    F, a, bw = t["flops_per_s"], t["alpha_intra_s"], t["bw_intra_Bps"]
    c_MM, c_R, c_LG = 2 * m * d * d / F, m * d / F, 3 * m * d / F
    c_RG, c_MMG, c_Add, c_SGD = m * d / F, 4 * m * d * d / F, d * d / F, 2 * d * d / F
    c_B = c_Red = a + d * d * e / bw
    X = 4 * c_B + 2 * c_MM + 2 * c_R + c_LG + 2 * c_RG + 2 * c_MMG + c_Red
    r = oracle.eval_config(W.mlp(2, 64, zero=1), t, 2, 1, 1, 1, 64)
    assert r["clocks"].tolist() == [X + c_Add + c_Red + c_SGD,
                                    X + c_Add + c_Red + c_Add + c_SGD]
    assert r["makespan"] == X + 2 * c_Add + c_Red + c_SGD


def test_fig8_hand_trace_peak_and_sum():
    """Fig. 8 shape on W1 (d = 64, B = 64, e = 2: every tensor u = 8192 B),
    one device.  Params W0 W1 G0 G1 X Y = 6u.  Forward: MatMul0 +Z (7u),
    Relu0 +A1 (8u) -Z; MatMul1 +Z' (8u) -A1 (as_f dies); Relu1 +A2
    (8u) -Z' -> 7u.  LossGrad +dA2 (8u) -Y; recompute MatMul0 +Zb (8u),
    Relu0 +A1b (9u = peak) -Zb; ReluGrad1 +dZ1 (9u) -A2 -dA2; MatMulGrad1
    +dA1 +dW1 (9u) -dZ1; Add1 +G1' (9u) -G1 -dW1; ReluGrad0 +dZ0 -A1b -dA1;
    MatMulGrad0 +dA0 +dW0 -X -dZ0 -dA0; Add0; SGD0; SGD1 -> final live
    W0' + W1' = 2u.  Peak 9u = 73,728 B; 13 + 2 recompute ops = 15 ops;
    one device, so the makespan is the sequential sum: FLOPs 3,198,976 (P2)
    + 2 * 64^3 + 64^2 = 3,727,360, with F = 1e12 and o = 5e-6:
    3.72736e-06 + 15 * 5e-06 = 7.872736e-05 s."""
    model = W.mlp(2, 64, recompute=1)
    t = dict(W.TOPOLOGIES["TB200"], flops_per_s=1e12)
    r = oracle.eval_config(model, t, 1, 1, 1, 1, 64)
    assert r["n_ops"] == 15 and r["peak"] == 73728
    assert r["makespan"] == pytest.approx(7.872736e-05, rel=1e-12)
    ops = oracle.program_ops(model, t, 1, 1, 1, 1, 64)
    assert int(ops["work"].sum()) == 3727360
    vals, ops = oracle.export_program(model, t, 1, 1, 1, 1, 64)
    raw = oracle.simulate_raw(1, [(o[0], o[1], o[2], o[3]) for o in ops], vals)
    assert raw["live"][0] == 16384 and raw["peak"][0] == 73728


@pytest.mark.parametrize("T,P,K,L", [(1, 1, 1, 2), (2, 1, 2, 4), (1, 2, 4, 4),
                                     (2, 4, 2, 8), (4, 2, 3, 5)])
def test_zero_with_one_replica_is_the_baseline(T, P, K, L):
    """ZeRO partitions over the data-parallel replicas: with D = 1 the owner
    is the only replica and the program is the baseline's (C.3)."""
    t = W.TOPOLOGIES["TB200"]
    for sched in (0, 1):
        a = oracle.eval_config(W.mlp(L, 64, schedule=sched), t, 1, T, P, K, 64 * K)
        b = oracle.eval_config(W.mlp(L, 64, schedule=sched, zero=1), t, 1, T, P, K, 64 * K)
        assert (a["makespan"], a["peak"], a["n_ops"]) == (b["makespan"], b["peak"], b["n_ops"])


@pytest.mark.parametrize("D,T,P,K", [(1, 1, 2, 2), (2, 2, 4, 3), (2, 1, 8, 4)])
def test_checkpointing_one_layer_per_stage_is_the_baseline(D, T, P, K):
    """A stage keeps its input and output activations (Fig. 8 keeps x and
    p); with one layer per stage nothing is recomputed."""
    t = W.TOPOLOGIES["TB200"]
    a = oracle.eval_config(W.mlp(P, 64), t, D, T, P, K, 64 * D * K)
    b = oracle.eval_config(W.mlp(P, 64, recompute=1), t, D, T, P, K, 64 * D * K)
    assert (a["makespan"], a["peak"], a["n_ops"]) == (b["makespan"], b["peak"], b["n_ops"])


def test_checkpointing_never_raises_the_peak():
    """Gradient checkpointing is a memory-saving optimisation: over
    a sweep of small configurations the checkpointed peak never exceeds the
    baseline's, and with many microbatches of a deep stage it is lower
    (GPipe keeps K microbatches x L layers of activations; checkpointing
    only K stage inputs and outputs)."""
    t = W.TOPOLOGIES["TB200"]
    for L in (3, 4, 6):
        for D, T, P, K in [(1, 1, 1, 1), (1, 1, 1, 4), (2, 1, 1, 2), (1, 2, 1, 2),
                           (1, 1, 2, 4), (2, 2, 2, 2), (1, 2, 3, 3)]:
            for sched in (0, 1):
                a = oracle.eval_config(W.mlp(L, 64, schedule=sched), t, D, T, P, K, 64 * D * K)
                b = oracle.eval_config(W.mlp(L, 64, schedule=sched, recompute=1), t, D, T, P,
                                       K, 64 * D * K)
                assert b["peak"] <= a["peak"], (L, D, T, P, K, sched)
                assert b["makespan"] >= a["makespan"]     # recompute costs time
    a = oracle.eval_config(W.mlp(8, 64), t, 1, 1, 1, 8, 64 * 8)
    b = oracle.eval_config(W.mlp(8, 64, recompute=1), t, 1, 1, 1, 8, 64 * 8)
    assert b["peak"] < a["peak"]


@pytest.mark.parametrize("D,T,P,K,L", [(2, 1, 1, 1, 2), (2, 2, 2, 2, 4), (4, 1, 2, 3, 6),
                                       (4, 2, 1, 2, 5), (8, 1, 2, 2, 8)])
def test_zero_parameter_bytes_partitioned(D, T, P, K, L):
    """parameters and gradients are partitioned over the replicas:
    rank (i, j, s) holds W_l and its gradient buffer only for the layers l of
    its stage with l mod D = i, so over the D replicas of a (j, s) group the
    weight bytes add up to one baseline replica's, and each holds ~1/D."""
    t = W.TOPOLOGIES["TB200"]
    B = 64 * D * K
    vb, _ = oracle.export_program(W.mlp(L, 64), t, D, T, P, K, B)
    vz, _ = oracle.export_program(W.mlp(L, 64, zero=1), t, D, T, P, K, B)
    n = D * T * P
    base = [sum(b for (dv, b, p, r) in vb if p and dv == x) for x in range(n)]
    zero = [sum(b for (dv, b, p, r) in vz if p and dv == x) for x in range(n)]
    m = B // (D * K)
    for s in range(P):
        lo, hi = s * L // P, (s + 1) * L // P
        for j in range(T):
            ranks = [j + T * (i + D * s) for i in range(D)]
            # X_k (m x d) on stage 0, Y_k (m x d_out of the last layer: d / T
            # for a column-parallel last layer) on stage P-1
            d_last = 64 // T if (T > 1 and (L - 1) % 2 == 0) else 64
            io = (K * m * 64 * 2 if s == 0 else 0) + (K * m * d_last * 2 if s == P - 1 else 0)
            wsum = sum(zero[r] - io for r in ranks)
            assert wsum == base[ranks[0]] - io
            for i, r in enumerate(ranks):
                mine = [l for l in range(lo, hi) if l % D == i]
                # W_l + G_l, each d x d / T elements of 2 bytes (col or row shard)
                assert zero[r] - io == len(mine) * 2 * (64 * 64 // T) * 2


@pytest.mark.parametrize("D,T,P,K,L", [(1, 1, 1, 1, 2), (2, 1, 1, 1, 2), (2, 2, 2, 2, 4),
                                       (4, 1, 2, 3, 6), (1, 2, 4, 2, 9), (2, 4, 2, 2, 5)])
def test_f4_op_count_closed_forms(D, T, P, K, L):
    """Op counts from the structure of the variants (a collective counts
    once).  Checkpointing adds, per microbatch and stage, the forward of
    every layer but the stage's last (MatMul + Relu per rank, a TP AllReduce
    per replica for row layers when T > 1).  ZeRO (D > 1) adds per
    microbatch and layer a Broadcast per TP index before the forward, one
    before the backward (and one per recomputed layer) and a Reduce after
    it; Adds and SGDs run on the owner only and the DP AllReduce is gone."""
    t = W.TOPOLOGIES["TB200"]
    B = 64 * D * K
    base = (5 * K * D * T * L + D * T * L + K * D * T + (T > 1) * K * D * L
            + 2 * K * D * T * (P - 1) + (D > 1) * T * L)
    stage_last = {(s + 1) * L // P - 1 for s in range(P)}
    recomputed = [l for l in range(L) if l not in stage_last]
    rows = sum(1 for l in recomputed if l % 2 == 1)
    ck = K * (2 * D * T * len(recomputed) + (T > 1) * D * rows)
    r = oracle.eval_config(W.mlp(L, 64, recompute=1), t, D, T, P, K, B)
    assert r["n_ops"] == base + ck
    if D > 1:
        z = (base - (D - 1) * K * T * L - (D - 1) * T * L - T * L + 3 * K * T * L)
        r = oracle.eval_config(W.mlp(L, 64, zero=1), t, D, T, P, K, B)
        assert r["n_ops"] == z
        r = oracle.eval_config(W.mlp(L, 64, zero=1, recompute=1), t, D, T, P, K, B)
        assert r["n_ops"] == z + ck + K * T * len(recomputed)


def _f4_cases():
    out = []
    for (rc, z) in [(1, 0), (0, 1), (1, 1)]:
        for sched in (0, 1):
            for D, T, P, K, L in [(1, 1, 1, 1, 3), (2, 1, 1, 2, 2), (2, 2, 2, 2, 4),
                                  (4, 1, 2, 2, 5), (2, 1, 3, 3, 6), (1, 2, 2, 3, 4)]:
                out.append((W.mlp(L, 32, schedule=sched, recompute=rc, zero=z), D, T, P, K,
                            8 * D * K))
    return out


@pytest.mark.parametrize("case", range(len(_f4_cases())))
def test_f4_programs_bruteforce(case):
    """P7 on the variant programs: the walk equals the per-device
    co-simulation (P:471 + rendezvous) and per-device peaks equal
    live-interval stabbing, both independent formulations."""
    model, D, T, P, K, B = _f4_cases()[case]
    t = W.TOPOLOGIES["TB200"]
    r = oracle.eval_config(model, t, D, T, P, K, B)
    vals, ops = oracle.export_program(model, t, D, T, P, K, B)
    n = D * T * P
    assert bf.cosimulate(n, ops)[2] == r["makespan"]
    assert bf.interval_peaks(n, ops, vals) == r["peaks"].tolist()


@pytest.mark.parametrize("D,T,P,K,L", [(1, 1, 2, 2, 4), (1, 1, 4, 8, 8), (2, 1, 2, 3, 4),
                                       (1, 2, 2, 5, 4), (2, 2, 4, 4, 8)])
def test_checkpointing_gpipe_flowshop(D, T, P, K, L):
    """P3 with checkpointing: with zero-cost communication a stage's
    backward per microbatch is its recompute plus its layer gradients (B'),
    and GPipe is still the identical-jobs flow shop: (P-1+K)(F+B') + K g +
    tail_0.  Per-op costs are read from a 1-stage
    checkpointed program of the same layer shapes (dyadic: exact)."""
    t = dict(dyadic_topo(), op_overhead_s=2.0 ** -20, alpha_intra_s=0.0, bw_intra_Bps=math.inf,
             alpha_inter_s=0.0, bw_inter_Bps=math.inf)
    d, m, nl = 64, 16, L // P
    one = oracle.program_ops(W.mlp(nl, d, recompute=1), t, 1, T, 1, 1, m)
    costs = [c for c, d0, cl in zip(one["cost"], one["dev0"], one["cls"]) if d0 == 0 or cl != 0]
    nfwd = sum(3 if (T > 1 and l % 2 == 1) else 2 for l in range(nl))
    F = sum(costs[:nfwd])
    g = costs[nfwd]
    rest = costs[nfwd + 1:]
    Bp = sum(rest[:len(rest) - nl])
    tail = sum(rest[len(rest) - nl:])
    r = oracle.eval_config(W.mlp(L, d, recompute=1), t, D, T, P, K, m * D * K)
    assert r["makespan"] == (P - 1 + K) * (F + Bp) + K * g + tail
