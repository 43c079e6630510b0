"""Pins of the CPU oracle against what the paper and mathematics fix.

Each test names the passage (P:<line> = PAPER.md, S:<line> = SPEC.md,
SURVEY C.10 pin id).  None of them retypes the oracle's own formulas: the
expected values are the paper's printed numbers, closed forms from textbook
results, independent brute-force formulations (oracle.bruteforce), or
invariants that any correct simulator must satisfy.
"""
import json
import math
import os
import random

import numpy as np
import pytest

import oracle
from oracle import bruteforce as bf
import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def dyadic_topo(**over):
    """A topology whose costs are dyadic rationals, so every sum in a
    makespan is exact in binary64 and closed forms can be compared with ==."""
    t = dict(W.TOPOLOGIES["TB200"])
    t.update(flops_per_s=2.0 ** 30, op_overhead_s=2.0 ** -20,
             alpha_intra_s=0.0, bw_intra_Bps=math.inf, alpha_inter_s=0.0,
             bw_inter_Bps=math.inf)
    t.update(over)
    return t


# ------------------------------------------------------------ P1, P11 -------

def _fig3():
    with open(os.path.join(GOLDEN, "fig3_trace.json")) as f:
        g = json.load(f)
    top = [(e[1], float(e[2])) for e in g["events_top"]]
    names = [e[0] for e in g["events_top"]]
    i, j = names.index(g["swap"][0]), names.index(g["swap"][1])
    swapped = list(top)
    swapped[i], swapped[j] = swapped[j], swapped[i]
    return g, names, top, swapped, i, j


def test_fig3_pipeline_trace_makespans():
    """P1: Fig. 3 -- @mlpPP and its swapped variant."""
    g, names, top, swapped, i, j = _fig3()
    a = oracle.simulate_raw(2, top)
    b = oracle.simulate_raw(2, swapped)
    assert a["makespan"] == g["derived_makespan_top"] == 88
    assert b["makespan"] == g["derived_makespan_swapped"] == 94
    assert max(a["makespan"], b["makespan"]) <= g["axis_max"]
    st = dict(zip(names, a["start"]))
    # Splits in parallel; as_1 then ar_1 in sequence;
    # as_2 and p_1 simultaneously.
    assert st["x_1"] == st["y_1"] == 0
    assert st["ar_1"] == a["end"][names.index("as_1")]
    assert st["as_2"] == st["p_1"] == 17
    # swapped, the Send ar_2 blocks p_1 on device 2 (starts at 29).
    sw_names = list(names)
    sw_names[i], sw_names[j] = sw_names[j], sw_names[i]
    stb = dict(zip(sw_names, b["start"]))
    enb = dict(zip(sw_names, b["end"]))
    assert stb["p_1"] == enb["ar_2"] == 29


@pytest.mark.parametrize("c", [0.0, 1e-9, 0.5, 3.0, 6.0, 100.0])
def test_fig3_swap_penalty_any_send_cost(c):
    """P11: whatever the Send cost, swapping p_1 and ar_2 costs
    exactly one p_1 duration (6) more."""
    g, names, top, swapped, i, j = _fig3()
    re = lambda prog: [(d, c if len(d) == 2 else t) for d, t in prog]
    a = oracle.simulate_raw(2, re(top))["makespan"]
    b = oracle.simulate_raw(2, re(swapped))["makespan"]
    assert b - a == pytest.approx(6.0, rel=0, abs=1e-12 * max(1.0, b))


# ------------------------------------------------------------------ P10 -----

def test_cost_examples_from_paper_and_spec():
    """P10: "Add's cost ... returns N/f"; S:369-371 examples."""
    t = dict(W.TOPOLOGIES["TB200"], flops_per_s=1e9, op_overhead_s=0.0)
    # Relu over N = m*d = 10*100 = 1000 elements at f = 1e9 -> 1e-6 s.
    ops = oracle.program_ops(W.mlp(1, 100), t, 1, 1, 1, 1, 10)
    relu = [c for w, c in zip(ops["work"], ops["cost"]) if w == 1000]
    assert relu and relu[0] == 1e-6
    # Send of 1e6 bytes (m*d*e = 500*1000*2) at bw 1e9, alpha 1e-5 ->
    # 1.01e-3 s.
    t2 = dict(t, alpha_intra_s=1e-5, bw_intra_Bps=1e9, node_size=8)
    ops = oracle.program_ops(W.mlp(2, 1000), t2, 1, 1, 2, 1, 500)
    sends = ops["cost"][ops["cls"] == 1]
    assert len(sends) == 2 and sends[0] == pytest.approx(1.01e-3, rel=1e-15)
    # MatMul (64,64)x(64,64) at 1e12 -> 2*64^3/1e12 = 5.24288e-7.
    t3 = dict(t, flops_per_s=1e12)
    ops = oracle.program_ops(W.mlp(1, 64), t3, 1, 1, 1, 1, 64)
    mm = ops["cost"][ops["work"] == 2 * 64 ** 3]
    assert mm[0] == pytest.approx(5.24288e-7, rel=1e-15)
    # Ring all-reduce over g = 2: 2*alpha + bytes/bw (2(g-1)/g = 1).
    t4 = dict(t, alpha_intra_s=1e-5, bw_intra_Bps=1e9, node_size=8)
    ops = oracle.program_ops(W.mlp(1, 64), t4, 2, 1, 1, 1, 128)
    ar = ops["cost"][ops["cls"] == 2]
    assert ar[0] == pytest.approx(2e-5 + 64 * 64 * 2 / 1e9, rel=1e-15)


# ------------------------------------------------------------------- P2 -----

def test_one_rank_is_sequential_sum():
    """P2 (north_star): with D = T = P = 1 the makespan is the
    sequential sum of the op costs.  W1 (1,1,1,1) has 13 ops and
    sum FLOPs = 2*(2*64^3 + 3*64^2 + 4*64^3) + 3*64^2 + 2*2*64^2 = 3,198,976
    (hand count of the training step of a 2-layer MLP), so with F = 1e12 and
    o = 5e-6 the makespan is 3,198,976/1e12 + 13*5e-6 = 6.8198976e-05 s."""
    t = dict(W.TOPOLOGIES["TB200"], flops_per_s=1e12)
    ops = oracle.program_ops(W.MODELS["mlp_w1"], t, 1, 1, 1, 1, 64)
    assert len(ops["work"]) == 13
    assert int(ops["work"].sum()) == 3198976
    r = oracle.eval_config(W.MODELS["mlp_w1"], t, 1, 1, 1, 1, 64)
    assert r["makespan"] == pytest.approx(6.8198976e-05, rel=1e-12)
    # exact with dyadic costs: F = 2^30, o = 2^-20
    td = dyadic_topo()
    r = oracle.eval_config(W.MODELS["mlp_w1"], td, 1, 1, 1, 1, 64)
    assert r["makespan"] == 3198976 / 2.0 ** 30 + 13 * 2.0 ** -20


# ------------------------------------------------------------------- P3 -----

def _stage_phase_costs(model, t, D, T, P, K, B):
    """Per-stage costs of the first microbatch read off the oracle's program
    (forward ops of k = 0 and backward ops of k = 0, by device)."""
    ops = oracle.program_ops(model, t, D, T, P, K, B)
    return ops


@pytest.mark.parametrize("D,T,P,K,L", [
    (1, 1, 2, 2, 4), (1, 1, 4, 8, 8), (2, 1, 2, 3, 4), (1, 2, 2, 5, 4),
    (2, 2, 4, 4, 8), (1, 4, 2, 8, 8), (1, 1, 8, 16, 8), (2, 1, 4, 1, 8)])
def test_gpipe_training_flowshop_closed_form(D, T, P, K, L):
    """P3: with zero-cost communication and uniform
    stages, GPipe training is a permutation flow shop with identical jobs:
    makespan = (P - 1 + K) * (F + B) + K * g + tail_0, where F (B) is a
    stage's forward (backward) time per microbatch, g the LossGrad time and
    tail_0 stage 0's weight-update time.  The per-op costs are read from a
    1-stage program of the same layer shapes; costs are dyadic (exact)."""
    t = dyadic_topo()
    d = 64
    m = 16
    model = W.mlp(L, d)
    # one stage, one microbatch, one replica: the ops of a single stage of
    # L/P layers, in order: fwd (MatMul, [AR], Relu) * layers,
    # LossGrad, bwd (ReluGrad, MatMulGrad, [AR], Add) * layers, SGD * layers.
    one = oracle.program_ops(W.mlp(L // P, d), t, 1, T, 1, 1, m)
    # only rank 0's ops, comm costs are exactly zero
    mine = [(w, c) for w, c, d0, cl in zip(one["work"], one["cost"],
                                           one["dev0"], one["cls"])
            if d0 == 0 or cl != 0]
    costs = [c for _, c in mine]
    nl = L // P
    per_fwd = 3 if T > 1 else 2
    nfwd = sum(per_fwd if (T > 1 and l % 2 == 1) else 2 for l in range(nl))
    # forward: MatMul + Relu per layer, AR after odd (row) layers when T > 1
    F = sum(costs[:nfwd])
    g = costs[nfwd]
    rest = costs[nfwd + 1:]
    B = sum(rest[:len(rest) - nl])
    tail = sum(rest[len(rest) - nl:])
    expect = (P - 1 + K) * (F + B) + K * g + tail
    r = oracle.eval_config(model, t, D, T, P, K, m * D * K)
    assert r["makespan"] == expect


@pytest.mark.parametrize("D,T,P,K,L", [
    (1, 1, 2, 4, 4), (1, 1, 4, 8, 6), (2, 2, 2, 3, 5), (1, 2, 4, 16, 12),
    (1, 1, 3, 7, 7)])
def test_gpipe_inference_flowshop(D, T, P, K, L):
    """P3, forward only (GPT-2 inference): with zero-cost communication the
    makespan is the flow-shop value sum_s F_s + (K - 1) max_s F_s for
    arbitrary (non-uniform) stage times F_s.  F_s is read
    from the oracle's own 1-stage programs of each stage's block count."""
    t = dyadic_topo()
    base = dict(W.MODELS["gpt2_small"], n_layer=L)
    m = 2
    times = []
    for s in range(P):
        nb = (s + 1) * L // P - s * L // P
        # stage s alone: blocks + prologue (s == 0) + epilogue (s == P-1)
        ops = oracle.program_ops(dict(base, n_layer=max(nb, 1)), t, 1, T, 1,
                                 1, m)
        ct = [c for c, cl, d0 in zip(ops["cost"], ops["cls"], ops["dev0"])
              if cl == 0 and d0 == 0]
        # ops per block on one rank: 12 compute; prologue 1; epilogue 2
        pro, epi = 1, 2
        blk = ct[pro:pro + 12 * nb]
        Fs = sum(blk)
        if s == 0:
            Fs += sum(ct[:pro])
        if s == P - 1:
            Fs += sum(ct[pro + 12 * nb:])
        times.append(Fs)
    r = oracle.eval_config(base, t, D, T, P, K, m * D * K)
    assert r["makespan"] == pytest.approx(bf.gpipe_flowshop(times, K),
                                          rel=1e-13)


# ------------------------------------------------------------------- P4 -----

def test_grid_counts_table1():
    """P4: Table 1 N_grid = 75 for W = 16 at one batch;
    9 for W = 2 and 1 for W = 1; 155 for W <= 16."""
    g = W.grid(["mlp_1b"], ["TV100"], [16], [65536])
    assert len(oracle.enumerate_grid(g)) == 75
    assert len(oracle.enumerate_grid(dict(g, world=[2]))) == 9
    assert len(oracle.enumerate_grid(dict(g, world=[1]))) == 1
    assert len(oracle.enumerate_grid(dict(g, world=[1, 2, 4, 8, 16]))) == 155


def test_grid_counts_gpt2_1035():
    """P4: Table 1 GPT-2 rows N_grid = 1035 with batch swept over
    2^7..2^20: 1050 tuples of which D*K | B holds for 1035."""
    g = W.GRIDS["PG"]
    f = oracle.enumerate_grid(g)
    assert len(f) == 3 * 1050
    rs = oracle.grid_validity(g)
    for mi in range(3):
        sel = rs[f[:, 0] == mi]
        assert int(((sel & 1) == 0).sum()) == 1035


def test_enumeration_matches_exhaustive_search():
    """P7(iii): the canonical index order equals exhaustive search over all
    integer triples, sorted lexicographically."""
    for name in ["W1", "W2", "W3", "W4", "PM_1B"]:
        g = W.GRIDS[name]
        f = oracle.enumerate_grid(g)
        brute = bf.enumerate_bruteforce(g)
        assert [tuple(x) for x in f[:, :8].tolist()] == brute, name


def test_workload_sizes():
    """SURVEY §8d D.1 counts: W1 20/18, W2 1860/1839, W3 8680/7104, W4 56/56."""
    for name, n, nv in [("W1", 20, 18), ("W2", 1860, 1839),
                        ("W3", 8680, 7104), ("W4", 56, 56)]:
        rs = oracle.grid_validity(W.GRIDS[name])
        assert len(rs) == n and int((rs == 0).sum()) == nv, name


# ------------------------------------------------------------- P5, P9 -------

@pytest.mark.parametrize("name,gb", [("mlp_1b", 2.2), ("mlp_17b", 34.4),
                                     ("mlp_103b", 206.2)])
def test_mlp_parameter_bytes_table1(name, gb):
    """P5: Table 1 model sizes at 16-bit.  The oracle's
    1-rank program holds W_l and G_l (same size) per layer plus X and Y
    (m x d each): weight bytes = (params - 2*m*d*e) / 2."""
    model = W.MODELS[name]
    vals, ops = oracle.export_program(model, dyadic_topo(capacity=1 << 62),
                                      1, 1, 1, 1, 1)
    pbytes = sum(v[1] for v in vals if v[2])
    wbytes = (pbytes - 2 * 1 * model["d_model"] * 2) // 2
    assert wbytes == model["n_layer"] * model["d_model"] ** 2 * 2
    # Table 1 prints the size rounded UP to 0.1 GB: 2.147 -> 2.2,
    # 34.36 -> 34.4, 206.16 -> 206.2 (the only rounding consistent with all
    # three rows).
    assert math.ceil(wbytes / 1e8) / 10 == gb


def test_weight_sharding_one_over_tp():
    """P5: a rank holds exactly 1/(T*P) of the weights when P | L."""
    model = W.MODELS["mlp_1b"]
    for (T, P) in [(2, 1), (4, 2), (1, 4), (16, 1), (2, 8)]:
        vals, _ = oracle.export_program(model, dyadic_topo(capacity=1 << 62),
                                        1, T, P, 1, 1)
        # weights + grads on rank 0, minus X (m x d on stage 0) and, when
        # P = 1, Y (m x d: the last layer is row-parallel or full)
        p0 = sum(v[1] for v in vals if v[2] and v[0] == 0) - 8192 * 2 * (
            1 + (P == 1))
        assert p0 // 2 == 16 * 8192 ** 2 * 2 // (T * P)


def test_capacity_facts_table2():
    """P9: Table 2 '-' entries: MLP 17B with T*P = 1 holds 32 GiB
    of weights plus as much gradient -> over the 32 GiB V100 limit;
    MLP 103B with T*P <= 4 holds >= 48 GiB of weights -> infeasible."""
    tv = W.TOPOLOGIES["TV100"]
    r = oracle.eval_config(W.MODELS["mlp_17b"], tv, 16, 1, 1, 1, 65536)
    assert r["reason"] == 1 << 5 and r["peak"] > tv["capacity_bytes"]
    for (D, T, P, K) in [(4, 4, 1, 1), (4, 1, 4, 2), (4, 2, 2, 2)]:
        r = oracle.eval_config(W.MODELS["mlp_103b"], tv, D, T, P, K, 256)
        assert r["reason"] == 1 << 5


# ------------------------------------------------------------------- P6 -----

def test_hand_traced_peak_w1():
    """P6 ("live from the time it is created until its last usage").
    W1 (1,1,1,1): d = 64, m = 64, e = 2 -> every tensor is 8192 B.
    Params W0 W1 G0 G1 X Y = 6 tensors = 49152.  Forward: MatMul0 +Z (57344),
    Relu0 +A1 -Z, MatMul1 +Z', Relu1 +A2 -> 73728 (peak), -Z' -> 65536.
    LossGrad +dA2 (73728), -Y; ReluGrad1 +dZ (73728) -A2 -dA2; MatMulGrad1
    +dA1 +dW1 (73728) -dZ; Add1 +G1' (73728) -G1 -dW1 -> 57344; ReluGrad0
    +dZ0 -A1 -dA1; MatMulGrad0 +dA0(dead) +dW0 -X -dZ0 -dA0; Add0; SGD0 +W0'
    -W0 -G0'; SGD1 -> final live = W0' + W1' = 16384."""
    r = oracle.eval_config(W.MODELS["mlp_w1"], W.TOPOLOGIES["TB200"],
                           1, 1, 1, 1, 64)
    assert r["peak"] == 73728
    vals, ops = oracle.export_program(W.MODELS["mlp_w1"],
                                      W.TOPOLOGIES["TB200"], 1, 1, 1, 1, 64)
    raw = oracle.simulate_raw(1, [(o[0], o[1], o[2], o[3]) for o in ops], vals)
    assert raw["live"][0] == 16384 and raw["peak"][0] == 73728


# ------------------------------------------------------------------- P7 -----

@pytest.mark.parametrize("seed", range(200))
def test_random_programs_bruteforce(seed):
    """P7(i): on random programs (<= 30 ops, <= 4 devices)
    the oracle walk equals the per-device co-simulation (P:471 projection +
    rendezvous) and the longest path, exactly (dyadic costs)."""
    n_dev, ops = W.random_program(seed)
    r = oracle.simulate_raw(n_dev, ops)
    s, e, ms = bf.cosimulate(n_dev, ops)
    assert r["makespan"] == ms == bf.longest_path(n_dev, ops)
    assert list(r["start"]) == s and list(r["end"]) == e
    # events on one device never overlap, program order kept
    for d in range(n_dev):
        mine = [i for i, op in enumerate(ops) if d in op[0]]
        for a, b in zip(mine, mine[1:]):
            assert r["end"][a] <= r["start"][b]


def _small_cases():
    mlp = W.MODELS["mlp_w1"]
    cases = []
    for D, T, P, K in [(1, 1, 1, 1), (2, 1, 1, 2), (1, 2, 1, 2), (1, 1, 2, 2),
                       (2, 2, 1, 1), (1, 2, 2, 2), (2, 1, 2, 2), (1, 4, 1, 2),
                       (1, 1, 2, 1), (2, 2, 2, 2)]:
        cases.append((mlp, D, T, P, K, 64))
    mlp3 = W.mlp(3, 32)
    for D, T, P, K in [(1, 2, 2, 4), (2, 2, 2, 2), (1, 1, 2, 3)]:
        cases.append((mlp3, D, T, P, K, 24))
    g = dict(W.MODELS["gpt2_small"], n_layer=3, d_model=64, n_head=4,
             vocab_pad=128, n_ctx=16)
    for D, T, P, K in [(1, 1, 1, 1), (1, 2, 2, 2), (2, 2, 1, 2), (1, 1, 2, 4),
                       (2, 1, 2, 2), (1, 4, 1, 1)]:
        cases.append((g, D, T, P, K, D * K * 2))
    cases.append((dict(g, lm_head=0), 1, 2, 2, 2, 4))
    return cases


@pytest.mark.parametrize("case", range(len(_small_cases())))
def test_generated_programs_bruteforce(case):
    """P7 on the oracle's own generated MLP / GPT-2 programs: makespan equals
    the per-device co-simulation, and per-device peaks equal live-interval
    stabbing -- both independent formulations in oracle.bruteforce."""
    model, D, T, P, K, B = _small_cases()[case]
    t = W.TOPOLOGIES["TB200"]
    r = oracle.eval_config(model, t, D, T, P, K, B)
    vals, ops = oracle.export_program(model, t, D, T, P, K, B)
    n = D * T * P
    assert bf.cosimulate(n, ops)[2] == r["makespan"]
    assert bf.interval_peaks(n, ops, vals) == r["peaks"].tolist()


def test_topk_equals_python_sort():
    """P7(ii): top-k = Python sort on (throughput desc, peak asc, index asc)
    over feasible entries, including ties."""
    rng = np.random.default_rng(7)
    n = 500
    ms = rng.choice([1.0, 2.0, 4.0, 0.5], size=n)
    batch = rng.choice([128, 256], size=n).astype(np.int64)
    peak = rng.integers(0, 4, size=n).astype(np.int64)
    reason = (rng.random(n) < 0.2).astype(np.uint32)
    idx = np.arange(n, dtype=np.int64)
    for k in [1, 10, 64, 600]:
        pos, tp = oracle.topk(idx, batch, ms, peak, reason, k)
        ref = bf.topk_sorted(idx, batch / ms, peak, reason == 0, k)
        assert pos.tolist() == ref


# ------------------------------------------------------------------- P8 -----

def test_invariants_scaling_and_topology_independence():
    """P8: scaling every cost by 2 scales the makespan by exactly 2;
    peaks do not depend on costs or topology (SURVEY C.7 Theorem 4)."""
    t = W.TOPOLOGIES["TB200"]
    t2 = dict(t, flops_per_s=t["flops_per_s"] / 2, op_overhead_s=2 *
              t["op_overhead_s"], alpha_intra_s=2 * t["alpha_intra_s"],
              alpha_inter_s=2 * t["alpha_inter_s"], bw_intra_Bps=t[
                  "bw_intra_Bps"] / 2, bw_inter_Bps=t["bw_inter_Bps"] / 2)
    for (D, T, P, K) in [(2, 2, 2, 4), (1, 4, 4, 8), (4, 1, 2, 2)]:
        for m in [W.MODELS["mlp_1b"], W.MODELS["gpt2_small"]]:
            a = oracle.eval_config(m, t, D, T, P, K, 1024)
            b = oracle.eval_config(m, t2, D, T, P, K, 1024)
            c = oracle.eval_config(m, W.TOPOLOGIES["TV100"], D, T, P, K, 1024)
            assert b["makespan"] == 2 * a["makespan"]
            assert (a["peaks"] == b["peaks"]).all()
            assert (a["peaks"] == c["peaks"]).all()


def test_invariant_stage_symmetry():
    """P8 / SURVEY C.6 Theorem 2: with power-of-two sizes all D*T ranks of a
    stage end with the same clock and the same peak."""
    for m in [W.MODELS["mlp_1b"], W.MODELS["gpt2_medium"]]:
        for t in [W.TOPOLOGIES["TB200"], W.TOPOLOGIES["TM0"]]:
            for (D, T, P, K) in [(2, 2, 4, 4), (4, 2, 2, 2), (1, 8, 2, 2),
                                 (2, 4, 8, 2)]:
                r = oracle.eval_config(m, t, D, T, P, K, 2048)
                ck = r["clocks"].reshape(P, D * T)
                pk = r["peaks"].reshape(P, D * T)
                assert (ck == ck[:, :1]).all() and (pk == pk[:, :1]).all()


def test_reorder_invariance_random_linear_extensions():
    """P8 / Theorem 1: any global order keeping each device's
    op subsequence gives bit-identical op end times."""
    rng = random.Random(3)
    for seed in range(40):
        n_dev, ops = W.random_program(1000 + seed)
        base = oracle.simulate_raw(n_dev, ops)
        # random linear extension of the per-device order
        remaining = list(range(len(ops)))
        order = []
        while remaining:
            ready = [i for i in remaining
                     if all(not (set(ops[j][0]) & set(ops[i][0]))
                            for j in remaining if j < i)]
            pick = rng.choice(ready)
            order.append(pick)
            remaining.remove(pick)
        r = oracle.simulate_raw(n_dev, [ops[i] for i in order])
        assert [r["end"][order.index(i)] for i in range(len(ops))] == \
            list(base["end"])


# ---------------------------------------------------------- op counts -------

@pytest.mark.parametrize("D,T,P,K,L", [
    (1, 1, 1, 1, 2), (2, 1, 1, 1, 2), (1, 2, 1, 1, 2), (1, 1, 2, 2, 4),
    (2, 2, 2, 2, 4), (4, 1, 2, 8, 8), (1, 4, 4, 2, 5), (2, 2, 4, 3, 7)])
def test_mlp_op_count_closed_form(D, T, P, K, L):
    """SURVEY C.3 op count, counted from the structure of one GPipe training
    step: per microbatch and rank 5 ops per layer (MatMul, Relu, ReluGrad,
    MatMulGrad, Add), one SGD per layer, one LossGrad per last-stage rank,
    one TP AllReduce per layer per microbatch per replica when T > 1, a
    forward and a backward Send per stage boundary, and one DP AllReduce per
    layer per TP index when D > 1."""
    r = oracle.eval_config(W.mlp(L, 64), W.TOPOLOGIES["TB200"], D, T, P, K,
                           64 * D * K)
    expect = (5 * K * D * T * L + D * T * L + K * D * T + (T > 1) * K * D * L
              + 2 * K * D * T * (P - 1) + (D > 1) * T * L)
    assert r["n_ops"] == expect


@pytest.mark.parametrize("D,T,P,K,L", [
    (1, 1, 1, 1, 1), (1, 2, 1, 1, 2), (2, 2, 2, 2, 4), (1, 1, 4, 8, 12),
    (2, 4, 2, 2, 6)])
def test_gpt2_op_count_closed_form(D, T, P, K, L):
    """SURVEY C.4 op count: 12 compute ops per block, embedding + final LN +
    LM head per microbatch, 2 TP AllReduces per block plus one after the
    embedding and one logits AllGather per replica when T > 1, one Send per
    stage boundary."""
    m = dict(W.MODELS["gpt2_small"], n_layer=L, d_model=64, n_head=4)
    r = oracle.eval_config(m, W.TOPOLOGIES["TB200"], D, T, P, K, 2 * D * K)
    expect = (12 * K * D * T * L + 3 * K * D * T + (T > 1) * K * D * (2 * L + 2)
              + K * D * T * (P - 1))
    assert r["n_ops"] == expect


def test_gpt2_flops_match_transformer_rule():
    """Textbook forward FLOPs of a transformer: about 2 x (12 L d^2 + V d)
    per token, the rest O(L d + S) per token (Kaplan et al.).  The oracle's
    one-rank GPT-2 program must land within 1.5 % of it for GPT-2 small."""
    m = W.MODELS["gpt2_small"]
    ops = oracle.program_ops(m, W.TOPOLOGIES["TB200"], 1, 1, 1, 1, 4)
    tokens = 4 * m["seq_len"]
    rule = 2 * tokens * (12 * m["n_layer"] * m["d_model"] ** 2 +
                         m["vocab_pad"] * m["d_model"])
    assert abs(ops["work"].sum() - rule) / rule < 0.015


# ------------------------------------------------------------- P12 ----------

@pytest.mark.parametrize("cfg,ops,ms,peaks", [
    ((1, 1, 1, 1), 13, 6.500236086789668e-05, [73728]),
    ((2, 1, 1, 1), 28, 7.301939394702747e-05, [61440, 61440]),
    ((1, 2, 1, 1), 28, 7.301939243558835e-05, [53248, 53248]),
    ((1, 1, 2, 1), 15, 6.402055926658468e-05, [49152, 49152]),
    ((1, 1, 2, 2), 28, 9.801997887396474e-05, [45056, 49152]),
    ((2, 1, 1, 2), 50, 1.280193999927839e-04, [63488, 63488]),
    ((1, 2, 1, 2), 52, 1.360193954584666e-04, [49152, 49152])])
def test_spec_regression_values_survey_p12(cfg, ops, ms, peaks):
    """P12: values a throwaway model of C.3 + C.5-C.7 printed
    during the survey (W1 model on TB200).  Not independent of the spec --
    a regression check that this oracle reads §8c the same way."""
    D, T, P, K = cfg
    r = oracle.eval_config(W.MODELS["mlp_w1"], W.TOPOLOGIES["TB200"],
                           D, T, P, K, 64)
    assert r["n_ops"] == ops
    assert r["makespan"] == pytest.approx(ms, rel=1e-15)
    assert r["peaks"].tolist() == peaks


def test_synth_generator_matches_workloads():
    """The oracle's counter-based W5 generator (C++) equals workloads'
    Python one on the first 2000 indices (same recipe)."""
    g = dict(W.GRIDS["W5"], synth_count=2000)
    f, mo = oracle.enumerate_grid(g, with_models=True)
    for i in range(2000):
        model, ts, D, T, P, K, B = W.synth_config(g["synth_seed"], i)
        assert tuple(f[i, 1:8]) == (ts, D * T * P, D, T, P, K, B)
        assert mo[i].tolist() == oracle.model_fields(model).tolist()
