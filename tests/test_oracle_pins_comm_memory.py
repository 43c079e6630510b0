"""Pins for the oracle parts round 1 left unpinned:

* ring AllReduce and AllGather at g > 2 (`op_cost`; the paper's
  "network bandwidths" coefficients, §4 Implementation);
* the intra/inter-node link class of a group (`intra`, C.5; same passage);
* GPT-2 value lifetimes: "live from the time it is created until its last
  usage" (§3.3), the one-rank and two-stage peaks and final live bytes
  (`build_gpt2`; the P6 analogue for the inference program).

None of the expected values re-types the oracle's formulas:

* Collective times come from a chunk-level simulation of the textbook ring
  algorithms (reduce-scatter then all-gather; Patarasuk & Yuan 2009), which
  moves explicit chunk contributor sets around a ring until every node holds
  the complete result, and charges each synchronous step alpha + chunk / bw
  (the alpha-beta link model named by north_star).  The step count and chunk
  size fall out of the data movement, not out of a formula.  All constants
  are dyadic, so the oracle's binary64 makespan must equal the exact rational
  (fractions.Fraction) value.
* Compute costs are made exactly zero (F = inf, o = 0) so the makespan is the
  sum of the communication steps on the busiest device.
* Liveness values are hand traces written out op by op in the docstrings
  (C.7 event order: allocate outputs, record peaks, free inputs at their last
  use; parameters live from t = 0; returned values never freed).
"""
import math
from fractions import Fraction as Fr

import pytest

import oracle
import workloads as W

ALPHA_I, BW_I = 2.0 ** -10, 2.0 ** 30      # intra-node link (dyadic)
ALPHA_X, BW_X = 2.0 ** -7, 2.0 ** 27       # inter-node link (dyadic, distinct)


def comm_only_topo(node_size):
    """Compute ops cost exactly 0 (flops / inf + 0); links are dyadic."""
    t = dict(W.TOPOLOGIES["TB200"])
    t.update(flops_per_s=math.inf, op_overhead_s=0.0, node_size=node_size,
             alpha_intra_s=ALPHA_I, bw_intra_Bps=BW_I,
             alpha_inter_s=ALPHA_X, bw_inter_Bps=BW_X, capacity_bytes=1 << 60)
    return t


# ------------------------------------------- textbook ring, chunk by chunk --

def ring_allreduce(g, nbytes, alpha, bw):
    """Ring all-reduce of an nbytes buffer over g nodes, simulated on chunk
    contributor sets.  The buffer is cut into g chunks; each synchronous step
    every node sends one chunk to its successor.  Reduce-scatter: a node
    forwards the chunk it last accumulated (it starts with its own chunk r),
    the receiver adds its contribution.  All-gather: a node forwards the
    complete chunk it last obtained, the receiver overwrites.  Returns
    (steps, exact time) with each step costing alpha + chunk / bw."""
    have = [[frozenset([r]) for _ in range(g)] for r in range(g)]
    full = frozenset(range(g))
    steps = 0
    sending = list(range(g))                    # chunk node r sends next
    # phase 1: reduce-scatter, until some node holds a complete chunk
    while not any(have[r][c] == full for r in range(g) for c in range(g)):
        msgs = [((r + 1) % g, sending[r], have[r][sending[r]]) for r in range(g)]
        for dst, c, s in msgs:
            have[dst][c] = have[dst][c] | s
        sending = [msgs[(r - 1) % g][1] for r in range(g)]   # forward what arrived
        steps += 1
    # phase 2: all-gather of the complete chunks
    sending = [next(c for c in range(g) if have[r][c] == full) for r in range(g)]
    while not all(have[r][c] == full for r in range(g) for c in range(g)):
        msgs = [((r + 1) % g, sending[r], have[r][sending[r]]) for r in range(g)]
        for dst, c, s in msgs:
            assert s == full
            have[dst][c] = s
        sending = [msgs[(r - 1) % g][1] for r in range(g)]
        steps += 1
    chunk = Fr(nbytes) / g
    return steps, steps * (Fr(alpha) + chunk / Fr(bw))


def ring_allgather(g, gathered_bytes, alpha, bw):
    """Ring all-gather: node r starts with block r of gathered_bytes / g; each
    step every node forwards the block it received last.  Returns (steps,
    exact time)."""
    have = [{r} for r in range(g)]
    sending = list(range(g))
    steps = 0
    while not all(len(h) == g for h in have):
        msgs = [((r + 1) % g, sending[r]) for r in range(g)]
        for dst, b in msgs:
            have[dst].add(b)
        sending = [msgs[(r - 1) % g][1] for r in range(g)]
        steps += 1
    block = Fr(gathered_bytes) / g
    return steps, steps * (Fr(alpha) + block / Fr(bw))


def p2p(nbytes, alpha, bw):
    return Fr(alpha) + Fr(nbytes) / Fr(bw)


@pytest.mark.parametrize("g", [2, 3, 4, 5, 8, 16])
def test_ring_models_move_every_byte(g):
    """Sanity of the brute-force ring itself: 2(g-1) steps for all-reduce,
    g-1 for all-gather, every node ends with every contribution; each node
    sends 2(g-1)/g of the buffer, the known bandwidth-optimal volume."""
    s_ar, _ = ring_allreduce(g, 1024, 0.0, 1.0)
    s_ag, _ = ring_allgather(g, 1024, 0.0, 1.0)
    assert s_ar == 2 * (g - 1) and s_ag == g - 1


# --------------------------------------------------- the small GPT-2 model --

def tiny_gpt2(L=1):
    # d = 64, h = 8 heads, S = 8, V_pad = 128, n_ctx = 16 -> T in {2, 4, 8}
    return W.gpt2(L, 64, 8, seq_len=8, vocab_pad=128, n_ctx=16)


@pytest.mark.parametrize("g", [2, 4, 8])
def test_tp_allreduce_allgather_ring_g(g):
    """One-stage GPT-2 (L = 1, D = P = K = 1, T = g, m = 2 -> n = 16 tokens)
    on one node: each TP rank runs three TP AllReduces of the n x d
    activation (after the embedding and after the attention projection and
    FC2 of the block, C.4) and one AllGather of the n x V_pad logits; with
    zero compute cost the makespan is exactly their sum."""
    t = comm_only_topo(node_size=8)
    n, d, V, e = 16, 64, 128, 2
    r = oracle.eval_config(tiny_gpt2(), t, 1, g, 1, 1, 2)
    _, ar = ring_allreduce(g, n * d * e, ALPHA_I, BW_I)
    _, ag = ring_allgather(g, n * V * e, ALPHA_I, BW_I)
    assert Fr(r["makespan"]) == 3 * ar + ag
    assert all(Fr(c) == 3 * ar + ag for c in r["clocks"])


@pytest.mark.parametrize("g", [4, 8])
def test_tp_group_spanning_two_nodes_is_inter(g):
    """Link class (C.5): with node_size = g / 2 the TP group {0..g-1} spans
    two nodes, so every TP collective runs on the inter-node constants."""
    t = comm_only_topo(node_size=g // 2)
    n, d, V, e = 16, 64, 128, 2
    r = oracle.eval_config(tiny_gpt2(), t, 1, g, 1, 1, 2)
    _, ar = ring_allreduce(g, n * d * e, ALPHA_X, BW_X)
    _, ag = ring_allgather(g, n * V * e, ALPHA_X, BW_X)
    assert Fr(r["makespan"]) == 3 * ar + ag


@pytest.mark.parametrize("D,node_size,inter", [(4, 8, False), (8, 8, False),
                                               (4, 2, True), (8, 4, True)])
def test_dp_allreduce_ring_g(D, node_size, inter):
    """MLP training (L = 2, d = 64, T = P = K = 1, D replicas, m = 8): with
    zero compute cost a rank's time is the tail's two DP AllReduces of the
    d x d gradients (C.3), each over the D replicas."""
    t = comm_only_topo(node_size)
    a, bw = (ALPHA_X, BW_X) if inter else (ALPHA_I, BW_I)
    r = oracle.eval_config(W.mlp(2, 64), t, D, 1, 1, 1, 8 * D)
    _, ar = ring_allreduce(D, 64 * 64 * 2, a, bw)
    assert Fr(r["makespan"]) == 2 * ar


def test_mixed_link_classes_tp_intra_dp_inter():
    """D = T = 2, node_size = 2: ranks j + 2i, so TP groups {0,1}, {2,3}
    are each inside a node and DP groups {0,2}, {1,3} cross nodes.  MLP
    L = 2, d = 64, m = 8: layer 1 (row) has a forward TP AllReduce and layer 0
    (col) a backward one, both of m x d; the tail has one DP AllReduce per
    layer of the local (d x d/2) gradient shard."""
    t = comm_only_topo(node_size=2)
    m, d, e = 8, 64, 2
    r = oracle.eval_config(W.mlp(2, 64), t, 2, 2, 1, 1, 2 * m)
    _, tp = ring_allreduce(2, m * d * e, ALPHA_I, BW_I)
    _, dp = ring_allreduce(2, d * (d // 2) * e, ALPHA_X, BW_X)
    assert Fr(r["makespan"]) == 2 * tp + 2 * dp
    # the same program on one node: everything intra
    r1 = oracle.eval_config(W.mlp(2, 64), comm_only_topo(8), 2, 2, 1, 1, 2 * m)
    _, dp1 = ring_allreduce(2, d * (d // 2) * e, ALPHA_I, BW_I)
    assert Fr(r1["makespan"]) == 2 * tp + 2 * dp1


@pytest.mark.parametrize("node_size,inter", [(1, True), (2, False)])
def test_pipeline_send_link_class(node_size, inter):
    """MLP L = 2, P = 2, K = 1, m = 8: one forward and one backward Send of
    m x d between ranks 0 and 1 (C.3); on separate nodes they use the
    inter-node link."""
    t = comm_only_topo(node_size)
    a, bw = (ALPHA_X, BW_X) if inter else (ALPHA_I, BW_I)
    r = oracle.eval_config(W.mlp(2, 64), t, 1, 1, 2, 1, 8)
    assert Fr(r["makespan"]) == 2 * p2p(8 * 64 * 2, a, bw)


# ------------------------------------------------- GPT-2 liveness ---

def _final_live(model, D, T, P, K, B):
    vals, ops = oracle.export_program(model, W.TOPOLOGIES["TB200"], D, T, P,
                                      K, B)
    raw = oracle.simulate_raw(D * T * P, [(o[0], o[1], o[2], o[3]) for o in ops],
                              vals)
    return raw["live"].tolist(), raw["peak"].tolist()


def test_gpt2_one_rank_hand_traced_liveness():
    """Hand trace (C.7) of GPT-2 L = 1, d = 64, h = 8, S = 8,
    V_pad = 128, n_ctx = 16, e = 2, ids 8 B, one rank, K = 1, m = 2 (n = 16
    tokens, so an n x d activation is 2048 B).

    Parameters live from t = 0: block ln_1 256, W_qkv 24576, b_qkv 384,
    W_proj 8192, b_proj 128, ln_2 256, W_fc1 32768, b_fc1 512, W_fc2 32768,
    b_fc2 128 (= 99968); wte 16384, wpe 2048, ids 128, ln_f 256 -> 118784.
      Embed  +x 2048 -> 120832;  -ids -wpe              -> 118656
      LN1    +2048   -> 120704;  -ln_1                   -> 120448
      QKV    +6144   -> 126592 (peak); -h1 -W_qkv -b_qkv -> 99584
      Scores +2048 (m h S^2 e) -> 101632 (qkv still needed)
      Softmax +2048 -> 103680; -scores -> 101632
      Context +2048 -> 103680; -probs -qkv -> 95488
      Proj   +2048 -> 97536;  -ctx -W_proj -b_proj -> 87168
      Add    +2048 -> 89216;  -x -proj               -> 85120
      LN2    +2048 -> 87168;  -ln_2                  -> 86912
      FC1    +8192 -> 95104;  -h2 -W_fc1 -b_fc1      -> 59776
      GeLU   +8192 -> 67968;  -fc1                   -> 59776
      FC2    +2048 -> 61824;  -gelu -W_fc2 -b_fc2    -> 20736
      Add    +2048 -> 22784;  -x2 -fc2               -> 18688
      LN_f   +2048 -> 20736;  -x3 -ln_f              -> 18432
      LMhead +4096 (n V e, returned) -> 22528; -hf -wte -> 4096
    Peak 126592, final live 4096 (the logits)."""
    m = tiny_gpt2()
    r = oracle.eval_config(m, W.TOPOLOGIES["TB200"], 1, 1, 1, 1, 2)
    assert r["peak"] == 126592
    live, peak = _final_live(m, 1, 1, 1, 1, 2)
    assert live == [4096] and peak == [126592]
    # without the LM head wte dies at the Embed (its last use), so the peak
    # moves to the Embed (120832; QKV reaches only 126592 - 16384), and the
    # final-LayerNorm output is the returned value (2048)
    live, peak = _final_live(dict(m, lm_head=0), 1, 1, 1, 1, 2)
    assert live == [2048] and peak == [120832]


def test_gpt2_two_stage_hand_traced_liveness():
    """Hand trace of GPT-2 L = 2 on P = 2 stages, K = 2 microbatches,
    m = 2 (B = 4), same shapes as above.  Parameters are used by both
    microbatches and die at their use in k = 1 (DESIGN R2).

    Rank 0 (embedding + block 0) starts at 99968 + wte 16384 + wpe 2048 +
    ids 2 x 128 = 118656.  k = 0: Embed +2048 -> 120704, -ids_0 -> 120576;
    LN1 +2048 -> 122624; QKV +6144 -> 128768, -h1 -> 126720; Scores +2048
    -> 128768; Softmax +2048 -> 130816, -sc -> 128768; Context +2048 ->
    130816, -probs -qkv -> 122624; Proj +2048 -> 124672, -ctx -> 122624;
    Add +2048 -> 124672, -x -proj -> 120576; LN2 +2048 -> 122624; FC1 +8192
    -> 130816, -h2 -> 128768; GeLU +8192 -> 136960 (peak), -fc1 -> 128768;
    FC2 +2048 -> 130816, -gelu -> 122624; Add +2048 -> 124672, -x2 -fc2 ->
    120576; Send -x3 -> 118528.  k = 1 runs the same ops and frees every
    parameter at its use (wte and wpe at the Embed), ending at 0.

    Rank 1 (block 1 + ln_f + tied wte shard) starts at 99968 + 256 + 16384
    = 116608.  k = 0: Recv +2048 -> 118656; LN1 +2048 -> 120704; QKV +6144
    -> 126848, -h1 -> 124800; Scores -> 126848; Softmax -> 128896 -> 126848;
    Context -> 128896, -> 120704; Proj -> 122752 -> 120704; Add -> 122752
    -> 118656; LN2 -> 120704; FC1 +8192 -> 128896, -h2 -> 126848; GeLU
    +8192 -> 135040 (peak), -> 126848; FC2 -> 128896 -> 120704; Add ->
    122752 -> 118656; LN_f -> 120704, -x3 -> 118656; LM head +4096 (returned)
    -> 122752, -hf -> 120704.  k = 1 frees all parameters; two 4096-B
    logits remain: final live 8192."""
    m = tiny_gpt2(L=2)
    r = oracle.eval_config(m, W.TOPOLOGIES["TB200"], 1, 1, 2, 2, 4)
    assert r["peaks"].tolist() == [136960, 135040]
    live, peak = _final_live(m, 1, 1, 2, 2, 4)
    assert live == [0, 8192] and peak == [136960, 135040]


def test_gpt2_tp2_hand_traced_final_live():
    """T = 2 (L = 1, one stage, m = 2): every rank ends holding the gathered
    n x V_pad logits (4096 B, returned); its shard (n x V_pad/2, 2048 B) dies
    at the AllGather.  Peak: parameters per rank are the block's TP shards
    (ln_1 256 + W_qkv 12288 + b_qkv 192 + W_proj 4096 + b_proj 128 + ln_2 256
    + W_fc1 16384 + b_fc1 256 + W_fc2 16384 + b_fc2 128 = 50368) + wte shard
    8192 + wpe 2048 + ids 128 + ln_f 256 = 60992.  Embed +2048 -> 63040,
    -ids -wpe -> 60864; AllReduce +2048 -> 62912, -partial -> 60864; LN1
    +2048 -> 62912, -ln_1 -> 62656; QKV +3072 -> 65728 (peak), -h1 -W_qkv
    -b_qkv -> 51072; every later op stays below (the largest is FC1/GeLU:
    +4096 on <= 47000)."""
    m = tiny_gpt2()
    r = oracle.eval_config(m, W.TOPOLOGIES["TB200"], 1, 2, 1, 1, 2)
    assert r["peaks"].tolist() == [65728, 65728]
    live, _ = _final_live(m, 1, 2, 1, 1, 2)
    assert live == [4096, 4096]
