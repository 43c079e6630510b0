"""Seeded, synthetic inputs shared by the oracle and the CUDA path.

This module holds DATA ONLY -- model shapes, hardware (topology) constants,
grid specifications and two seeded input generators.  It contains none of the
method's arithmetic (no op expansion, no costs, no timeline, no memory walk,
no ranking).  It is the one module both `oracle/` and the product binding may
import (task rule: "only the seeded input generators serve both").

Citations: `P:n` = /root/reference/PAPER.md line n; `SURVEY §x` = SURVEY.md.

* Models: MLP training (Table 1; square bias-free
  layers, 16-bit values P:543) and GPT-2 inference (HF shapes; paper
  sizes P:537-539 with the 13B d_model read as 5120).
* Topologies: illustrative constants, not calibrations -- the
  paper's fitted coefficients are unpublished.
* Grids W1..W5, PM, PG.
* `synth_config(seed, index)`: the counter-based W5 generator,
  re-implemented independently by the oracle (C++) and the CUDA enumerator.
* `random_program(seed, ...)`: random small raw DistIR programs for the
  brute-force pin P7.
"""
from __future__ import annotations

import random

MLP_TRAIN = 0
GPT2_INFER = 1

# ----------------------------------------------------------------------------
# Models.  Fields mirror the paper's vocabulary: n_layer, d_model (Table 1),
# n_head, seq_len S, padded vocab, n_ctx, dtype bytes e (16-bit), token-id
# bytes, lm_head flag.
# ----------------------------------------------------------------------------

GPIPE = 0
ONE_F_ONE_B = 1


def mlp(n_layer, d_model, dtype_bytes=2, schedule=GPIPE, recompute=0, zero=0):
    """schedule: the pipeline schedule of the training transform -- GPipe
    (north_star) or the paper's synchronous 1F1B (NEXT row f1).
    recompute / zero: the memory-saving variants of the Appendix (NEXT row
    f4): gradient checkpointing (Fig. 8) and ZeRO-2/3 parameter and
    gradient partitioning over the data-parallel replicas (Fig. 9)."""
    return dict(kind=MLP_TRAIN, n_layer=n_layer, d_model=d_model, n_head=1,
                seq_len=1, vocab_pad=0, n_ctx=0, dtype_bytes=dtype_bytes,
                id_bytes=8, lm_head=0, schedule=schedule, recompute=recompute,
                zero=zero)


def gpt2(n_layer, d_model, n_head, seq_len=8, vocab_pad=50304, n_ctx=1024,
         dtype_bytes=2, lm_head=1):
    return dict(kind=GPT2_INFER, n_layer=n_layer, d_model=d_model,
                n_head=n_head, seq_len=seq_len, vocab_pad=vocab_pad,
                n_ctx=n_ctx, dtype_bytes=dtype_bytes, id_bytes=8,
                lm_head=lm_head, schedule=GPIPE, recompute=0, zero=0)


MODELS = {
    # W1 (BASELINE configs[0]): 2-layer MLP, dim 64.
    "mlp_w1": mlp(2, 64),
    # Table 1 MLP rows.
    "mlp_1b": mlp(16, 8192),
    "mlp_17b": mlp(64, 16384),
    "mlp_103b": mlp(96, 32768),
    # W4 deep-pipeline stress (BASELINE configs[3]).
    "mlp_w4": mlp(64, 8192),
    # the paper's own pipeline schedule (1F1B; NEXT row f1)
    "mlp_w1_1f1b": mlp(2, 64, schedule=1),
    "mlp_1b_1f1b": mlp(16, 8192, schedule=1),
    "mlp_w4_1f1b": mlp(64, 8192, schedule=1),
    # memory-saving variants (Appendix Figs. 8/9; NEXT row f4)
    "mlp_w1_ckpt": mlp(2, 64, recompute=1),
    "mlp_w1_zero": mlp(2, 64, zero=1),
    "mlp_1b_ckpt": mlp(16, 8192, recompute=1),
    "mlp_1b_zero": mlp(16, 8192, zero=1),
    "mlp_1b_zero_ckpt": mlp(16, 8192, recompute=1, zero=1),
    # HF GPT-2 family (W3, BASELINE configs[2]).
    "gpt2_small": gpt2(12, 768, 12),
    "gpt2_medium": gpt2(24, 1024, 16),
    "gpt2_large": gpt2(36, 1280, 20),
    "gpt2_xl": gpt2(48, 1600, 25),
    # Table 1 GPT-2 rows; heads h = d/128.
    "gpt2_1_6b": gpt2(24, 2048, 16),
    "gpt2_13b": gpt2(40, 5120, 40),
    "gpt2_175b": gpt2(96, 12288, 96),
    # W4 under ZeRO (D = 1 on W4: the plain kernels; P up to 64)
    "mlp_w4_zero": mlp(64, 8192, zero=1),
    # ZeRO under the paper's 1F1B schedule
    "mlp_w1_zero_1f1b": mlp(2, 64, zero=1, schedule=1),
    "mlp_1b_zero_1f1b": mlp(16, 8192, zero=1, schedule=1),
}

HF_GPT2 = ["gpt2_small", "gpt2_medium", "gpt2_large", "gpt2_xl"]

# ----------------------------------------------------------------------------
# Topologies.  capacity in bytes.
# ----------------------------------------------------------------------------

def topo(world_max, node_size, flops, overhead, a_intra, bw_intra, a_inter,
         bw_inter, capacity, regression=None):
    """regression: None (analytic flops/F + o) or the six coefficients of the
    paper's regression cost functions (NEXT row f2) as a dict
    with keys mm_c0_s, mm_s_per_flop, mm_s_per_byte, ew_c0_s, ew_s_per_flop,
    ew_s_per_byte."""
    t = dict(world_max=world_max, node_size=node_size, flops_per_s=flops,
             op_overhead_s=overhead, alpha_intra_s=a_intra,
             bw_intra_Bps=bw_intra, alpha_inter_s=a_inter,
             bw_inter_Bps=bw_inter, capacity_bytes=capacity, cost_model=0)
    if regression is not None:
        t["cost_model"] = 1
        for k in REGRESSION_KEYS:
            t[k] = float(regression[k])
    return t


REGRESSION_KEYS = ("mm_c0_s", "mm_s_per_flop", "mm_s_per_byte",
                   "ew_c0_s", "ew_s_per_flop", "ew_s_per_byte")


def _load_calibration():
    """The B200 coefficients fitted by `python -m
    paper_2111_05426_b200.calibrate` (data file, committed)."""
    import json
    import os
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "calib_b200.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        return json.load(f)


TOPOLOGIES = {
    # paper-shaped DGX-2: 16 x V100 32 GB on NVLink; 32 GiB (C.9 A24).
    "TV100": topo(16, 16, 125e12, 1e-5, 5e-6, 150e9, 5e-6, 150e9,
                  34359738368),
    # B200 HGX: 8 GPUs per node, NVLink 5 900 GB/s per direction,
    # F = MEASURED_PEAKS bf16 sustained 1355 TF/s.
    "TB200": topo(64, 8, 1.355e15, 5e-6, 2e-6, 900e9, 5e-6, 50e9,
                  180000000000),
}
for _i in range(8):
    _ns = 8 if (_i & 4) else 4
    _bwi = 900e9 if (_i & 2) else 450e9
    _bwx = 50e9 if (_i & 1) else 25e9
    TOPOLOGIES["TM%d" % _i] = topo(64, _ns, 1.355e15, 5e-6, 2e-6, _bwi,
                                   5e-6, _bwx, 180000000000)

TM = ["TM%d" % i for i in range(8)]

# TB200 with the regression cost functions calibrated on a B200 (row f2).
_CAL = _load_calibration()
if _CAL is not None:
    TOPOLOGIES["TB200R"] = topo(64, 8, 1.355e15, 5e-6, 2e-6, 900e9, 5e-6, 50e9,
                                180000000000, regression=_CAL)
# A regression topology with dyadic coefficients (exact sums; parity tests).
TOPOLOGIES["TRD"] = topo(64, 8, 2.0 ** 50, 2.0 ** -18, 2.0 ** -19, 2.0 ** 39,
                         2.0 ** -17, 2.0 ** 35, 180000000000,
                         regression=dict(mm_c0_s=2.0 ** -18, mm_s_per_flop=2.0 ** -50,
                                         mm_s_per_byte=2.0 ** -43, ew_c0_s=2.0 ** -19,
                                         ew_s_per_flop=2.0 ** -46, ew_s_per_byte=2.0 ** -42))

# ----------------------------------------------------------------------------
# Grid specifications (SURVEY C.1 enumeration, §8d D.1 workloads).
# k_mode 0: K = 1 when P == 1 else k_set (paper); k_mode 1: k_set always.
# dp/tp/pp masks: bit e set <=> degree 2**e allowed (all ones = unrestricted).
# ----------------------------------------------------------------------------

POW2_K = [2, 4, 8, 16, 32, 64, 128]
ALL = 0xFF


def grid(models, topos, world, batch, k_mode=0, k_set=POW2_K, dp_mask=ALL,
         tp_mask=ALL, pp_mask=ALL, synth_seed=0, synth_count=0):
    return dict(models=list(models), topos=list(topos), world=list(world),
                batch=list(batch), k_mode=k_mode, k_set=list(k_set),
                dp_mask=dp_mask, tp_mask=tp_mask, pp_mask=pp_mask,
                synth_seed=synth_seed, synth_count=synth_count)


GRIDS = {
    # W1: 2-layer MLP dim 64, batch 64, W <= 4, K in {1,2} for every P.
    "W1": grid(["mlp_w1"], ["TB200"], [1, 2, 4], [64], k_mode=1,
               k_set=[1, 2]),
    # W2: the paper's MLP-1B grid, W <= 16, the 12 batch sizes of Table 2.
    "W2": grid(["mlp_1b"], ["TB200"], [1, 2, 4, 8, 16],
               [2 ** e for e in range(7, 19)]),
    # W3: GPT-2 small..XL inference, W <= 16, B in 2^7..2^20.
    "W3": grid(HF_GPT2, ["TB200"], [1, 2, 4, 8, 16],
               [2 ** e for e in range(7, 21)]),
    # W4: 64-layer MLP, D = T = 1, P up to 64, K up to 128 (GPipe).
    "W4": grid(["mlp_w4"], ["TB200"], [1, 2, 4, 8, 16, 32, 64], [1024],
               k_mode=1, k_set=[1, 2, 4, 8, 16, 32, 64, 128], dp_mask=1,
               tp_mask=1),
    # W5: 10^6 synthetic configs, W <= 64, mixed topologies TM0..TM7.
    "W5": grid([], TM, [], [], synth_seed=20211105426, synth_count=10 ** 6),
    # Paper-shaped Table 1 grids (context; W = 16 exactly).
    "PM_1B": grid(["mlp_1b"], ["TV100"], [16], [65536]),
    "PM_17B": grid(["mlp_17b"], ["TV100"], [16], [65536]),
    "PM_103B": grid(["mlp_103b"], ["TV100"], [16], [256]),
    "PG": grid(["gpt2_1_6b", "gpt2_13b", "gpt2_175b"], ["TV100"], [16],
               [2 ** e for e in range(7, 21)]),
}


def grid_with(name, **over):
    g = dict(GRIDS[name])
    g.update(over)
    return g


# ----------------------------------------------------------------------------
# Counter-based W5 generator.  uint64 wrap-around arithmetic.
# Re-implemented independently in oracle/ (C++) and the CUDA enumerator.
# ----------------------------------------------------------------------------

M64 = (1 << 64) - 1


def _mix(z):
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def pow2_triples(world):
    """(D, T, P) powers of two with D*T*P == world, lexicographic (C.1)."""
    out = []
    e = world.bit_length() - 1
    for a in range(e + 1):
        for b in range(e + 1 - a):
            out.append((1 << a, 1 << b, 1 << (e - a - b)))
    return out


def synth_config(seed, index, n_topos=8):
    """Config `index` of the synthetic sweep: returns (model dict, topo slot,
    D, T, P, K, B)."""
    r = [_mix(seed + 0x9E3779B97F4A7C15 * (8 * index + t + 1))
         for t in range(8)]
    kind = r[0] & 1
    world = 1 << (r[1] % 7)
    tr = pow2_triples(world)
    D, T, P = tr[r[2] % len(tr)]
    K = 1 if P == 1 else 1 << (1 + r[3] % 5)
    B = 1 << (7 + r[4] % 12)
    if kind == MLP_TRAIN:
        model = mlp(1 << (1 + r[5] % 6), 1 << (8 + r[6] % 7))
    else:
        model = dict(MODELS[HF_GPT2[r[5] % 4]])
    return model, r[7] % n_topos, D, T, P, K, B


# ----------------------------------------------------------------------------
# Random raw programs for the brute-force pin P7 (<= 30 ops, <= 4 devices).
# An op is (devices, cost).  Costs are small integers scaled by 2^-3 so that
# every sum is exact in binary64 and the brute force can be compared exactly.
# ----------------------------------------------------------------------------

def random_program(seed, max_ops=30, max_devices=4):
    rng = random.Random(seed)
    n_dev = rng.randint(1, max_devices)
    ops = []
    for _ in range(rng.randint(1, max_ops)):
        g = rng.randint(1, n_dev)
        devs = sorted(rng.sample(range(n_dev), g))
        ops.append((devs, rng.randint(0, 40) / 8.0))
    return n_dev, ops
