"""DistIR CPU oracle -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  It wraps
`distir_oracle.cpp` (a plain C++17 explicit-program simulator written from
PAPER.md; see its header for the passages it follows) through ctypes, and
adds pure-Python brute-force checkers (`oracle.bruteforce`).  It shares no
code with `paper_2111_05426_b200/`; both read their inputs from `workloads/`.

Parity status of each oracle function is recorded in DESIGN.md §"Oracle pins".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "distir_oracle.cpp")
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

I64P = ctypes.POINTER(ctypes.c_int64)
I32P = ctypes.POINTER(ctypes.c_int32)
U32P = ctypes.POINTER(ctypes.c_uint32)
U8P = ctypes.POINTER(ctypes.c_uint8)
F64P = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> str:
    """Compile the oracle (g++ -O2 -ffp-contract=off: no FMA contraction)."""
    if force or not os.path.exists(_SO) or (
            os.path.getmtime(_SO) < os.path.getmtime(_SRC)):
        subprocess.check_call([
            "g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fPIC",
            "-shared", "-pthread", "-o", _SO, _SRC])
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        L.oracle_simulate_raw.restype = ctypes.c_int
        L.oracle_eval_config.restype = ctypes.c_int
        L.oracle_program_ops.restype = ctypes.c_int64
        L.oracle_enumerate.restype = ctypes.c_int64
        L.oracle_grid_eval.restype = ctypes.c_int64
        L.oracle_topk.restype = ctypes.c_int32
        L.oracle_grid_validity.restype = ctypes.c_int64
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


MODEL_KEYS = ("kind", "n_layer", "d_model", "n_head", "seq_len", "vocab_pad",
              "n_ctx", "dtype_bytes", "id_bytes", "lm_head", "schedule",
              "recompute", "zero")


def model_fields(m) -> np.ndarray:
    return np.array([int(m.get(k, 0)) for k in MODEL_KEYS], dtype=np.int64)


REGRESSION_KEYS = ("mm_c0_s", "mm_s_per_flop", "mm_s_per_byte",
                   "ew_c0_s", "ew_s_per_flop", "ew_s_per_byte")


def topo_arrays(t):
    """Topology -> (int64[4], float64[12]); cost_model 1 selects the paper's
    regression cost functions (NEXT row f2)."""
    ti = np.array([t["world_max"], t["node_size"], t["capacity_bytes"],
                   int(t.get("cost_model", 0))], dtype=np.int64)
    td = np.array([t["flops_per_s"], t["op_overhead_s"], t["alpha_intra_s"],
                   t["bw_intra_Bps"], t["alpha_inter_s"], t["bw_inter_Bps"]] +
                  [float(t.get(k, 0.0)) for k in REGRESSION_KEYS], dtype=np.float64)
    return ti, td


# ----------------------------------------------------------------- configs --

def eval_config(model, topo, D, T, P, K, B):
    """Simulate one configuration.  Returns dict(makespan, peak, reason,
    n_ops, peaks[W], clocks[W])."""
    L = lib()
    mf = model_fields(model)
    ti, td = topo_arrays(topo)
    W = D * T * P
    pk = np.zeros(W, dtype=np.int64)
    ck = np.zeros(W, dtype=np.float64)
    ms = ctypes.c_double()
    peak = ctypes.c_int64()
    rs = ctypes.c_uint32()
    nops = ctypes.c_int64()
    err = L.oracle_eval_config(
        _p(mf, I64P), _p(ti, I64P), _p(td, F64P), ctypes.c_int64(D),
        ctypes.c_int64(T), ctypes.c_int64(P), ctypes.c_int64(K),
        ctypes.c_int64(B), ctypes.byref(ms), ctypes.byref(peak),
        ctypes.byref(rs), ctypes.byref(nops), _p(pk, I64P), _p(ck, F64P))
    if err:
        raise AssertionError("oracle self-check failed (placement/readiness)")
    return dict(makespan=ms.value, peak=peak.value, reason=rs.value,
                n_ops=nops.value, peaks=pk, clocks=ck)


def program_ops(model, topo, D, T, P, K, B, cap=1 << 22):
    """The explicit program's ops: cls (0 compute, 1 Send, 2 AllReduce,
    3 AllGather), ndev, dev0, work, cost, start, end."""
    L = lib()
    mf = model_fields(model)
    ti, td = topo_arrays(topo)
    a = dict(cls=np.zeros(cap, np.int32), ndev=np.zeros(cap, np.int32),
             dev0=np.zeros(cap, np.int32), work=np.zeros(cap, np.int64),
             cost=np.zeros(cap), start=np.zeros(cap), end=np.zeros(cap))
    n = L.oracle_program_ops(
        _p(mf, I64P), _p(ti, I64P), _p(td, F64P), ctypes.c_int64(D),
        ctypes.c_int64(T), ctypes.c_int64(P), ctypes.c_int64(K),
        ctypes.c_int64(B), ctypes.c_int64(cap), _p(a["cls"], I32P),
        _p(a["ndev"], I32P), _p(a["dev0"], I32P), _p(a["work"], I64P),
        _p(a["cost"], F64P), _p(a["start"], F64P), _p(a["end"], F64P))
    if n < 0:
        raise ValueError("invalid configuration")
    return {k: v[:n] for k, v in a.items()}


def export_program(model, topo, D, T, P, K, B):
    """The explicit global program: values [(dev, bytes, param, returned)]
    and ops [(devs, cost, ins, outs, cls)]."""
    L = lib()
    L.oracle_export_program.restype = ctypes.c_int
    mf = model_fields(model)
    ti, td = topo_arrays(topo)
    sz = np.zeros(5, np.int64)
    base = (_p(mf, I64P), _p(ti, I64P), _p(td, F64P), ctypes.c_int64(D),
            ctypes.c_int64(T), ctypes.c_int64(P), ctypes.c_int64(K),
            ctypes.c_int64(B), _p(sz, I64P))
    if L.oracle_export_program(*base, *([None] * 11)) != 0:
        raise ValueError("invalid configuration")
    nv, no, nd, ni, nout = (int(x) for x in sz)
    vd = np.zeros(nv, np.int32); vb = np.zeros(nv, np.int64)
    vf = np.zeros(nv, np.uint8); oc = np.zeros(no, np.int32)
    ocost = np.zeros(no); ondev = np.zeros(no, np.int32)
    odevs = np.zeros(nd, np.int32); onin = np.zeros(no, np.int32)
    oins = np.zeros(ni, np.int32); onout = np.zeros(no, np.int32)
    oouts = np.zeros(nout, np.int32)
    L.oracle_export_program(
        *base, _p(vd, I32P), _p(vb, I64P), _p(vf, U8P), _p(oc, I32P),
        _p(ocost, F64P), _p(ondev, I32P), _p(odevs, I32P), _p(onin, I32P),
        _p(oins, I32P), _p(onout, I32P), _p(oouts, I32P))
    values = [(int(vd[i]), int(vb[i]), bool(vf[i] & 1), bool(vf[i] & 2))
              for i in range(nv)]
    ops = []
    a = b = c = 0
    for i in range(no):
        devs = odevs[a:a + ondev[i]].tolist(); a += ondev[i]
        ins = oins[b:b + onin[i]].tolist(); b += onin[i]
        outs = oouts[c:c + onout[i]].tolist(); c += onout[i]
        ops.append((devs, float(ocost[i]), ins, outs, int(oc[i])))
    return values, ops


# ------------------------------------------------------------- raw programs --

def simulate_raw(n_dev, ops, values=None):
    """Simulate an explicit program.

    ops: list of (devices, cost) or (devices, cost, inputs, outputs).
    values: list of (device, bytes, is_param, is_returned); default none.
    Returns dict(start, end, clocks, peak, live, makespan, ready_ok)."""
    L = lib()
    values = values or []
    vdev = np.array([v[0] for v in values] or [0], np.int32)
    vb = np.array([v[1] for v in values] or [0], np.int64)
    vf = np.array([(1 if v[2] else 0) | (2 if v[3] else 0) for v in values]
                  or [0], np.uint8)
    ndev, devs, nin, ins, nout, outs, cost = [], [], [], [], [], [], []
    for op in ops:
        d, c = op[0], op[1]
        i = op[2] if len(op) > 2 else []
        o = op[3] if len(op) > 3 else []
        ndev.append(len(d)); devs += list(d)
        nin.append(len(i)); ins += list(i)
        nout.append(len(o)); outs += list(o)
        cost.append(c)
    n = len(ops)
    arr = lambda x, t: np.array(x or [0], t)
    ndev_a, devs_a = arr(ndev, np.int32), arr(devs, np.int32)
    nin_a, ins_a = arr(nin, np.int32), arr(ins, np.int32)
    nout_a, outs_a = arr(nout, np.int32), arr(outs, np.int32)
    cost_a = arr(cost, np.float64)
    st = np.zeros(max(n, 1)); en = np.zeros(max(n, 1))
    ck = np.zeros(n_dev); pk = np.zeros(n_dev, np.int64)
    lv = np.zeros(n_dev, np.int64)
    ms = ctypes.c_double()
    rc = L.oracle_simulate_raw(
        ctypes.c_int32(n_dev), ctypes.c_int32(len(values)), _p(vdev, I32P),
        _p(vb, I64P), _p(vf, U8P), ctypes.c_int32(n), _p(ndev_a, I32P),
        _p(devs_a, I32P), _p(nin_a, I32P), _p(ins_a, I32P),
        _p(nout_a, I32P), _p(outs_a, I32P), _p(cost_a, F64P), _p(st, F64P),
        _p(en, F64P), _p(ck, F64P), _p(pk, I64P), _p(lv, I64P),
        ctypes.byref(ms))
    return dict(start=st[:n], end=en[:n], clocks=ck, peak=pk, live=lv,
                makespan=ms.value, ready_ok=(rc == 0))


# -------------------------------------------------------------------- grids --

def spec_arrays(grid, models=None, topos=None):
    """Pack a workloads grid dict into the oracle's flat spec."""
    from workloads import MODELS, TOPOLOGIES
    models = models or MODELS
    topos = topos or TOPOLOGIES
    mt = np.concatenate([model_fields(models[m]) for m in grid["models"]]) \
        if grid["models"] else np.zeros(13, np.int64)
    tis, tds = zip(*[topo_arrays(topos[t]) for t in grid["topos"]])
    ti = np.concatenate(tis)
    td = np.concatenate(tds)
    nm = len(grid["models"])
    hdr = np.array([nm, len(grid["topos"]), len(grid["world"]),
                    len(grid["batch"]), len(grid["k_set"]), grid["k_mode"],
                    grid["dp_mask"], grid["tp_mask"], grid["pp_mask"],
                    np.int64(np.uint64(grid["synth_seed"]).view(np.int64)),
                    grid["synth_count"]], dtype=np.int64)
    lists = np.array(list(range(nm)) + list(range(len(grid["topos"])))
                     + list(grid["world"]) + list(grid["batch"])
                     + list(grid["k_set"]) + [0], dtype=np.int64)
    return (max(nm, 1), mt, len(grid["topos"]), ti, td, hdr, lists)


def enumerate_grid(grid, with_models=False):
    """Nested-loop enumeration (C.1).  Returns int64 [N, 9]:
    model_slot, topo_slot, W, D, T, P, K, B, kind  (and [N, 13] models)."""
    L = lib()
    nm, mt, nt, ti, td, hdr, lists = spec_arrays(grid)
    args = (ctypes.c_int32(nm), _p(mt, I64P), ctypes.c_int32(nt),
            _p(ti, I64P), _p(td, F64P), _p(hdr, I64P), _p(lists, I64P))
    n = L.oracle_enumerate(*args, ctypes.c_int64(0), None, None)
    f = np.zeros((max(n, 1), 9), np.int64)
    mo = np.zeros((max(n, 1), 13), np.int64)
    L.oracle_enumerate(*args, ctypes.c_int64(n), _p(f, I64P),
                       _p(mo, I64P) if with_models else None)
    return (f[:n], mo[:n]) if with_models else f[:n]


def grid_validity(grid):
    """Validity reason bits (C.2) of every config, without simulating."""
    L = lib()
    nm, mt, nt, ti, td, hdr, lists = spec_arrays(grid)
    args = (ctypes.c_int32(nm), _p(mt, I64P), ctypes.c_int32(nt),
            _p(ti, I64P), _p(td, F64P), _p(hdr, I64P), _p(lists, I64P))
    n = L.oracle_grid_validity(*args, ctypes.c_int64(0), None)
    r = np.zeros(max(n, 1), np.uint32)
    L.oracle_grid_validity(*args, ctypes.c_int64(n), _p(r, U32P))
    return r[:n]


def grid_eval(grid, indices=None, threads=1):
    """Simulate the configs of `grid` at canonical `indices` (all if None).
    Returns dict(makespan, peak, reason, n_ops) arrays aligned with indices."""
    L = lib()
    nm, mt, nt, ti, td, hdr, lists = spec_arrays(grid)
    if indices is None:
        n = len(enumerate_grid(grid))
        idx_p = None
    else:
        idx = np.ascontiguousarray(indices, dtype=np.int64)
        n = len(idx)
        idx_p = _p(idx, I64P)
    ms = np.zeros(max(n, 1)); pk = np.zeros(max(n, 1), np.int64)
    rs = np.zeros(max(n, 1), np.uint32); no = np.zeros(max(n, 1), np.int64)
    bad = L.oracle_grid_eval(
        ctypes.c_int32(nm), _p(mt, I64P), ctypes.c_int32(nt), _p(ti, I64P),
        _p(td, F64P), _p(hdr, I64P), _p(lists, I64P), idx_p,
        ctypes.c_int64(n), ctypes.c_int32(threads), _p(ms, F64P),
        _p(pk, I64P), _p(rs, U32P), _p(no, I64P))
    if bad:
        raise AssertionError("oracle self-check failed on %d configs" % bad)
    return dict(makespan=ms[:n], peak=pk[:n], reason=rs[:n], n_ops=no[:n])


def topk(index, batch, makespan, peak, reason, k):
    """Full-stable-sort top-k (C.8).  Returns (positions, throughputs)."""
    L = lib()
    n = len(index)
    ix = np.ascontiguousarray(index, np.int64)
    bt = np.ascontiguousarray(batch, np.int64)
    ms = np.ascontiguousarray(makespan, np.float64)
    pk = np.ascontiguousarray(peak, np.int64)
    rs = np.ascontiguousarray(reason, np.uint32)
    pos = np.zeros(max(k, 1), np.int64)
    tp = np.zeros(max(k, 1))
    nk = L.oracle_topk(ctypes.c_int64(n), _p(ix, I64P), _p(bt, I64P),
                       _p(ms, F64P), _p(pk, I64P), _p(rs, U32P),
                       ctypes.c_int32(k), _p(pos, I64P), _p(tp, F64P))
    return pos[:nk], tp[:nk]


def grid_result(grid, k=10, threads=1):
    """Whole-grid oracle run: per-config arrays plus the top-k (C.8)."""
    f = enumerate_grid(grid)
    r = grid_eval(grid, threads=threads)
    n = len(f)
    pos, tp = topk(np.arange(n), f[:, 7], r["makespan"], r["peak"],
                   r["reason"], k)
    r.update(fields=f, topk_index=pos, topk_throughput=tp)
    return r
