"""paper_2111_05426_b200 -- B200-native DistIR grid-search simulator pass.

Thin Python binding over ``libdistir.so`` (C ABI in ``include/distir.h``).
This module only marshals arguments: every step of the path (enumerate,
expand, cost, timeline, memory, feasibility, top-k, merge) runs in the CUDA
kernels of ``csrc/``.  PyTorch is used for device memory (the workspace and
device output tensors), streams and process groups.  There is no CPU
fallback: if the shared library is missing, importing the binding raises.

The function names are the C names (``distir_sim_create`` ...); ``Simulator``
is a convenience wrapper that owns a handle and a workspace.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(_HERE)
SO_PATH = os.path.join(_HERE, "libdistir.so")


def _build_lib():
    """csrc/build_lib.py, loaded by path (importing this package needs the
    library it builds)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "distir_build_lib", os.path.join(_HERE, "csrc", "build_lib.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libdistir.so for sm_100a in-tree (nvcc cross-compiles here);
    without `force`, only when a csrc/ source or include/distir.h is newer."""
    return _build_lib().build(out=SO_PATH, verbose=verbose, force=force)


# ------------------------------------------------------------ C structs -----

class distir_model(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "kind", "n_layer", "d_model", "n_head", "seq_len", "vocab_pad",
        "n_ctx", "dtype_bytes", "id_bytes", "lm_head", "schedule", "recompute", "zero")]


class distir_topology(ctypes.Structure):
    _fields_ = [("world_max", ctypes.c_int32), ("node_size", ctypes.c_int32),
                ("flops_per_s", ctypes.c_double),
                ("op_overhead_s", ctypes.c_double),
                ("alpha_intra_s", ctypes.c_double),
                ("bw_intra_Bps", ctypes.c_double),
                ("alpha_inter_s", ctypes.c_double),
                ("bw_inter_Bps", ctypes.c_double),
                ("capacity_bytes", ctypes.c_int64),
                ("cost_model", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("mm_c0_s", ctypes.c_double), ("mm_s_per_flop", ctypes.c_double),
                ("mm_s_per_byte", ctypes.c_double), ("ew_c0_s", ctypes.c_double),
                ("ew_s_per_flop", ctypes.c_double), ("ew_s_per_byte", ctypes.c_double)]


class distir_config(ctypes.Structure):
    _fields_ = [("dp", ctypes.c_int32), ("tp", ctypes.c_int32),
                ("pp", ctypes.c_int32), ("microbatches", ctypes.c_int32),
                ("batch", ctypes.c_int64), ("model", ctypes.c_int32),
                ("topo", ctypes.c_int32)]


class distir_grid_spec(ctypes.Structure):
    _fields_ = [("n_world", ctypes.c_int32), ("world", ctypes.c_int32 * 8),
                ("k_mode", ctypes.c_int32), ("n_k", ctypes.c_int32),
                ("k_set", ctypes.c_int32 * 16), ("n_batch", ctypes.c_int32),
                ("batch", ctypes.c_int64 * 32), ("n_models", ctypes.c_int32),
                ("models", ctypes.c_int32 * 8), ("n_topos", ctypes.c_int32),
                ("topos", ctypes.c_int32 * 8), ("dp_mask", ctypes.c_uint32),
                ("tp_mask", ctypes.c_uint32), ("pp_mask", ctypes.c_uint32),
                ("synth_seed", ctypes.c_uint64),
                ("synth_count", ctypes.c_int64)]


class distir_topk_entry(ctypes.Structure):
    _fields_ = [("index", ctypes.c_int64), ("makespan_s", ctypes.c_double),
                ("throughput", ctypes.c_double),
                ("peak_bytes", ctypes.c_int64)]


class distir_profile_data(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64), ("kernels", ctypes.c_int64),
                ("ms_prepare", ctypes.c_double), ("ms_simulate", ctypes.c_double),
                ("ms_topk", ctypes.c_double), ("ms_merge", ctypes.c_double)]


class distir_stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "n_configs", "n_valid", "n_feasible", "op_events", "stage_steps",
        "n_buckets", "n_items", "h2d_bytes", "d2h_bytes", "tasks", "slow_tasks",
        "wave_steps")]


_STATS_FIELDS = tuple(f for f, _ in distir_stats._fields_)


class distir_raw_op(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "n_dev", "dev_off", "n_in", "in_off", "n_out", "out_off")] + [
        ("cost", ctypes.c_double)]


class distir_raw_value(ctypes.Structure):
    _fields_ = [("dev", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("bytes", ctypes.c_int64)]


class distir_raw_program(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "n_dev", "n_ops", "op_base", "n_values", "value_base", "out_base")]


TOPK_DTYPE = np.dtype([("index", "<i8"), ("makespan_s", "<f8"),
                       ("throughput", "<f8"), ("peak_bytes", "<i8")])

STATUS = {0: "DISTIR_OK", 1: "DISTIR_E_INVALID_ARG", 2: "DISTIR_E_UNSUPPORTED",
          3: "DISTIR_E_OUT_OF_MEMORY", 4: "DISTIR_E_CUDA", 5: "DISTIR_E_NCCL",
          6: "DISTIR_E_WORKSPACE"}

# Every symbol include/distir.h declares (checked by the CPU tests).
EXPORTS = ("distir_sim_create", "distir_sim_destroy", "distir_grid_size",
           "distir_workspace_size", "distir_grid_eval", "distir_grid_upload",
           "distir_grid_launch", "distir_last_stats", "distir_profile",
           "distir_grid_eval_sharded", "distir_nccl_unique_id",
           "distir_nccl_comm_init", "distir_nccl_comm_destroy",
           "distir_shard_indices", "distir_raw_workspace_size",
           "distir_raw_eval", "distir_topk_merge", "distir_last_error",
           "distir_version", "distir_result_layout")


class DistirError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status


def _load():
    if not os.path.exists(SO_PATH):
        raise ImportError(
            "libdistir.so not built (%s); run __graft_entry__.build() -- the "
            "DistIR path has no CPU fallback" % SO_PATH)
    L = ctypes.CDLL(SO_PATH)
    vp, i32, i64, u32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
    P = ctypes.POINTER
    L.distir_last_error.restype = ctypes.c_char_p
    L.distir_version.restype = ctypes.c_char_p
    L.distir_sim_create.argtypes = [P(distir_model), i32, P(distir_topology), i32,
                                    i32, vp, P(vp)]
    L.distir_sim_destroy.argtypes = [vp]
    L.distir_sim_destroy.restype = None
    L.distir_grid_size.argtypes = [vp, P(distir_grid_spec), P(i64)]
    L.distir_workspace_size.argtypes = [vp, i64, P(ctypes.c_size_t)]
    L.distir_result_layout.argtypes = [vp, i64, P(i64), P(ctypes.c_size_t)]
    L.distir_grid_eval.argtypes = [vp, P(distir_grid_spec), P(distir_config), i64,
                                   i32, vp, ctypes.c_size_t, vp, vp, vp, vp,
                                   P(i32), P(distir_stats)]
    L.distir_grid_upload.argtypes = [vp, P(distir_grid_spec), P(distir_config), i64,
                                     i32, i32, vp, ctypes.c_size_t, P(i64)]
    L.distir_grid_launch.argtypes = [vp, i32, vp, vp, ctypes.c_size_t, vp, vp, vp, vp, vp]
    L.distir_profile.argtypes = [vp, i32, P(distir_profile_data)]
    L.distir_last_stats.argtypes = [vp, vp, P(distir_stats)]
    L.distir_grid_eval_sharded.argtypes = [vp, P(distir_grid_spec), P(distir_config),
                                           i64, i32, i32, vp, i32, vp, ctypes.c_size_t,
                                           vp, vp, vp, vp, P(i32), P(distir_stats)]
    L.distir_nccl_unique_id.argtypes = [ctypes.c_char_p]
    L.distir_nccl_comm_init.argtypes = [ctypes.c_char_p, i32, i32, i32, P(vp)]
    L.distir_nccl_comm_destroy.argtypes = [vp]
    L.distir_shard_indices.argtypes = [i64, i32, i32, P(i64), i64]
    L.distir_raw_workspace_size.argtypes = [i32, i64, i64, i64, i64, P(ctypes.c_size_t)]
    L.distir_raw_eval.argtypes = [vp, P(distir_raw_program), i32, P(distir_raw_op), i64,
                                  P(i32), i64, P(distir_raw_value), i64, i64, vp,
                                  ctypes.c_size_t, vp, vp, vp, vp, vp]
    L.distir_topk_merge.argtypes = [vp, vp, vp, i32, i32, i32, vp, vp]
    L.distir_shard_indices.restype = i64
    for f in EXPORTS:
        if f not in ("distir_sim_destroy", "distir_last_error", "distir_version",
                     "distir_shard_indices"):
            getattr(L, f).restype = ctypes.c_int
    return L


lib = _load()


def _check(status):
    if status != 0:
        raise DistirError(status, lib.distir_last_error().decode())


# ------------------------------------------------------ marshalling ---------

def model_struct(m) -> distir_model:
    return distir_model(*[int(m.get(k, 0)) for k in (
        "kind", "n_layer", "d_model", "n_head", "seq_len", "vocab_pad",
        "n_ctx", "dtype_bytes", "id_bytes", "lm_head", "schedule", "recompute", "zero")])


def topo_struct(t) -> distir_topology:
    return distir_topology(int(t["world_max"]), int(t["node_size"]),
                           float(t["flops_per_s"]), float(t["op_overhead_s"]),
                           float(t["alpha_intra_s"]), float(t["bw_intra_Bps"]),
                           float(t["alpha_inter_s"]), float(t["bw_inter_Bps"]),
                           int(t["capacity_bytes"]), int(t.get("cost_model", 0)), 0,
                           *[float(t.get(k, 0.0)) for k in (
                               "mm_c0_s", "mm_s_per_flop", "mm_s_per_byte",
                               "ew_c0_s", "ew_s_per_flop", "ew_s_per_byte")])


def spec_struct(grid, model_index, topo_index) -> distir_grid_spec:
    """workloads grid dict -> distir_grid_spec; model/topo names are mapped
    through the handle's index dicts."""
    s = distir_grid_spec()
    s.n_world = len(grid["world"])
    for i, w in enumerate(grid["world"]):
        s.world[i] = w
    s.k_mode = grid["k_mode"]
    s.n_k = len(grid["k_set"])
    for i, k in enumerate(grid["k_set"]):
        s.k_set[i] = k
    s.n_batch = len(grid["batch"])
    for i, b in enumerate(grid["batch"]):
        s.batch[i] = b
    s.n_models = len(grid["models"])
    for i, m in enumerate(grid["models"]):
        s.models[i] = model_index[m]
    s.n_topos = len(grid["topos"])
    for i, t in enumerate(grid["topos"]):
        s.topos[i] = topo_index[t]
    s.dp_mask, s.tp_mask, s.pp_mask = (grid["dp_mask"], grid["tp_mask"],
                                       grid["pp_mask"])
    s.synth_seed = grid["synth_seed"]
    s.synth_count = grid["synth_count"]
    return s


def configs_array(configs):
    """[(model_idx, topo_idx, D, T, P, K, B)] -> ctypes array."""
    arr = (distir_config * max(len(configs), 1))()
    for i, (mi, ti, D, T, P, K, B) in enumerate(configs):
        arr[i] = distir_config(D, T, P, K, B, mi, ti)
    return arr


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


# ------------------------------------------------------------ wrapper -------

class Simulator:
    """Owns a distir_sim handle bound to one GPU and one torch stream."""

    def __init__(self, models, topologies, device=0, stream=None):
        import torch
        self.torch = torch
        self.model_names = list(models)
        self.topo_names = list(topologies)
        self.model_index = {n: i for i, n in enumerate(self.model_names)}
        self.topo_index = {n: i for i, n in enumerate(self.topo_names)}
        ms = (distir_model * len(models))(*[model_struct(models[n])
                                            for n in self.model_names])
        ts = (distir_topology * len(topologies))(
            *[topo_struct(topologies[n]) for n in self.topo_names])
        self.device = torch.device("cuda", device)
        self.stream = stream or torch.cuda.current_stream(self.device)
        h = ctypes.c_void_p()
        _check(lib.distir_sim_create(ms, len(models), ts, len(topologies),
                                     device, ctypes.c_void_p(self.stream.cuda_stream),
                                     ctypes.byref(h)))
        self.handle = h
        self.ws = None

    def close(self):
        if self.handle:
            lib.distir_sim_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- sizes
    def spec(self, grid):
        return spec_struct(grid, self.model_index, self.topo_index)

    def grid_size(self, grid) -> int:
        n = ctypes.c_int64()
        _check(lib.distir_grid_size(self.handle, ctypes.byref(self.spec(grid)),
                                    ctypes.byref(n)))
        return n.value

    def workspace(self, n_configs):
        if getattr(self, "_ws_n", None) == n_configs and self.ws is not None:
            return self.ws
        b = ctypes.c_size_t()
        _check(lib.distir_workspace_size(self.handle, n_configs, ctypes.byref(b)))
        self._ws_n = n_configs
        if self.ws is None or self.ws.numel() < b.value:
            self.ws = self.torch.empty(b.value, dtype=self.torch.uint8,
                                       device=self.device)
        return self.ws

    # -- synchronous evaluation with host buffers (the e2e path)
    def eval(self, grid=None, configs=None, k=10, per_config=True, pinned=True,
             rank=0, n_ranks=1, comm=None, copy=True):
        """Synchronous evaluation through distir_grid_eval_sharded with host
        buffers (spec H2D and results D2H inside the call).  Per-config
        outputs are global-indexed numpy arrays (only this rank's entries are
        written when n_ranks > 1): copies, or with copy=False views of the
        handle's pinned buffers that the next call overwrites."""
        torch = self.torch
        if grid is not None:
            # re-marshal the spec only when the grid changed (dict equality,
            # against a copy, so in-place edits of the caller's dict count)
            src = getattr(self, "_spec_src", None)
            if src is None or grid != src:
                self._spec_cache = (self.spec(grid), self.grid_size(grid))
                self._spec_src = {k: (list(v) if isinstance(v, list) else v)
                                  for k, v in grid.items()}
            sp, n = self._spec_cache
            cf, ncf = None, 0
        else:
            sp = None
            cf = configs_array(configs)
            n = ncf = len(configs)
        ws = self.workspace(n)
        outs = {}
        if per_config:
            bufs = getattr(self, "_host_bufs", None)
            if bufs is None or bufs[4] != n or bufs[3] != pinned:
                # the library's packed result layout for n configurations
                # (distir_result_layout): the three arrays arrive in one
                # copy.  One pinned buffer, grown when too small, carved per n
                # (so copy=False views are overwritten by the next call)
                m = max(n, 1)
                off = (ctypes.c_int64 * 3)()
                nb = ctypes.c_size_t()
                _check(lib.distir_result_layout(self.handle, m, off, ctypes.byref(nb)))
                raw = getattr(self, "_host_raw", None)
                if raw is None or raw.numel() < nb.value or self._host_raw_pinned != pinned:
                    raw = self._host_raw = torch.empty(nb.value, dtype=torch.uint8, pin_memory=pinned)
                    self._host_raw_pinned = pinned
                bufs = (raw[off[0]:off[0] + 8 * m].view(torch.float64),
                        raw[off[1]:off[1] + 8 * m].view(torch.int64),
                        raw[off[2]:off[2] + 4 * m].view(torch.int32), pinned, n)
                self._host_bufs = bufs
                # numpy views and raw pointers, made once per carving
                self._host_np = tuple(t.numpy() for t in bufs[:3])
                self._host_ptr = tuple(ctypes.c_void_p(t.data_ptr()) for t in bufs[:3])
            outs = {"makespan": bufs[0], "peak": bufs[1], "reason": bufs[2]}
            if n_ranks > 1:       # entries of other ranks stay untouched: mark them
                bufs[0][:n].fill_(float("nan"))
                bufs[1][:n].fill_(-2)
                bufs[2][:n].fill_(-1)
            ptrs = self._host_ptr
        else:
            ptrs = (None, None, None)
        topk = np.zeros(max(k, 1), dtype=TOPK_DTYPE) if copy else self._topk_buf(k)
        ntopk = ctypes.c_int32()
        st = distir_stats()
        _check(lib.distir_grid_eval_sharded(
            self.handle, ctypes.byref(sp) if sp is not None else None,
            cf, ncf, rank, n_ranks, comm, k, ctypes.c_void_p(ws.data_ptr()),
            ws.numel(), ptrs[0], ptrs[1], ptrs[2],
            topk.ctypes.data_as(ctypes.c_void_p), ctypes.byref(ntopk),
            ctypes.byref(st)))
        res = dict(topk=topk[:ntopk.value], n=n,
                   stats={f: getattr(st, f) for f in _STATS_FIELDS})
        if per_config:
            for name, a in zip(("makespan", "peak", "reason"), self._host_np):
                res[name] = a[:n].copy() if copy else a[:n]
            res["reason"] = res["reason"].view(np.uint32)
        return res

    def _topk_buf(self, k):
        b = getattr(self, "_topk_host", None)
        if b is None or len(b) < max(k, 1):
            b = self._topk_host = np.zeros(max(k, 1), dtype=TOPK_DTYPE)
        return b[:max(k, 1)]

    # -- device-resident pipeline (the timed `value` path)
    def upload(self, grid=None, configs=None, rank=0, n_ranks=1):
        if grid is not None:
            self._sp = self.spec(grid)
            n = self.grid_size(grid)
            self._cf, ncf = None, 0
        else:
            self._sp = None
            self._cf = configs_array(configs)
            n = ncf = len(configs)
        ws = self.workspace(n)
        nl = ctypes.c_int64()
        _check(lib.distir_grid_upload(
            self.handle, ctypes.byref(self._sp) if self._sp is not None else None,
            self._cf, ncf, rank, n_ranks, ctypes.c_void_p(ws.data_ptr()), ws.numel(),
            ctypes.byref(nl)))
        return nl.value

    def device_outputs(self, n_local, k=10):
        torch = self.torch
        return dict(
            makespan=torch.empty(max(n_local, 1), dtype=torch.float64, device=self.device),
            peak=torch.empty(max(n_local, 1), dtype=torch.int64, device=self.device),
            reason=torch.empty(max(n_local, 1), dtype=torch.int32, device=self.device),
            topk=torch.empty((max(k, 1), 4), dtype=torch.int64, device=self.device),
            ntopk=torch.zeros(1, dtype=torch.int32, device=self.device))

    def launch(self, outs, k=10, per_config=True, comm=None):
        ws = self.ws
        _check(lib.distir_grid_launch(
            self.handle, k, comm, ctypes.c_void_p(ws.data_ptr()), ws.numel(),
            _ptr(outs["makespan"]) if per_config else None,
            _ptr(outs["peak"]) if per_config else None,
            _ptr(outs["reason"]) if per_config else None,
            _ptr(outs["topk"]), _ptr(outs["ntopk"])))

    def merge_topk(self, lists, counts=None, k=10):
        """Device merge of sorted top-k lists (row a8, distir_topk_merge).
        lists: int64 CUDA tensor (n_lists, k_in, 4) of records as
        distir_grid_launch writes them; counts: int32 CUDA tensor (n_lists,)
        or None (records with index >= 0).  Returns (topk (k, 4) int64
        tensor, n (1,) int32 tensor), asynchronously on the handle's stream."""
        torch = self.torch
        assert lists.is_cuda and lists.dtype == torch.int64 and lists.dim() == 3
        lists = lists.contiguous()
        out = torch.empty((max(k, 1), 4), dtype=torch.int64, device=lists.device)
        n = torch.zeros(1, dtype=torch.int32, device=lists.device)
        if counts is not None:
            counts = counts.to(torch.int32).contiguous()
        _check(lib.distir_topk_merge(self.handle, _ptr(lists),
                                     _ptr(counts) if counts is not None else None,
                                     lists.shape[0], lists.shape[1], k, _ptr(out), _ptr(n)))
        return out, n

    # -- raw-program mode (f3)
    def eval_raw(self, programs, per_op=True):
        """Simulate explicit programs on the GPU.  programs: list of
        (n_dev, ops, values) with ops = [(devs, cost, ins, outs), ...] and
        values = [(dev, bytes, is_param, is_returned), ...] (ids local to the
        program).  Returns a list of dicts (makespan, clocks, peak, start,
        end)."""
        progs = (distir_raw_program * max(len(programs), 1))()
        ops_l, idx, vals = [], [], []
        out_base = 0
        for p, (n_dev, ops, values) in enumerate(programs):
            progs[p] = distir_raw_program(n_dev, len(ops), len(ops_l), len(values),
                                          len(vals), out_base)
            out_base += n_dev
            for op in ops:
                devs, cost = op[0], op[1]
                ins = op[2] if len(op) > 2 else []
                outs = op[3] if len(op) > 3 else []
                rec = (len(devs), len(idx), len(ins), len(idx) + len(devs), len(outs),
                       len(idx) + len(devs) + len(ins), float(cost))
                idx.extend(list(devs) + list(ins) + list(outs))
                ops_l.append(rec)
            for v in values:
                vals.append((int(v[0]), (1 if v[2] else 0) | (2 if v[3] else 0), int(v[1])))
        n_ops, n_idx, n_vals = len(ops_l), len(idx), len(vals)
        ops_a = (distir_raw_op * max(n_ops, 1))(*[distir_raw_op(*r) for r in ops_l])
        idx_a = (ctypes.c_int32 * max(n_idx, 1))(*idx)
        vals_a = (distir_raw_value * max(n_vals, 1))(*[distir_raw_value(*v) for v in vals])
        b = ctypes.c_size_t()
        _check(lib.distir_raw_workspace_size(len(programs), n_ops, n_idx, n_vals, out_base,
                                             ctypes.byref(b)))
        ws = self.torch.empty(b.value, dtype=self.torch.uint8, device=self.device)
        ms = np.zeros(max(len(programs), 1))
        clk = np.zeros(max(out_base, 1))
        pk = np.zeros(max(out_base, 1), dtype=np.int64)
        st = np.zeros(max(n_ops, 1))
        en = np.zeros(max(n_ops, 1))
        vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)
        _check(lib.distir_raw_eval(self.handle, progs, len(programs), ops_a, n_ops, idx_a,
                                   n_idx, vals_a, n_vals, out_base,
                                   ctypes.c_void_p(ws.data_ptr()), ws.numel(), vp(ms), vp(clk),
                                   vp(pk), vp(st) if per_op else None,
                                   vp(en) if per_op else None))
        res = []
        for p, (n_dev, ops, values) in enumerate(programs):
            o, ob = progs[p].op_base, progs[p].out_base
            res.append(dict(makespan=ms[p], clocks=clk[ob:ob + n_dev].copy(),
                            peak=pk[ob:ob + n_dev].copy(),
                            start=st[o:o + len(ops)].copy() if per_op else None,
                            end=en[o:o + len(ops)].copy() if per_op else None))
        return res

    def profile(self, enable=True):
        """Kernel times (ms) accumulated since the previous call; then turn
        CUDA-event recording on or off."""
        pd = distir_profile_data()
        _check(lib.distir_profile(self.handle, 1 if enable else 0, ctypes.byref(pd)))
        return {f: getattr(pd, f) for f, _ in distir_profile_data._fields_}

    def last_stats(self):
        st = distir_stats()
        _check(lib.distir_last_stats(self.handle, ctypes.c_void_p(self.ws.data_ptr()),
                                     ctypes.byref(st)))
        return {f: getattr(st, f) for f, _ in distir_stats._fields_}


def topk_from_device(t, n):
    """Device top-k tensor [k, 4] (int64 view of distir_topk_entry) -> numpy."""
    a = t.cpu().numpy()[:n].copy()
    return a.view(TOPK_DTYPE).reshape(-1)


# ---------------------------------------------------------------- NCCL ------

def distir_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib.distir_nccl_unique_id(buf))
    return buf.raw


def distir_nccl_comm_init(uid: bytes, n_ranks: int, rank: int, device: int):
    comm = ctypes.c_void_p()
    _check(lib.distir_nccl_comm_init(uid, n_ranks, rank, device, ctypes.byref(comm)))
    return comm


def distir_nccl_comm_destroy(comm):
    _check(lib.distir_nccl_comm_destroy(comm))


def distir_shard_indices(n_configs: int, rank: int, n_ranks: int) -> np.ndarray:
    n = lib.distir_shard_indices(n_configs, rank, n_ranks, None, 0)
    out = np.zeros(max(n, 1), dtype=np.int64)
    lib.distir_shard_indices(n_configs, rank, n_ranks,
                             out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), n)
    return out[:n]


def distir_version() -> str:
    return lib.distir_version().decode()
