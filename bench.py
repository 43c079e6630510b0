#!/usr/bin/env python
"""bench.py -- the DistIR grid-search simulator pass on B200 (driver contract).

One "step" = one pass of the whole hot path over one
grid: enumerate, expand (D/T/P + GPipe), cost, timeline, memory, feasibility,
top-k and (N > 1) the all-gather merge.

Workload (BASELINE.json north_star: ">= 10^8 simulated op-events/sec per B200
on the GPT-2 grid"): W3, the GPT-2 small/medium/large/XL inference grid,
W <= 16, B in 2^7..2^20, on the TB200 topology -- 8,680 configs.  With N GPUs
the grid is widened to N topologies (TB200, TM0, ..., TM{N-2}) and dealt
round-robin over the ranks, so per-GPU work stays fixed ("scaling": "weak").

  value       op-events/s, device-timed (CUDA events around each launch,
              inputs resident in HBM, L2 flushed between steps), max over ranks
  e2e         the same metric through the public API with host buffers
              (spec H2D, per-config results + top-k D2H inside the timing)
  roofline    k_simulate (the dominant kernel) against the SM issue ceiling
              (warp instructions per launch from the committed ncu capture of
              this source tree), with the HBM-equivalent logical rate and the
              measured DRAM bytes beside it
  strong      fixed grids (W3 x 8 topologies, W5) dealt over the N ranks:
              strong scaling, time = max over ranks
  cpu_baseline the CPU oracle on a bounded sample of the same grid (rank 0,
              N=1): all host threads and one thread, CPU model

`--impl reference` times the CPU oracle (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "simulated op-events/sec (GPT-2 inference grid W3, DistIR simulator pass)"
UNIT = "op-events/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="distir", choices=["distir", "reference"])
    ap.add_argument("--workload", default="W3")
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--e2e-steps", type=int, default=0,
                    help="end-to-end steps (default: min(steps, 50))")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--nccl", action="store_true",
                    help="N=1: run row a8 (NCCL all-gather of the top-k + device merge) "
                         "through a 1-rank communicator inside the timed loop")
    ap.add_argument("--no-strong", action="store_true",
                    help="skip the fixed-grid (strong-scaling) legs")
    return ap.parse_args()


def bench_grid(name, n_gpus):
    g = dict(W.GRIDS[name])
    if n_gpus > 1 and g["synth_count"] == 0:
        g["topos"] = (list(g["topos"]) + W.TM)[:n_gpus]
    return g


def bench_config(name, grid, n_total, k, n_gpus):
    return {"workload": "%s: %s x %s, %d configs" % (
        name, "+".join(grid["models"]) or "synthetic", "+".join(grid["topos"]), n_total),
        "configs": n_total, "k": k, "l2_flush": "256 MiB memset between steps",
        "parallelism": ("round-robin config shards x %d GPUs, NCCL all-gather of top-k"
                        % n_gpus) if n_gpus > 1 else "1 GPU"}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


# -------------------------------------------------------------- clocks ------

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        time.sleep(0.15)
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()

    def summary(self):
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for r in rows:
            r = [x.strip() for x in r]
            if len(r) < 9:
                continue
            try:
                sm.append(float(r[1]))
                mx.append(float(r[2]))
            except ValueError:
                continue
            for nm, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.f.name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        load = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": float(np.median(load)), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------- CPU baseline -----

def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_oracle_rate(grid, seconds, seed=20211105426, threads=None):
    """Time the oracle (as it stands) on a seeded random sample of the grid
    for about `seconds` of wall time on `threads` host threads (configs are
    handed out one at a time); op-events/s.  Calls grow geometrically, each
    sized to about half the remaining time at the rate measured so far, so
    the threads rarely wait for each other at a call's end and the total
    stays near `seconds` (configs differ in size by orders of magnitude)."""
    import oracle
    oracle.build()
    threads = threads or os.cpu_count() or 1
    n = len(oracle.enumerate_grid(grid)) if grid["synth_count"] == 0 else grid["synth_count"]
    order = np.random.default_rng(seed).permutation(n)
    ops, cfgs, dt, pos = 0, 0, 0.0, 0
    while pos < n and dt < 0.9 * seconds:
        if cfgs == 0:
            m = threads
        else:
            m = max(threads, int(0.5 * (seconds - dt) * cfgs / dt))
        m = min(m, n - pos)
        idx = np.sort(order[pos:pos + m])
        pos += m
        t = time.perf_counter()
        r = oracle.grid_eval(grid, indices=idx, threads=threads)
        dt += time.perf_counter() - t
        ops += int(r["n_ops"][(r["reason"] & 0x1F) == 0].sum())
        cfgs += len(idx)
    return dict(value=ops / dt, ops=ops, configs=cfgs, seconds=dt, threads=threads)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    grid = bench_grid(args.workload, args.gpus)
    import oracle
    oracle.build()
    n = len(oracle.enumerate_grid(grid))
    rng = np.random.default_rng(11)
    order = rng.permutation(n)
    threads = os.cpu_count() or 1
    # each step: seeded random configs of the grid, 4 per thread at a time, for
    # a bounded time, so that the whole --steps/--warmup run ends in minutes
    budget = min(0.25, 100.0 / max(args.steps + args.warmup, 1))
    pos = 0
    cfg_total = 0

    def step():
        nonlocal pos, cfg_total
        ops, dt = 0, 0.0
        while True:
            idx = np.sort(order[pos % n: pos % n + 4 * threads])
            pos += 4 * threads
            t = time.perf_counter()
            r = oracle.grid_eval(grid, indices=idx, threads=threads)
            dt += time.perf_counter() - t
            ops += int(r["n_ops"][(r["reason"] & 0x1F) == 0].sum())
            cfg_total += len(idx)
            if dt >= budget:
                return ops, dt

    for _ in range(args.warmup):
        step()
    ops = 0
    tt = 0.0
    for _ in range(args.steps):
        o, dt = step()
        ops += o
        tt += dt
    v = ops / tt
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * tt / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": bench_config(args.workload, grid, n, args.k, args.gpus),
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                            "sample": "%d seeded random configs of %s over %d steps "
                                      "(%.2f s each), %d threads"
                                      % (cfg_total, args.workload, args.steps + args.warmup,
                                         budget, threads)},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


# ------------------------------------------------------------- roofline -----

def source_sha():
    """sha256 over the library's sources (csrc/*.cu*, include/distir.h): the
    key under which an ncu capture of k_simulate is valid for this build."""
    import hashlib
    h = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_2111_05426_b200", "csrc")
    for f in sorted(os.listdir(csrc)):
        if f.endswith((".cu", ".cuh")):
            with open(os.path.join(csrc, f), "rb") as fh:
                h.update(f.encode() + fh.read())
    with open(os.path.join(ROOT, "include", "distir.h"), "rb") as fh:
        h.update(fh.read())
    return h.hexdigest()[:16]


def ncu_capture():
    """The committed `ncu --set full` summary of the dominant kernel
    (profiles/ncu_simulate_summary.json, written by tools/ncu_capture.py)."""
    p = os.path.join(ROOT, "profiles", "ncu_simulate_summary.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        return json.load(f)


def roofline(prof, stats, n_sm, sm_mhz, peaks, peak_kind):
    """k_simulate (the dominant kernel) against the bound that binds it: SM
    instruction issue.  It is a latency-/issue-bound integer + fp64 scalar
    kernel (no tensor cores: nothing on the path is a dense contraction; HBM
    traffic is ~150 KB per launch).  achieved = warp instructions per launch
    (ncu capture of this source tree) / its live CUDA-event time; peak = SMs x
    4 schedulers x 1 warp instruction / clock.  Beside it: north_star's
    HBM-equivalent rate (16 B per op-event, SURVEY D.3 -- a LOGICAL rate: the
    kernel never moves those bytes, exact aggregation skips the per-op work)
    and the DRAM bytes ncu measured."""
    sim_ms = prof["ms_simulate"] / max(prof["launches"], 1)
    sim_s = sim_ms / 1e3
    cap = ncu_capture()
    sha = source_sha()
    fresh = cap is not None and cap.get("source_sha") == sha
    inst = cap.get("inst_executed_per_launch") if cap else None
    dram = cap.get("dram_bytes_per_launch") if cap else None
    issue_peak = n_sm * 4 * sm_mhz * 1e6
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    achieved = inst / sim_s if inst else None
    logical = 16.0 * stats["op_events"] / sim_s / 1e9
    return {
        "bound": "alu", "unit": "warp-instructions/s",
        "achieved": achieved, "peak": issue_peak,
        "frac": achieved / issue_peak if achieved else None,
        "traffic": dram,
        "kernel": "k_simulate (a2-a6)", "kernel_ms": sim_ms,
        "instructions_per_launch": inst,
        "capture": {"file": "profiles/ncu_simulate_summary.json",
                    "source_sha": cap.get("source_sha") if cap else None,
                    "this_source_sha": sha, "fresh": fresh,
                    "workload": cap.get("workload") if cap else None},
        "peak_note": "%d SMs x 4 SMSPs x 1 warp-instr/clk x %.0f MHz (SM clock under load)"
                     % (n_sm, sm_mhz),
        "dram": {"bytes_per_launch": dram,
                 "GBps": dram / sim_s / 1e9 if dram else None,
                 "frac_of_hbm": dram / sim_s / 1e9 / hbm if dram else None},
        "hbm_equivalent": {"bytes_per_op_event": 16, "GBps": logical,
                           "peak_GBps": hbm, "frac": logical / hbm,
                           "peak_kind": peak_kind,
                           "note": "logical rate (op-events x 16 B / k_simulate time); "
                                   "not traffic -- see dram"},
    }


# --------------------------------------------------------------- main -------

def timed(sim, outs, k, comm, steps, flush, stream, barrier):
    """Device time per launch (ms, CUDA events on the library's stream, L2
    flushed before each launch)."""
    import torch
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    barrier()
    for i in range(steps):
        flush.zero_()
        evs[i][0].record(stream)
        sim.launch(outs, k=k, comm=comm)
        evs[i][1].record(stream)
    barrier()
    return sum(a.elapsed_time(b) for a, b in evs) / steps


def strong_leg(sim, name, grid, k, comm, rank, world, steps, warmup, flush, stream, barrier,
               reduce_max, reduce_sum):
    """A FIXED grid dealt round-robin over the `world` ranks (strong scaling):
    op-events/s of the whole grid, time = max over ranks."""
    n_total = sim.grid_size(grid)
    n_local = sim.upload(grid, rank=rank, n_ranks=world)
    outs = sim.device_outputs(n_local, k=k)
    for _ in range(warmup):
        sim.launch(outs, k=k, comm=comm)
    barrier()
    ops = float(sim.last_stats()["op_events"])
    ms = reduce_max(timed(sim, outs, k, comm, steps, flush, stream, barrier))
    ops = reduce_sum(ops)
    return {"workload": "%s: %d configs (%s x %s)" % (
                name, n_total, "+".join(grid["models"]) or "synthetic",
                "+".join(grid["topos"])),
            "value": ops / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "n_gpus": world,
            "steps": steps, "configs_per_s": n_total / (ms / 1e3)}


STRONG = [("W3x8", dict(W.GRIDS["W3"], topos=["TB200"] + W.TM[:7])), ("W5", W.GRIDS["W5"])]


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    from paper_2111_05426_b200 import (Simulator, distir_nccl_comm_init,
                                       distir_nccl_comm_destroy,
                                       distir_nccl_unique_id)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n_gpus = world
    grid = bench_grid(args.workload, n_gpus)
    sim = Simulator(W.MODELS, W.TOPOLOGIES, device=local)
    comm = None
    if world > 1 or args.nccl:
        if world > 1:
            obj = [distir_nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid = obj[0]
        else:
            uid = distir_nccl_unique_id()
        comm = distir_nccl_comm_init(uid, world, rank, local)
    k = args.k
    n_total = sim.grid_size(grid)
    n_local = sim.upload(grid, rank=rank, n_ranks=world)
    outs = sim.device_outputs(n_local, k=k)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    stream = sim.stream

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def reduce_max(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def reduce_sum(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # warm-up
    for _ in range(args.warmup):
        sim.launch(outs, k=k, comm=comm)
    barrier()
    stats = sim.last_stats()

    # ---- device-timed region (inputs resident in HBM; the library's own
    # per-phase CUDA events are off here: they add event-record nodes)
    K = args.steps
    with ClockSampler(local) as clk:
        ms_step = timed(sim, outs, k, comm, K, flush, stream, barrier)
    clocks = clk.summary()
    # ---- per-kernel breakdown (distir_profile: CUDA events on the library's
    # stream around each phase) over a separate pass of the same launches
    sim.profile(True)
    timed(sim, outs, k, comm, min(K, 200), flush, stream, barrier)
    prof = sim.profile(False)
    kernels_per_launch = prof["kernels"] / max(prof["launches"], 1)
    tk_dev = outs["topk"].cpu()
    ntk = int(outs["ntopk"].item())

    # ---- end-to-end through the public API (host buffers)
    E = args.e2e_steps or min(K, 50)
    # (copy=False: the results are read into the handle's pinned buffers
    # every step -- the D2H is inside the timing -- without an extra host copy)
    for _ in range(2):
        sim.eval(grid, k=k, rank=rank, n_ranks=world, comm=comm, copy=False)
    barrier()
    t0 = time.perf_counter()
    for _ in range(E):
        res = sim.eval(grid, k=k, rank=rank, n_ranks=world, comm=comm, copy=False)
    barrier()
    e2e_ms = 1e3 * (time.perf_counter() - t0) / E
    est = res["stats"]
    assert res["topk"]["index"].tolist() == \
        tk_dev.numpy()[:ntk].view(np.int64).reshape(-1, 4)[:, 0].tolist()

    # ---- fixed-grid legs (strong scaling: the same grid at every N)
    strong = []
    if not args.no_strong:
        for name, g in STRONG:
            strong.append(strong_leg(sim, name, g, k, comm, rank, world,
                                     min(K, 50 if name == "W5" else 200), 3, flush, stream,
                                     barrier, reduce_max, reduce_sum))

    # ---- reduce over ranks
    ms_step = reduce_max(ms_step)
    e2e_ms = reduce_max(e2e_ms)
    ops_all = reduce_sum(float(stats["op_events"]))
    steps_all = reduce_sum(float(stats["stage_steps"]))
    h2d_all = reduce_sum(float(est["h2d_bytes"]))
    d2h_all = reduce_sum(float(est["d2h_bytes"]))

    if rank == 0:
        peaks, peak_kind = measured_peaks()
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
        sm_mhz = clocks["sm_mhz"] or float(peaks.get("sm_max_mhz", 1965.0))
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            c = cpu_oracle_rate(grid, args.cpu_seconds)
            c1 = cpu_oracle_rate(grid, args.cpu_seconds / 3, seed=7, threads=1)
            cpu = {"value": c["value"], "unit": UNIT, "cores": c["threads"],
                   "kind": "oracle", "cpu_model": cpu_model(),
                   "sample": "seeded random %d of %d %s configs (%d op-events), %.1f s, "
                             "%d threads (configs handed out one at a time)"
                             % (c["configs"], n_total, args.workload, c["ops"],
                                c["seconds"], c["threads"]),
                   "one_thread": {"value": c1["value"], "unit": UNIT, "cores": 1,
                                  "sample": "seeded random %d configs (%d op-events), %.1f s"
                                            % (c1["configs"], c1["ops"], c1["seconds"])}}
        value = ops_all / (ms_step / 1e3)
        cfg = bench_config(args.workload, grid, n_total, k, n_gpus)
        cfg["nccl_merge"] = comm is not None
        if comm is not None:   # the a8 communicator: one rank per GPU, made by distir_nccl_comm_init
            cfg["nccl_comm"] = {"n_ranks": world, "init": "ncclCommInitRank via distir_nccl_comm_init"}
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n_gpus,
            "steps": K, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": cfg,
            "configs_per_s": n_total / (ms_step / 1e3),
            "time_to_best_ms": e2e_ms,
            "roofline": roofline(prof, stats, n_sm, sm_mhz, peaks, peak_kind),
            "kernel_ms_per_step": {x: prof[x] / max(prof["launches"], 1) for x in
                                   ("ms_prepare", "ms_simulate", "ms_topk", "ms_merge")},
            "cpu_baseline": cpu,
            "e2e": {"value": ops_all / (e2e_ms / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d_all), "d2h_bytes_per_step": int(d2h_all)},
            "strong": strong,
            "gpu_launches": int(round(kernels_per_launch * K)),
            "clocks": clocks,
            "stats": {"op_events": int(ops_all), "stage_steps": int(steps_all),
                      "n_valid": stats["n_valid"], "n_feasible": stats["n_feasible"],
                      "n_buckets": stats["n_buckets"], "n_items": stats["n_items"],
                      "tasks": stats["tasks"], "slow_tasks": stats["slow_tasks"],
                      "wave_steps": stats["wave_steps"],
                      "note": "op_events: logical program ops; tasks / slow_tasks / "
                              "wave_steps: work k_simulate performed (a fast-path task "
                              "is one add + one binade test)"},
            "top1": {"index": int(res["topk"]["index"][0]),
                     "throughput": float(res["topk"]["throughput"][0])} if len(res["topk"]) else None,
        }
        print(json.dumps(out))
    if comm is not None:
        distir_nccl_comm_destroy(comm)
    sim.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
