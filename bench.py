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
  cpu_baseline the CPU oracle on a bounded sample of the same grid (rank 0, N=1)

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
ISSUE_PEAK_NOTE = "148 SMs x 4 SMSPs x 32 lanes x 1 instr/clk x sm_max_mhz"


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

def cpu_oracle_rate(grid, seconds, seed=20211105426, threads=None):
    """Time the oracle (as it stands) on seeded random configs of the grid
    until `seconds` of wall time, on all host threads (each thread owns
    whole configurations); op-events/s."""
    import oracle
    oracle.build()
    threads = threads or os.cpu_count() or 1
    n = len(oracle.enumerate_grid(grid)) if grid["synth_count"] == 0 else grid["synth_count"]
    rng = np.random.default_rng(seed)
    order = rng.permutation(n)
    done, ops, cfgs, t0 = 0, 0, 0, time.perf_counter()
    chunk = max(16, 8 * threads)
    while time.perf_counter() - t0 < seconds and done < n:
        idx = np.sort(order[done:done + chunk])
        r = oracle.grid_eval(grid, indices=idx, threads=threads)
        valid = (r["reason"] & 0x1F) == 0
        ops += int(r["n_ops"][valid].sum())
        cfgs += len(idx)
        done += chunk
    dt = time.perf_counter() - t0
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


# --------------------------------------------------------------- main -------

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
    if world > 1:
        obj = [distir_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = distir_nccl_comm_init(obj[0], world, rank, local)
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

    # warm-up
    for _ in range(args.warmup):
        sim.launch(outs, k=k, comm=comm)
    barrier()
    stats = sim.last_stats()

    # ---- device-timed region (inputs resident in HBM)
    K = args.steps
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(K)]
    sim.profile(True)
    with ClockSampler(local) as clk:
        barrier()
        for i in range(K):
            flush.zero_()
            evs[i][0].record(stream)
            sim.launch(outs, k=k, comm=comm)
            evs[i][1].record(stream)
        barrier()
    prof = sim.profile(False)
    clocks = clk.summary()
    t_ms = sum(a.elapsed_time(b) for a, b in evs)
    ms_step = t_ms / K
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

    # ---- reduce over ranks
    vals = torch.tensor([ms_step, e2e_ms, float(stats["op_events"]),
                         float(stats["stage_steps"]), float(est["h2d_bytes"]),
                         float(est["d2h_bytes"])], dtype=torch.float64, device=dev)
    if world > 1:
        mx = vals[:2].clone()
        sm = vals[2:].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        vals = torch.cat([mx, sm])
    ms_step, e2e_ms, ops_all, steps_all, h2d_all, d2h_all = vals.tolist()
    assert res["topk"]["index"].tolist() == \
        tk_dev.numpy()[:ntk].view(np.int64).reshape(-1, 4)[:, 0].tolist()

    if rank == 0:
        peaks, peak_kind = measured_peaks()
        sm_max = float(peaks.get("sm_max_mhz", 1965.0))
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
        issue_peak = n_sm * 4 * 32 * sm_max * 1e6
        sim_ms = prof["ms_simulate"] / max(prof["launches"], 1)
        achieved = stats["stage_steps"] / (sim_ms / 1e3)
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_simulate_summary.json")
        if os.path.exists(tp):
            with open(tp) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            c = cpu_oracle_rate(grid, args.cpu_seconds)
            cpu = {"value": c["value"], "unit": UNIT, "cores": c["threads"],
                   "kind": "oracle",
                   "sample": "seeded random %d of %d %s configs (%d op-events), %.1f s, "
                             "%d threads" % (c["configs"], n_total, args.workload, c["ops"],
                                             c["seconds"], c["threads"])}
        value = ops_all / (ms_step / 1e3)
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n_gpus,
            "steps": K, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": bench_config(args.workload, grid, n_total, k, n_gpus),
            "configs_per_s": n_total / (ms_step / 1e3),
            "time_to_best_ms": e2e_ms,
            "roofline": {"bound": "alu", "achieved": achieved, "peak": issue_peak,
                         "unit": "stage-steps/s", "frac": achieved / issue_peak,
                         "traffic": traffic,
                         "kernel": "k_simulate", "kernel_ms": sim_ms,
                         "peak_note": ISSUE_PEAK_NOTE + " (%s sm_max_mhz)" % peak_kind},
            "kernel_ms_per_step": {x: prof[x] / max(prof["launches"], 1) for x in
                                   ("ms_prepare", "ms_simulate", "ms_topk", "ms_merge")},
            "cpu_baseline": cpu,
            "e2e": {"value": ops_all / (e2e_ms / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d_all), "d2h_bytes_per_step": int(d2h_all)},
            "gpu_launches": int(prof["kernels"]),
            "clocks": clocks,
            "stats": {"op_events": int(ops_all), "stage_steps": int(steps_all),
                      "n_valid": stats["n_valid"], "n_feasible": stats["n_feasible"],
                      "n_buckets": stats["n_buckets"], "n_items": stats["n_items"]},
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
