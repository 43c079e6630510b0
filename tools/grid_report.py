#!/usr/bin/env python
"""Measurement report over every workload of SURVEY §8d (D.1, D.4, D.5), on
one B200 and the box's host cores.  Not the driver's bench line (bench.py);
this is the per-grid table DESIGN.md §6 cites.

Per grid (W1..W5, the paper-shaped PM / PG grids, and the NEXT-row variants
on the W2 grid):
  * GPU, device-timed: median of R launches of the whole pass (a1-a7, one
    CUDA graph), inputs resident, L2 flushed between launches; configs/s,
    op-events/s (valid configs, C.3 / C.4 counts), kernel breakdown.
  * GPU, end to end: time-to-best-config through distir_grid_eval with host
    buffers (spec H2D, per-config results + top-k D2H).
  * Projected multi-GPU scaling (this build's boxes have one GPU): the grid
    sharded round-robin over G ranks exactly as distir_grid_eval_sharded does,
    every shard timed alone on this GPU; the G-GPU time is the slowest shard
    (the NCCL all-gather of G x k x 32 B is not included).  Strong scaling
    (the grid split over G) for W3 and W5.
  * CPU oracle (test infrastructure, timed as it stands): 1 thread and all
    host threads, on the full grid or a seeded sample (W5: 1%), op-events/s.
  * Linearity of the oracle's per-configuration time in the op count
    ("linear scaling as a function of the op count"): R^2 on a sample.
Writes JSON to argv[1] (default profiles/r02_grid_report.json) and prints a
markdown table.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402


def gpu_time(sim, grid, reps, rank=0, n_ranks=1, flush=None):
    import torch
    n = sim.upload(grid, rank=rank, n_ranks=n_ranks)
    outs = sim.device_outputs(n, k=10)
    for _ in range(3):
        sim.launch(outs, k=10)
    torch.cuda.synchronize()
    st = sim.stream
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        sim.launch(outs, k=10)
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    # kernel breakdown from the library's per-phase events, in a separate
    # pass (the events add graph nodes; the timed launches above run without)
    sim.profile(True)
    for _ in range(min(reps, 10)):
        if flush is not None:
            flush.zero_()
        sim.launch(outs, k=10)
    prof = sim.profile(False)
    stats = sim.last_stats()
    L = max(prof["launches"], 1)
    return float(np.median(ts)), stats, {k: prof[k] / L for k in
                                         ("ms_prepare", "ms_simulate", "ms_topk")}


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(
        ROOT, "profiles", "r02_grid_report.json")
    import torch
    import oracle
    from paper_2111_05426_b200 import Simulator
    oracle.build()
    sim = Simulator(W.MODELS, W.TOPOLOGIES, device=0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
    threads = os.cpu_count() or 1
    grids = [("W1", W.GRIDS["W1"]), ("W2", W.GRIDS["W2"]), ("W3", W.GRIDS["W3"]),
             ("W4", W.GRIDS["W4"]), ("W5", W.GRIDS["W5"]),
             ("PM_1B", W.GRIDS["PM_1B"]), ("PM_17B", W.GRIDS["PM_17B"]),
             ("PM_103B", W.GRIDS["PM_103B"]), ("PG", W.GRIDS["PG"]),
             ("W2-1F1B", W.grid_with("W2", models=["mlp_1b_1f1b"])),
             ("W4-1F1B", W.grid_with("W4", models=["mlp_w4_1f1b"])),
             ("W2-ckpt", W.grid_with("W2", models=["mlp_1b_ckpt"])),
             ("W2-ZeRO", W.grid_with("W2", models=["mlp_1b_zero"])),
             ("W4-ZeRO", W.grid_with("W4", models=["mlp_w4_zero"])),
             ("W2-TB200R", W.grid_with("W2", topos=["TB200R"])),
             ("W3xTM", W.grid_with("W3", topos=["TB200"] + W.TM[:7]))]
    rows = []
    for name, g in grids:
        n = sim.grid_size(g)
        reps = 5 if name == "W5" else 30
        ms, st, kb = gpu_time(sim, g, reps, flush=flush)
        # end to end (host buffers), time-to-best
        sim.eval(g, k=10)
        t0 = time.perf_counter()
        E = 3 if name == "W5" else 10
        for _ in range(E):
            res = sim.eval(g, k=10)
        e2e = (time.perf_counter() - t0) / E * 1e3
        row = dict(grid=name, configs=n, valid=st["n_valid"], feasible=st["n_feasible"],
                   op_events=st["op_events"], gpu_ms=ms,
                   configs_per_s=n / (ms / 1e3), op_events_per_s=st["op_events"] / (ms / 1e3),
                   time_to_best_ms=e2e, kernel_ms=kb,
                   top1=int(res["topk"]["index"][0]) if len(res["topk"]) else None)
        # projected scaling (round-robin shards timed alone)
        if name in ("W3", "W5", "W3xTM"):
            sc = {}
            for G in (2, 4, 8):
                t = [gpu_time(sim, g, 3 if name == "W5" else 10, rank=r, n_ranks=G, flush=flush)[0]
                     for r in range(G)]
                sc[str(G)] = dict(max_shard_ms=max(t), min_shard_ms=min(t),
                                  op_events_per_s=st["op_events"] / (max(t) / 1e3),
                                  speedup=ms / max(t))
            row["projected_strong_scaling"] = sc
        # CPU oracle: full grid or a seeded sample
        fields = oracle.enumerate_grid(g) if g["synth_count"] == 0 else None
        n_all = n
        budget = 8.0
        rng = np.random.default_rng(7)
        if name == "W5":
            idx = np.sort(rng.choice(n_all, size=n_all // 100, replace=False))
            label = "seeded 1% sample (10^4 configs)"
        else:
            idx = np.arange(n_all)
            label = "full grid"
        cpu = {}
        for th in (1, threads):
            t0 = time.perf_counter()
            done, ops = 0, 0
            order = idx if th > 1 else rng.permutation(idx)
            step = 1000 if name == "W5" else max(16, 8 * th) if th > 1 else 16
            while done < len(order) and time.perf_counter() - t0 < budget * (1 if th == 1 else 2):
                chunk = np.sort(order[done:done + step])
                r = oracle.grid_eval(g, indices=chunk, threads=th)
                ops += int(r["n_ops"][(r["reason"] & 0x1F) == 0].sum())
                done += len(chunk)
            dt = time.perf_counter() - t0
            cpu[str(th)] = dict(threads=th, configs=int(done), op_events=ops,
                                seconds=dt, op_events_per_s=ops / dt,
                                sample=label if done >= len(order) else
                                "first %d configs of the %s (time-bounded)" % (done, label))
        row["cpu_oracle"] = cpu
        rows.append(row)
        print(json.dumps(row), flush=True)
    # linearity (oracle): per-config time vs op count on W2 + W3 samples
    lin = []
    rng = np.random.default_rng(744)
    for gname in ("W2", "W3"):
        g = W.GRIDS[gname]
        f = oracle.enumerate_grid(g)
        for i in rng.choice(len(f), size=60, replace=False):
            t0 = time.perf_counter()
            r = oracle.grid_eval(g, indices=np.array([i]), threads=1)
            dt = time.perf_counter() - t0
            if (r["reason"][0] & 0x1F) == 0:
                lin.append((int(r["n_ops"][0]), dt))
    x = np.array([a for a, _ in lin], float)
    y = np.array([b for _, b in lin], float)
    A = np.vstack([x, np.ones_like(x)]).T
    coef, res, *_ = np.linalg.lstsq(A, y, rcond=None)
    r2 = 1 - ((y - A @ coef) ** 2).sum() / ((y - y.mean()) ** 2).sum()
    report = dict(device=torch.cuda.get_device_name(0), host_threads=threads,
                  cpu_model=open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": ")
                  if os.path.exists("/proc/cpuinfo") else None,
                  grids=rows, oracle_linearity=dict(samples=len(lin), s_per_op=coef[0],
                                                    intercept_s=coef[1], r2=r2))
    with open(out_path, "w") as fo:
        json.dump(report, fo, indent=1)
    print("| grid | configs (valid) | op-events | GPU ms | op-events/s | configs/s | "
          "time-to-best ms | oracle 1 thr op-ev/s | oracle %d thr op-ev/s |" % threads)
    print("|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        c1, cn = r["cpu_oracle"]["1"], r["cpu_oracle"][str(threads)]
        print("| %s | %d (%d) | %.3g | %.4f | %.3g | %.3g | %.3f | %.3g | %.3g |" % (
            r["grid"], r["configs"], r["valid"], r["op_events"], r["gpu_ms"],
            r["op_events_per_s"], r["configs_per_s"], r["time_to_best_ms"],
            c1["op_events_per_s"], cn["op_events_per_s"]))
    print("oracle linearity R^2 = %.4f over %d configs" % (r2, len(lin)))
    sim.close()


if __name__ == "__main__":
    main()
