"""Calibration of the regression cost model.

The paper: "empirical cost functions (e.g., for MatMul and AllReduce) ...
are linear regression models in terms of the sizes of the input tensors.
We calibrate the simulator by fitting these regression models on
microbenchmarks where we run a single op on inputs of various sizes. Some of
the regression coefficients correspond to hardware parameters such as GPU
DRAM bandwidth, kernel launch overhead, and network bandwidths".

Here the model of a compute op is t = c0 + c_flop * flops + c_byte * bytes
(include/distir.h, DESIGN reading R7), with one coefficient set for
MatMul-type ops and one for the other (elementwise / normalisation) ops.
`fit_cost` is the least-squares fit (non-negative, relative error);
`measure_b200` times single ops on the local GPU (cuBLAS bf16 GEMMs and
PyTorch elementwise kernels, CUDA events) -- this is calibration of the
simulator's hardware description, not part of the simulated hot path.
Communication keeps the alpha-beta forms; their coefficients need >= 2 GPUs
and stay the topology's link constants on a 1-GPU box.

    python -m paper_2111_05426_b200.calibrate --out workloads/calib_b200.json
"""
from __future__ import annotations

import argparse
import json
import time

import numpy as np


def fit_cost(flops, nbytes, seconds, relative=True):
    """Non-negative least squares for t = c0 + c_flop*flops + c_byte*bytes.

    relative=True minimises the relative residual (rows scaled by 1/t), so
    microsecond and second-scale samples weigh alike.  Returns (c0, c_flop,
    c_byte)."""
    from scipy.optimize import nnls
    f = np.asarray(flops, dtype=np.float64)
    b = np.asarray(nbytes, dtype=np.float64)
    t = np.asarray(seconds, dtype=np.float64)
    if not (len(f) == len(b) == len(t)) or len(t) < 3:
        raise ValueError("need >= 3 aligned samples")
    # scale the columns so the solver sees O(1) numbers
    sf = max(f.max(), 1.0)
    sb = max(b.max(), 1.0)
    A = np.stack([np.ones_like(f), f / sf, b / sb], axis=1)
    y = t.copy()
    if relative:
        A = A / t[:, None]
        y = np.ones_like(t)
    x, _ = nnls(A, y)
    return float(x[0]), float(x[1] / sf), float(x[2] / sb)


def predict(coef, flops, nbytes):
    c0, cf, cb = coef
    return (c0 + cf * np.asarray(flops, dtype=np.float64)) + cb * np.asarray(nbytes, dtype=np.float64)


# ----------------------------------------------------------- measurement ----

def _time_op(fn, reps=7, inner=16, warmup=3):
    """Seconds per op with `inner` launches back to back between two CUDA
    events (an op inside a program follows other ops; its launch overhead
    is the steady-state per-launch cost, not one launch's round trip)."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(inner):
            fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3 / inner)
    return float(np.median(ts))


def measure_b200(device=0, quick=False):
    """Single-op microbenchmarks on the local GPU (bf16, 2-byte values as
    in the simulated programs).  Returns {"mm": [(flops, bytes, s)],
    "ew": [...]} with the model's feature definitions: MatMul (m,k)x(k,n):
    flops 2mkn, bytes 2(mk + kn + mn); elementwise over N values: flops and
    bytes as the simulated op counts them (Relu N / 2N*2, Add N / 3N*2, GeLU
    8N / 2N*2, LayerNorm 5N / (2N + 2d)*2, Softmax 5N / 2N*2)."""
    import torch
    torch.cuda.set_device(device)
    dt = torch.bfloat16
    e = 2
    mm, ew = [], []
    dims = [256, 512, 1024, 2048, 4096, 8192] if not quick else [256, 1024, 4096]
    for m_ in dims:
        for k_ in dims:
            for n_ in ([k_] if quick else [k_, 4 * k_ if 4 * k_ <= 16384 else k_]):
                A = torch.randn(m_, k_, device="cuda", dtype=dt)
                B = torch.randn(k_, n_, device="cuda", dtype=dt)
                t = _time_op(lambda: A @ B)
                mm.append((2 * m_ * k_ * n_, e * (m_ * k_ + k_ * n_ + m_ * n_), t))
                del A, B
    sizes = [1 << s for s in (range(14, 29, 2) if not quick else range(14, 27, 4))]
    for N in sizes:
        x = torch.randn(N, device="cuda", dtype=dt)
        y = torch.randn(N, device="cuda", dtype=dt)
        ew.append((N, 2 * N * e, _time_op(lambda: torch.relu(x))))
        ew.append((N, 3 * N * e, _time_op(lambda: x + y)))
        ew.append((8 * N, 2 * N * e, _time_op(lambda: torch.nn.functional.gelu(x))))
        d = 1024
        if N >= d:
            x2 = x.view(-1, d)
            w = torch.ones(d, device="cuda", dtype=dt)
            bb = torch.zeros(d, device="cuda", dtype=dt)
            ew.append((5 * N, (2 * N + 2 * d) * e,
                       _time_op(lambda: torch.nn.functional.layer_norm(x2, (d,), w, bb))))
            ew.append((5 * N, 2 * N * e, _time_op(lambda: torch.softmax(x2, dim=-1))))
        del x, y
    return {"mm": mm, "ew": ew}


def calibrate(samples):
    mm = np.array(samples["mm"], dtype=np.float64)
    ew = np.array(samples["ew"], dtype=np.float64)
    cm = fit_cost(mm[:, 0], mm[:, 1], mm[:, 2])
    ce = fit_cost(ew[:, 0], ew[:, 1], ew[:, 2])

    def err(c, s):
        p = predict(c, s[:, 0], s[:, 1])
        r = np.abs(p - s[:, 2]) / s[:, 2]
        return float(np.median(r)), float(r.max())
    return {
        "cost_model": 1,
        "mm_c0_s": cm[0], "mm_s_per_flop": cm[1], "mm_s_per_byte": cm[2],
        "ew_c0_s": ce[0], "ew_s_per_flop": ce[1], "ew_s_per_byte": ce[2],
        "fit": {"mm_rel_err_median_max": err(cm, mm), "ew_rel_err_median_max": err(ce, ew),
                "mm_samples": len(mm), "ew_samples": len(ew)},
    }


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args(argv)
    import torch
    samples = measure_b200(quick=a.quick)
    res = calibrate(samples)
    res["device"] = torch.cuda.get_device_name(0)
    res["when"] = time.strftime("%Y-%m-%d %H:%M:%S")
    res["samples"] = samples
    txt = json.dumps(res, indent=1)
    if a.out:
        with open(a.out, "w") as f:
            f.write(txt + "\n")
    print(json.dumps({k: v for k, v in res.items() if k != "samples"}, indent=1))


if __name__ == "__main__":
    main()
