"""Pure-Python brute-force checkers -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Independent formulations used to pin the C++ oracle (none of them calls it):

* `cosimulate`: the per-rank projection of a global program (P:467-471,
  "project the input program to every device d") executed by per-device
  queues with rendezvous semantics -- a multi-device op starts when it heads
  the queue of every member device, once all are free.
  There is no global program order in this model; SPEC S:540 states that
  co-simulating the per-rank programs equals the global simulation.
* `longest_path`: the makespan as the longest path of the DAG whose edges join
  consecutive ops of each device (SURVEY C.6 Theorem 1), by memoised recursion.
* `interval_peaks`: per-device peak live bytes by stabbing live intervals
  ("live from the time it is created until its last usage"): value v
  counts at op i on its device iff birth(v) <= i <= death(v).
* `enumerate_bruteforce`: the D/T/P/K/B grid by exhaustive search over all
  integer triples ("all possible power-of-two combinations"), then
  sorted into the canonical order.
* `gpipe_flowshop`: the textbook permutation-flow-shop makespan with identical
  jobs, sum_s t_s + (K - 1) * max_s t_s, for zero-cost communication
  (SURVEY C.10 P3, Appendix C).
"""
from __future__ import annotations

import functools
import itertools
import sys


def cosimulate(n_dev, ops):
    """ops: [(devs, cost, ...)] in global order.  Returns (start, end, makespan)."""
    queues = [[i for i, op in enumerate(ops) if d in op[0]]
              for d in range(n_dev)]
    head = [0] * n_dev
    free = [0.0] * n_dev
    start = [None] * len(ops)
    end = [None] * len(ops)
    progress = True
    while progress:
        progress = False
        for d in range(n_dev):
            if head[d] >= len(queues[d]):
                continue
            i = queues[d][head[d]]
            devs = ops[i][0]
            if all(head[x] < len(queues[x]) and queues[x][head[x]] == i
                   for x in devs):
                s = max(free[x] for x in devs)
                e = s + ops[i][1]
                for x in devs:
                    free[x] = e
                    head[x] += 1
                start[i], end[i] = s, e
                progress = True
    if any(h != len(q) for h, q in zip(head, queues)):
        raise AssertionError("deadlock in per-device co-simulation")
    return start, end, max(free) if free else 0.0


def longest_path(n_dev, ops):
    """Makespan = longest path through per-device predecessor edges."""
    prev = []
    last = {}
    for i, op in enumerate(ops):
        prev.append([last[d] for d in op[0] if d in last])
        for d in op[0]:
            last[d] = i
    sys.setrecursionlimit(max(10000, 4 * len(ops)))

    @functools.lru_cache(maxsize=None)
    def end(i):
        return max([end(p) for p in prev[i]], default=0.0) + ops[i][1]

    return max((end(i) for i in range(len(ops))), default=0.0)


def interval_peaks(n_dev, ops, values):
    """ops: [(devs, cost, ins, outs, ...)]; values: [(dev, bytes, param,
    returned)].  Returns per-device peak bytes."""
    INF = float("inf")
    birth = [-1 if v[2] else None for v in values]
    death = [None] * len(values)
    for i, op in enumerate(ops):
        for v in op[3]:
            birth[v] = i
        for v in op[2]:
            death[v] = i          # overwritten by later uses: the last use
    for v, val in enumerate(values):
        if val[3]:
            death[v] = INF        # returned: never freed
        elif death[v] is None:
            # never read: a parameter stays, a dead output dies at birth
            death[v] = INF if val[2] else birth[v]
    peak = [0] * n_dev
    for v, val in enumerate(values):
        if val[2]:
            peak[val[0]] += val[1]          # parameters live from t = 0
    by_dev = [[v for v, val in enumerate(values) if val[0] == d]
              for d in range(n_dev)]
    for i, op in enumerate(ops):
        for d in op[0]:
            live = sum(values[v][1] for v in by_dev[d]
                       if birth[v] <= i <= death[v])
            peak[d] = max(peak[d], live)
    return peak


def enumerate_bruteforce(grid):
    """All (model_slot, topo_slot, W, D, T, P, K, B) of a non-synthetic
    grid, by exhaustive search, in the canonical order of SURVEY C.1."""
    def is_pow2(x):
        return x > 0 and (x & (x - 1)) == 0

    def allowed(mask, x):
        return (mask >> (x.bit_length() - 1)) & 1

    out = []
    for mi, _ in enumerate(grid["models"]):
        for ti, _ in enumerate(grid["topos"]):
            for W in sorted(grid["world"]):
                trip = sorted((D, T, P)
                              for D in range(1, W + 1)
                              for T in range(1, W + 1)
                              for P in range(1, W + 1)
                              if D * T * P == W and is_pow2(D) and
                              is_pow2(T) and is_pow2(P) and
                              allowed(grid["dp_mask"], D) and
                              allowed(grid["tp_mask"], T) and
                              allowed(grid["pp_mask"], P))
                for (D, T, P) in trip:
                    ks = [1] if (grid["k_mode"] == 0 and P == 1) \
                        else sorted(grid["k_set"])
                    for K, B in itertools.product(ks, sorted(grid["batch"])):
                        out.append((mi, ti, W, D, T, P, K, B))
    return out


def gpipe_flowshop(stage_times, K):
    """Permutation flow shop, identical jobs, K jobs over the given
    machine times: sum_s t_s + (K - 1) * max_s t_s."""
    return sum(stage_times) + (K - 1) * max(stage_times)


def topk_sorted(index, throughput, peak, feasible, k):
    """Top-k by Python's sort on the key (throughput desc, peak asc, index
    asc) over feasible entries."""
    keys = sorted((-throughput[i], peak[i], index[i], i)
                  for i in range(len(index)) if feasible[i])
    return [t[3] for t in keys[:k]]
