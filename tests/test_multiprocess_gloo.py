"""World-size-2 CPU test of the multi-GPU host logic with the gloo backend:
the product's shard planner (distir_shard_indices, round-robin over canonical
indices), the exchange of the per-rank top-k lists through torch.distributed
(the same all-gather the GPU path does with NCCL), the broadcast of a
128-byte communicator id, and the merge order.  The per-shard results come
from the CPU oracle (test-side stand-in for each rank's GPU)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, grid_name, k, out):
    import torch.distributed as dist
    import oracle
    import workloads as W
    import paper_2111_05426_b200 as pkg
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    grid = W.GRIDS[grid_name]
    fields = oracle.enumerate_grid(grid)
    n = len(fields)
    idx = pkg.distir_shard_indices(n, rank, world)
    r = oracle.grid_eval(grid, indices=idx)
    pos, tp = oracle.topk(idx, fields[idx, 7], r["makespan"], r["peak"], r["reason"], k)
    local = [(float(tp[i]), int(r["peak"][pos[i]]), int(idx[pos[i]])) for i in range(len(pos))]
    gathered = [None] * world
    dist.all_gather_object(gathered, local)
    merged = sorted((rec for lst in gathered for rec in lst),
                    key=lambda t: (-t[0], t[1], t[2]))[:k]
    # communicator-id broadcast, as bench.py does before ncclCommInitRank
    uid = [bytes(range(128)) if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    sizes = [None] * world
    dist.all_gather_object(sizes, len(idx))
    out[rank] = (merged, uid[0], sizes, idx.tolist())
    dist.destroy_process_group()


@pytest.mark.parametrize("grid_name", ["W1", "W4"])
def test_two_rank_shards_merge_to_global_topk(grid_name):
    import oracle
    import workloads as W
    k = 10
    port = _free_port()
    with mp.Manager() as man:
        out = man.dict()
        mp.spawn(_worker, args=(2, port, grid_name, k, out), nprocs=2, join=True)
        res = dict(out)
    ref = oracle.grid_result(W.GRIDS[grid_name], k=k)
    want = ref["topk_index"].tolist()
    n = len(ref["reason"])
    for rank in range(2):
        merged, uid, sizes, idx = res[rank]
        assert [t[2] for t in merged] == want
        assert uid == bytes(range(128))
        assert sum(sizes) == n
    assert sorted(res[0][3] + res[1][3]) == list(range(n))
