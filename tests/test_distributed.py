"""Multi-rank sweep sharding on CPU: world_size 2 over gloo.

Each rank simulates its LPT shard (compute by the C oracle here: no GPU in
this container) and the metric rows are all-gathered; the merged rows must
equal a single-process run of the whole sweep.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2508_03148_b200.distributed import gather_rows, lpt_shards, merge_shards


def test_lpt_balances():
    costs = [100, 1, 1, 1, 50, 50, 2, 3]
    sh = lpt_shards(costs, 2)
    loads = [sum(costs[i] for i in s) for s in sh]
    assert sorted(i for s in sh for i in s) == list(range(len(costs)))
    assert max(loads) == 104 or max(loads) <= 106


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist

    from oracle import oracle
    from paper_2508_03148_b200 import workloads as W
    from paper_2508_03148_b200.api import instance_spec
    from paper_2508_03148_b200.config import parse_config
    from paper_2508_03148_b200.lower import lower

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    docs = W.c5_sweep(n_seeds=1, n_requests=16, configs=list(range(0, 64, 4)))
    specs = [instance_spec(parse_config(d)) for d in docs]
    full = lower(specs)
    shards = lpt_shards(full.descs["est_cost"], world)
    mine = lower([specs[i] for i in shards[rank]])
    rows = oracle.run(mine).rows
    gathered = gather_rows(rows, world)
    merged = merge_shards(shards, gathered, len(specs))
    if rank == 0:
        ref = oracle.run(full).rows
        out.put((merged["iterations"].tolist(), ref["iterations"].tolist(),
                 merged["ttft"].tolist(), ref["ttft"].tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gather_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    mi, ri, mt, rt = res
    assert mi == ri and mt == rt
