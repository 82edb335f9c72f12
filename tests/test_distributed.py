"""Multi-rank sharding of the product path: world_size 2 over gloo.

`simulate(configs)` and `simulate_rows(configs)` detect the initialised process
group, LPT-shard the instances, simulate each shard on the rank's engine and
all-gather the results. On CPU the engine slot is filled by the oracle behind the
Engine interface (oracle.OracleEngine: test infrastructure); the GPU-marked test
runs the CUDA engine on both ranks (one B200, gloo). Merged results must equal a
single-process run byte for byte.
"""

import os
import pickle
import socket
import time

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2508_03148_b200.distributed import lpt_shards


def test_lpt_balances():
    costs = [100, 1, 1, 1, 50, 50, 2, 3]
    sh = lpt_shards(costs, 2)
    loads = [sum(costs[i] for i in s) for s in sh]
    assert sorted(i for s in sh for i in s) == list(range(len(costs)))
    assert max(loads) <= 106


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _docs():
    from paper_2508_03148_b200 import workloads as W
    docs = W.c5_sweep(n_seeds=1, n_requests=16, configs=list(range(0, 64, 4)))
    bad = dict(docs[0])
    bad["model"] = {"name": "broken"}  # a point that fails to parse -> Failure row
    return docs + [bad]


def _engine(kind):
    if kind == "oracle":
        from oracle.oracle import OracleEngine
        return OracleEngine(threads=2)
    from paper_2508_03148_b200.engine import Engine
    return Engine(0)


def _worker(rank, world, port, kind, out, trace_dir):
    import faulthandler

    import torch.distributed as dist
    from paper_2508_03148_b200.api import simulate, simulate_rows

    # a hung rank dumps its Python stack (read back by _two_ranks) instead of
    # leaving the test to time out silently
    tf = open(os.path.join(trace_dir, f"rank{rank}.txt"), "w")
    faulthandler.dump_traceback_later(240, exit=True, file=tf)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    eng = _engine(kind)
    docs = _docs()
    bundles = simulate(docs, engine=eng)
    sr = simulate_rows(docs, engine=eng)
    if rank == 0:
        out.put(pickle.dumps(([b.to_dict() if hasattr(b, "to_dict") else b.status for b in bundles],
                              sr.rows.tobytes(), sr.failed, sr.config_hash)))
    dist.barrier()
    dist.destroy_process_group()
    faulthandler.cancel_dump_traceback_later()


def _two_ranks(kind):
    import queue
    import tempfile

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    trace_dir = tempfile.mkdtemp(prefix="fs_dist_")
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q, trace_dir)) for r in range(2)]
    for p in procs:
        p.start()
    deadline = time.monotonic() + 300
    res = None
    while res is None and time.monotonic() < deadline:
        try:
            res = pickle.loads(q.get(timeout=2))
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs):
                break
    if res is None:
        for p in procs:
            p.join(timeout=30)
        stacks = "".join(open(os.path.join(trace_dir, f)).read()
                         for f in sorted(os.listdir(trace_dir)))
        raise AssertionError(f"a rank hung or died (exit codes {[p.exitcode for p in procs]}):"
                             f"\n{stacks}")
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def _single(kind):
    from paper_2508_03148_b200.api import simulate, simulate_rows
    eng = _engine(kind)
    docs = _docs()
    bundles = simulate(docs, engine=eng, distributed=False)
    sr = simulate_rows(docs, engine=eng, distributed=False)
    return ([b.to_dict() if hasattr(b, "to_dict") else b.status for b in bundles],
            sr.rows.tobytes(), sr.failed, sr.config_hash)


def _check(two, one):
    assert two[0] == one[0]          # full MetricsBundles (per-request dicts included)
    assert two[1] == one[1]          # metric rows, byte for byte
    assert two[2] == one[2] and len(two[2]) == 1
    assert two[3] == one[3]


def test_two_rank_simulate_equals_single_process():
    _check(_two_ranks("oracle"), _single("oracle"))


@pytest.mark.gpu
def test_two_rank_engine_equals_single_process():
    _check(_two_ranks("engine"), _single("engine"))
