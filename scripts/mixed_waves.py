"""Heterogeneous-batch check (per-variant waves): the C5 sweep alone, one
dirichlet_skew DeepSeek-V3 instance and one DeepSeek-V3 EP instance alone, and all
of them in one batch. Prints one JSON line (device ms, CUDA events, 3 launches each)."""
import copy
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import workload_docs  # noqa: E402
from paper_2508_03148_b200 import workloads as W  # noqa: E402
from paper_2508_03148_b200.api import instance_spec  # noqa: E402
from paper_2508_03148_b200.config import parse_many  # noqa: E402
from paper_2508_03148_b200.engine import Engine  # noqa: E402
from paper_2508_03148_b200.lower import lower  # noqa: E402


def timed(eng, docs):
    low = lower([instance_spec(c) for c in parse_many(copy.deepcopy(docs))])
    eng.stage(low)
    eng.launch()
    torch.cuda.synchronize()
    ms = []
    st = torch.cuda.Stream()
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        eng.launch(st.cuda_stream)
        b.record(st)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    res = eng.fetch(low, per_request=False)
    assert (res.rows["status"] == 0).all()
    return min(ms), int(res.rows["iterations"].sum())


def main():
    eng = Engine(0)
    c5 = workload_docs(0, 64, 64)
    dsv3_dir = W.c4_colocated_ep(16, seed=5)
    dsv3_dir["routing"] = {"policy": "dirichlet_skew", "alpha": 0.3}
    extra = [dsv3_dir, W.c4_colocated_ep(16, seed=3)]
    t_c5, it5 = timed(eng, c5)
    t_x = [timed(eng, [d])[0] for d in extra]
    t_all, it_all = timed(eng, c5 + extra)
    print(json.dumps({"c5_ms": t_c5, "extra_alone_ms": t_x, "mixed_ms": t_all,
                      "sum_separate_ms": t_c5 + sum(t_x), "ratio": t_all / (t_c5 + sum(t_x)),
                      "iterations": it_all}))


if __name__ == "__main__":
    main()
