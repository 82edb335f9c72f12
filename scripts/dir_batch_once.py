"""One C4 dirichlet_skew batch (DeepSeek-V3 EP=8, alpha 0.3) on the device, for
ncu captures: python scripts/dir_batch_once.py [instances] [requests]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import _dirichlet, lower_docs  # noqa: E402
from paper_2508_03148_b200 import workloads as W  # noqa: E402
from paper_2508_03148_b200.engine import Engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
req = int(sys.argv[2]) if len(sys.argv) > 2 else 16
low = lower_docs([_dirichlet(W.c4_colocated_ep(req, seed=1 + i)) for i in range(n)])
eng = Engine(0)
t = time.perf_counter()
res = eng.run(low)
print(n, "instances", int(res.rows["iterations"].sum()), "iterations",
      f"{time.perf_counter() - t:.2f} s", "ok", bool((res.rows["status"] == 0).all()))
