"""Stage one BASELINE config as a batch of seeds and launch it once (ncu target).

usage: python scripts/config_once.py {c1|c3|c4af|c4ep} [instances]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import lower_docs  # noqa: E402
from paper_2508_03148_b200 import workloads as W  # noqa: E402
from paper_2508_03148_b200.engine import Engine  # noqa: E402

MAKE = {"c1": lambda s: W.c1_colocated(1000, seed=s), "c3": lambda s: W.c3_pd(300, seed=s),
        "c4af": lambda s: W.c4_af(64, seed=s), "c4ep": lambda s: W.c4_colocated_ep(64, seed=s)}
name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 148
low = lower_docs([MAKE[name](1 + i) for i in range(n)])
eng = Engine(0)
eng.stage(low)
eng.launch()  # warm-up (module load); ncu: capture with -c 1 sees this launch
rows = eng.fetch(low, per_request=False).rows
t0 = time.perf_counter()
eng.launch()
rows = eng.fetch(low, per_request=False).rows
print(f"{name} x{n}: {time.perf_counter() - t0:.3f}s, iterations {int(rows['iterations'].sum())}, "
      f"draws {int(rows['routing_draws'].sum())}, ok {bool((rows['status'] == 0).all())}")
