"""cProfile of simulate() on the C5 documents (GPU): where the host time goes.

    python scripts/profile_api.py [seeds] > gpurun_out/profile_api.txt
"""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import workload_docs  # noqa: E402
from paper_2508_03148_b200.api import simulate  # noqa: E402
from paper_2508_03148_b200.engine import Engine  # noqa: E402


def main():
    seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    eng = Engine(0)
    docs = workload_docs(0, seeds, 64)
    simulate(docs, engine=eng, device_workload=True, expert_imbalance=False)  # warm
    t = time.perf_counter()
    simulate(docs, engine=eng, device_workload=True, expert_imbalance=False)
    print("simulate wall s", time.perf_counter() - t)
    pr = cProfile.Profile()
    pr.enable()
    simulate(docs, engine=eng, device_workload=True, expert_imbalance=False)
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("cumulative").print_stats(45)
    st.sort_stats("tottime").print_stats(30)


if __name__ == "__main__":
    main()
