"""One C2 attention-cost launch (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import bench_attention_cost  # noqa: E402
from paper_2508_03148_b200.engine import Engine  # noqa: E402
print(bench_attention_cost(Engine(0), 0, 1, 1))
