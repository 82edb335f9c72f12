"""C2 attention-cost legs (analytic + learned forest) once; `steps` launches each.

usage: python scripts/c2_once.py [steps]   (steps=1 for an ncu capture)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import bench_attention_cost  # noqa: E402
from paper_2508_03148_b200.engine import Engine  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
print(json.dumps(bench_attention_cost(Engine(0), 0, steps, max(1, min(steps, 3)))))
