import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, numpy as np, torch
from paper_2508_03148_b200.engine import Engine
eng = Engine(0)
for T in (1, 64, 1024, 8192):
    n = 148
    tok = np.full(n, T, np.int64); seeds = np.arange(n, dtype=np.uint64) + 7
    eng.route_tokens(tok, seeds, 256, 8, "dirichlet_skew", 0.3)
    torch.cuda.synchronize(); t = time.perf_counter()
    c, st = eng.route_tokens(tok, seeds, 256, 8, "dirichlet_skew", 0.3)
    dt = time.perf_counter() - t
    print(f"T={T}: {n} calls in {dt*1e3:.1f} ms -> {dt/n*1e6*148:.0f} us per call-slot; draws/s {n*T*256/dt:.3e}")
