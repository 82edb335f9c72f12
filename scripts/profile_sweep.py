"""Per-instance cycle distribution of the C5 sweep on the device (profiling aid)."""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import lower_docs, workload_docs  # noqa: E402
from paper_2508_03148_b200.engine import Engine  # noqa: E402


def main():
    seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    docs = workload_docs(0, seeds, 64)
    fams = os.environ.get("FS_FAMILIES")  # e.g. "AB": profile a subset of the C5 families
    if fams:
        fam_of = ["A"] * 16 + ["B"] * 32 + ["C"] * 16
        docs = [d for i, d in enumerate(docs) if fam_of[i // seeds] in fams]
    low = lower_docs(docs)
    eng = Engine(0)
    eng.stage(low)
    for _ in range(2):
        eng.launch()
    res = eng.fetch(low, per_request=False)
    lib = eng.lib
    lib.fs_instance_cycles.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    cyc = np.zeros(low.n_instances, dtype=np.int64)
    lib.fs_instance_cycles(eng.h, cyc.ctypes.data)
    t0 = time.perf_counter()
    eng.launch()
    eng.fetch(low, per_request=False)
    wall = time.perf_counter() - t0
    its = res.rows["iterations"]
    fam = np.repeat(np.array(["A"] * 16 + ["B"] * 32 + ["C"] * 16), seeds)
    if fams:
        fam = np.array([f for f in fam if f in fams])
    print(f"sweep wall {wall*1e3:.1f} ms, iterations {its.sum()}, it/s {its.sum()/wall:.3e}")
    clk = 1.965e9
    for f in "ABC":
        m = fam == f
        if not m.any():
            continue
        print(f"family {f}: n={m.sum()} iters={its[m].sum()} cycles mean={cyc[m].mean():.3e} "
              f"max={cyc[m].max():.3e} ({cyc[m].max()/clk*1e3:.1f} ms) "
              f"sum={cyc[m].sum():.3e} cyc/iter={cyc[m].sum()/its[m].sum():.0f}")
    order = np.argsort(-cyc)[:8]
    for i in order:
        print("  slowest", i, fam[i], int(cyc[i]), int(its[i]), int(low.descs[i]["max_num_seqs"]))


if __name__ == "__main__":
    main()
