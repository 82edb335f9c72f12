"""Time the C2 attention-cost kernel variants (FS_C2) on the bench workload
(2^20 x 72-request batches) and check each against the default's bits.

    python scripts/c2_time.py [mode ...]      (GPU)
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2508_03148_b200 import workloads as W  # noqa: E402
from paper_2508_03148_b200.engine import Engine, attn_params  # noqa: E402


def main(modes):
    eng = Engine(0)
    n = 1 << 20
    q, kv, off, dec = W.attention_batches(n)
    t = [torch.from_numpy(a).cuda() for a in (q, kv, off, dec)]
    prm = attn_params(32, 8, 128, 2, 2.25e15, 8e12, 5.0)
    st = torch.cuda.Stream()
    alg = 8 * int(off[-1]) + 8 * (n + 1) + n + 8 * n + 4 * n
    ref = None
    for mode in ["tpb"] + list(modes):
        os.environ["FS_C2"] = mode
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        sts = torch.empty(n, dtype=torch.int32, device="cuda")

        def launch():
            eng.attention_cost_dev(t[0].data_ptr(), t[1].data_ptr(), t[2].data_ptr(),
                                   t[3].data_ptr(), n, prm, out.data_ptr(), sts.data_ptr(),
                                   st.cuda_stream)
        for _ in range(3):
            launch()
        torch.cuda.synchronize()
        ms = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            launch()
            b.record(st)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        o = out.cpu().numpy()
        if ref is None:
            ref = o
        same = bool(np.array_equal(o.view(np.uint64), ref.view(np.uint64)))
        med = float(np.median(ms))
        print(json.dumps({"mode": mode, "us_median": med * 1e3, "us_min": min(ms) * 1e3,
                          "GBps": alg / (med / 1e3) / 1e9, "same_bits": same,
                          "status_ok": bool((sts == 0).all().item())}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
