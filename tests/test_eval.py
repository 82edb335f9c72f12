"""Pure functions on the device (fs_eval) against the reference's golden vectors
and the host C library.

* libm: numpy's distributions.c gets exp / log / log1p / pow from glibc; the
  device's restatement (csrc/fs_glibm.h) must equal the host's on every
  argument -- including the ones where CUDA's own libm differs (found here by
  evaluating both on the device), which are exactly the arguments that could
  flip a gamma / ziggurat accept-reject test.
* cost model: tests/golden/pure.json.gz holds reference outputs of
  analytic.linear_us / grouped_gemm_us, topology.collective_time /
  transfer_time and costmodel.moe.moe_layer_latency, recorded by
  tests/golden/make_golden.py from /root/reference. The device evaluates them
  through the same device functions sim_kernel composes.

The CPU half (not gpu) checks the header compiled for the host against the
system libm with tests/glibm/glibm_check.c.
"""

import gzip
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HW = (2.25e15, 8e12, 5.0)  # make_golden: HardwareSpec(peak, mem_bw), default overhead 5 us
LINK = (5e-6, 900e9)


def _pure():
    with gzip.open(os.path.join(ROOT, "tests", "golden", "pure.json.gz")) as fh:
        return json.load(fh)["data"]


def test_glibm_header_matches_host_libm(tmp_path):
    """fs_glibm.h compiled for the host == glibc's exp/log/log1p/pow, 4 x 3M arguments."""
    exe = tmp_path / "glibm_check"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", str(exe),
                    os.path.join(ROOT, "tests", "glibm", "glibm_check.c"), "-lm"], check=True)
    out = subprocess.run([str(exe), "3000000", "11"], capture_output=True, text=True)
    res = json.loads(out.stdout)
    assert out.returncode == 0 and res == {"n": 3000000, "exp": 0, "log": 0, "log1p": 0,
                                           "pow": 0}, out.stderr


def _libm_args(rng, n):
    u = rng.random(n)
    return {
        "exp": np.concatenate([-rng.random(n) * 40.0, (rng.random(n) - 0.5) * 1400.0,
                               -0.5 * np.square(rng.normal(size=n) * 3.0)]),
        "log": np.concatenate([u, 1.0 + (rng.random(n) - 0.5) * 0.25, rng.random(n) * 1e6,
                               rng.integers(1, 500, n) / rng.integers(500, 10_000, n)]),
        "log1p": np.concatenate([-u, (rng.random(n) - 0.5) * 1e-3, rng.random(n) * 10]),
        "pow": (np.concatenate([u, 0.5 + rng.random(n) * 4.0]),
                np.concatenate([1.0 / (0.01 + rng.random(n)), 1.0 / (0.05 + rng.random(n))])),
    }


@pytest.mark.gpu
def test_device_libm_equals_host_libm():
    from oracle import oracle
    from paper_2508_03148_b200.engine import Engine

    eng = Engine(0)
    rng = np.random.default_rng(20251017)
    args = _libm_args(rng, 400_000)
    report = {}
    for fn, a in args.items():
        x, y = (a if fn == "pow" else (a, a))
        rec = np.stack([x, y], axis=1)
        dev, st = eng.eval(fn, rec)
        cud, _ = eng.eval("cuda_" + fn, rec)
        host = oracle.libm(fn, x, y)
        assert (st == 0).all()
        same = dev[:, 0].view(np.int64) == host.view(np.int64)
        cuda_diff = cud[:, 0].view(np.int64) != host.view(np.int64)
        report[fn] = (int((~same).sum()), int(cuda_diff.sum()))
        assert same.all(), (fn, x[~same][:5], y[~same][:5])
    # the arguments where CUDA's libm would have decided differently exist in numbers
    assert sum(c for _, c in report.values()) > 100, report


@pytest.mark.gpu
def test_cost_functions_vs_reference_vectors():
    from paper_2508_03148_b200.engine import Engine

    eng = Engine(0)
    data = _pure()
    lin = np.array([[m, n, k, *HW, 2] for m, n, k, _ in data["linear"]], dtype=np.float64)
    out, st = eng.eval("linear", lin)
    assert (st == 0).all()
    assert out[:, 0].tolist() == [v[3] for v in data["linear"]]

    gg = []
    for counts, d, dff, nm, _ in data["grouped_gemm"]:
        gg.append([sum(counts), sum(1 for c in counts if c > 0), d, dff, nm, *HW, 2])
    out, st = eng.eval("grouped_gemm", gg)
    assert (st == 0).all()
    assert out[:, 0].tolist() == [v[4] for v in data["grouped_gemm"]]

    kinds = {"all_to_all": 0, "all_reduce": 1, "all_gather": 2}
    for is_int in (True, False):
        rows = [v for v in data["collective"] if isinstance(v[1], int) == is_int]
        rec = [[kinds[k], b, n, *LINK] for k, b, n, _ in rows]
        out, st = eng.eval("collective_int" if is_int else "collective_flt", rec)
        assert (st == 0).all()
        assert out[:, 0].tolist() == [v[3] for v in rows], is_int
    assert len(data["collective"]) == 108

    rec = [[b, 20e-6, 50e9] for b, _ in data["transfer"]]
    out, _ = eng.eval("transfer", rec)
    assert out[:, 0].tolist() == [v[1] for v in data["transfer"]]


@pytest.mark.gpu
def test_moe_layer_vs_reference_breakdowns():
    from paper_2508_03148_b200.engine import Engine

    eng = Engine(0)
    data = _pure()["moe_layer"]
    width = 14 + max(v[0] for v in data)
    recs = []
    for E, k, ep, mtp, gated, T, _seed, counts, _total, _br in data:
        d_ff = 14336 if E == 8 else 2048
        r = [E, k, ep, mtp, 3 if gated else 2, T, 4096, d_ff, 2, *LINK, *HW] + list(counts)
        recs.append(r + [0] * (width - len(r)))
    out, st = eng.eval("moe_layer", recs, out_stride=2)
    assert (st == 0).all()
    for (E, k, ep, mtp, gated, T, _s, counts, total, br), o in zip(data, out):
        assert o[0] == total, (E, k, ep, T)
        per = br["per_rank_us"]
        assert o[1] == br["expert_us"] / (sum(per) / ep), (E, k, ep, T)
