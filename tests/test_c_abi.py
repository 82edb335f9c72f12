"""The C ABI from a plain C caller (tests/c_abi/abi_client.c): no Python, no
torch between the caller and libfrontier_b200.so.

CPU: the client compiles and links against include/frontier_b200.h and the
library. GPU: it runs a lowered batch through fs_run_batch, generates a
workload and routes tokens; its outputs must equal the Python binding's and
the oracle's.
"""

import os
import subprocess

import numpy as np
import pytest

from paper_2508_03148_b200 import abi, native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "c_abi", "abi_client.c")
BIN = os.path.join(ROOT, "tests", "c_abi", "abi_client")


def build_client() -> str:
    lib_dir = os.path.dirname(native.LIB)
    subprocess.run(["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    SRC, "-L", lib_dir, "-lfrontier_b200", f"-Wl,-rpath,{lib_dir}", "-o", BIN],
                   check=True)
    return BIN


def test_client_builds_against_header_and_library():
    if not os.path.exists(native.LIB):
        pytest.skip("engine library not built")
    assert os.path.exists(build_client())


def _write_batch(low, path):
    with open(path, "wb") as fh:
        np.array([low.n_instances, len(low.replicas), len(low.prefixes), len(low.trace_counts),
                  low.n_requests], dtype=np.int64).tofile(fh)
        for a in (low.descs, low.replicas, low.prefixes):
            np.ascontiguousarray(a).tofile(fh)
        np.ascontiguousarray(low.trace_counts, dtype=np.int64).tofile(fh)
        np.ascontiguousarray(low.arrival, dtype=np.int64).tofile(fh)
        for a in (low.prompt, low.output, low.id_rank):
            np.ascontiguousarray(a, dtype=np.int32).tofile(fh)


@pytest.mark.gpu
def test_c_client_matches_python_binding(engine, tmp_path):
    from oracle import oracle
    from paper_2508_03148_b200 import workloads as W
    from paper_2508_03148_b200.workload import (ArrivalSpec, LengthDist, WorkloadSpec,
                                                generate_arrays)
    from parity import specs_for
    from paper_2508_03148_b200.lower import lower

    docs = W.c5_sweep(n_seeds=1)[::4] + [W.c4_af(6, seed=2), W.c3_pd(20, seed=3, tight=True)]
    low = lower(specs_for(docs))
    _write_batch(low, tmp_path / "batch.bin")
    exe = build_client()
    out = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().splitlines()

    ref = engine.run(low)
    rows = np.fromfile(tmp_path / "rows.bin", dtype=abi.METRIC_ROW)
    req = np.fromfile(tmp_path / "req.bin", dtype=np.int64).reshape(2, -1)
    assert rows.tobytes() == ref.rows.tobytes()
    assert np.array_equal(req[0], ref.first_ns) and np.array_equal(req[1], ref.done_ns)
    assert lines[0].startswith("run_batch")
    assert f"launches={engine.last_launch_count}" in lines[0]  # same kernels as the binding

    spec = WorkloadSpec(ArrivalSpec("poisson", rate_rps=20.0),
                        LengthDist("lognormal", lo=8, hi=4096, mu=6.0, sigma=1.0),
                        LengthDist("lognormal", lo=1, hi=1024, mu=5.0, sigma=0.8), 8, seed=1)
    h = generate_arrays(spec)
    want = " ".join(f"{a}:{p}:{o}" for a, p, o in zip(h.arrival_ns, h.prompt, h.output))
    assert lines[1] == f"workload status=0 {want}"

    for line, (T, seed) in zip(lines[2:5], [(17, 3), (1, 4), (300, 3735928559)]):
        c, st = oracle.route(T, 8, 2, "uniform", seed)
        assert line == f"route status={st} counts " + " ".join(map(str, c))
