"""Synthetic workload generation (reference workload.py:131-216) off the host.

CPU: the C oracle's restatement of numpy's streams (Philox(key=SeedSequence(
[seed, stream])), ziggurat exponential / normal, exp, Lemire bounded integers
with numpy's 32-bit buffering) against the requests the reference generated
for the golden scenarios, and against the host generator on random specs.
GPU: fs_generate_workload against both, and simulate(device_workload=True)
against the host-generated run.
"""

import copy

import numpy as np
import pytest

from paper_2508_03148_b200.config import parse_config
from paper_2508_03148_b200.workload import (ArrivalSpec, LengthDist, WorkloadSpec,
                                            generate_arrays, workload_descs)


def _random_specs(n, seed=3):
    rs = np.random.default_rng(seed)
    specs = []
    for i in range(n):
        kind = ["poisson", "fixed_interval", "batch_at_zero"][i % 3]
        arr = ArrivalSpec(kind, rate_rps=float(rs.choice([0.5, 5, 20, 50, 1000])),
                          gap_ns=int(rs.integers(0, 10**7)))

        def ld(j):
            k = ["fixed", "uniform", "lognormal"][(i // 3 + j) % 3]
            lo = int(rs.integers(1, 50))
            hi = lo + int(rs.choice([0, 1, 7, 4000, 2**31 - 100]))
            return LengthDist(k, value=int(rs.integers(1, 900)), lo=lo, hi=min(hi, 2**31 - 1),
                              mu=float(rs.uniform(2, 7)), sigma=float(rs.uniform(0.2, 1.6)))
        specs.append(WorkloadSpec(arr, ld(0), ld(1), int(rs.integers(1, 400)),
                                  seed=int(rs.integers(0, 2**63))))
    return specs


def _ranks(n):
    ids = [f"r{j}" for j in range(n)]
    return np.argsort(np.argsort(ids, kind="stable"), kind="stable")


def _check(specs, descs, got):
    arr, pr, out, rk, st = got
    assert (st == 0).all()
    for i, s in enumerate(specs):
        h = generate_arrays(s)
        o, n = int(descs[i]["out_offset"]), s.num_requests
        assert h.ids == [f"r{k}" for k in range(n)]  # generation order is arrival order
        assert np.array_equal(h.arrival_ns, arr[o:o + n]), i
        assert np.array_equal(h.prompt, pr[o:o + n]), i
        assert np.array_equal(h.output, out[o:o + n]), i
        assert np.array_equal(_ranks(n), rk[o:o + n]), i


def _golden_workloads(golden_scenarios):
    specs, want = [], []
    for name, g in golden_scenarios.items():
        cfg = parse_config(copy.deepcopy(g["config"]))
        if cfg.trace_path is not None:
            continue
        specs.append(cfg.workload)
        want.append(g["requests"])
    return specs, want


def test_oracle_matches_reference_requests(golden_scenarios):
    from oracle import oracle
    specs, want = _golden_workloads(golden_scenarios)
    d = workload_descs(specs)
    arr, pr, out, rk, st = oracle.generate_workload(d)
    assert (st == 0).all()
    for i, w in enumerate(want):
        o, n = int(d[i]["out_offset"]), specs[i].num_requests
        assert w["ids"] == [f"r{k}" for k in range(n)]
        assert arr[o:o + n].tolist() == w["arrival_ns"]
        assert pr[o:o + n].tolist() == w["prompt"]
        assert out[o:o + n].tolist() == w["output"]


def test_oracle_matches_host_generator_random_specs():
    from oracle import oracle
    specs = _random_specs(200)
    d = workload_descs(specs)
    _check(specs, d, oracle.generate_workload(d))


@pytest.mark.gpu
def test_device_matches_reference_requests(engine, golden_scenarios):
    specs, want = _golden_workloads(golden_scenarios)
    d = workload_descs(specs)
    arr, pr, out, rk, st = engine.generate_workload(d)
    assert (st == 0).all()
    for i, w in enumerate(want):
        o, n = int(d[i]["out_offset"]), specs[i].num_requests
        assert arr[o:o + n].tolist() == w["arrival_ns"]
        assert pr[o:o + n].tolist() == w["prompt"]
        assert out[o:o + n].tolist() == w["output"]


@pytest.mark.gpu
def test_device_matches_host_generator_random_specs(engine):
    specs = _random_specs(600, seed=11)
    d = workload_descs(specs)
    _check(specs, d, engine.generate_workload(d))


@pytest.mark.gpu
def test_simulate_with_device_workload_equals_host(engine):
    from paper_2508_03148_b200 import workloads as W
    from paper_2508_03148_b200.api import simulate
    docs = W.c5_sweep(n_seeds=2)
    docs.append({"bad": "document"})  # a config-time failure keeps its slot
    a = simulate(copy.deepcopy(docs), engine=engine)
    b = simulate(copy.deepcopy(docs), engine=engine, device_workload=True)
    assert len(a) == len(b)
    for x, y in zip(a, b):
        assert type(x) is type(y)
        if hasattr(x, "to_dict"):
            assert x.to_dict() == y.to_dict()
