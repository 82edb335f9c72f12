"""Past the round-1 engine limits, against the reference.

tests/golden/capacity.json.gz (make_golden.py --only capacity, recorded from
/root/reference) holds instances with more than 64 replicas (PD 40 x 60, a
co-located MoE deployment with 80 replicas) and cluster ids long enough that the
router-seed prefix "{seed}:{id}/{i}:mb" exceeds the 192 bytes an fs_seed_prefix
holds inline (such prefixes travel as their tail plus a host-computed SHA-256
midstate, include/frontier_b200.h). The oracle (CPU) and the device (GPU) must
reproduce every recorded output bit for bit.
"""

import hashlib

import pytest

from conftest import load_golden
from parity import compare_to_golden, run_backend


@pytest.fixture(scope="module")
def golden_capacity():
    return load_golden("capacity")["data"]


def _check(backend, golden_capacity):
    names = list(golden_capacity)
    res = run_backend(backend, [golden_capacity[n]["config"] for n in names],
                      routes=True, threads=4)
    bad = {n: compare_to_golden(r, golden_capacity[n]) for n, r in zip(names, res)}
    assert {n: b for n, b in bad.items() if b} == {}
    return res


def test_oracle_past_engine_limits(golden_capacity):
    res = _check("oracle", golden_capacity)
    assert max(len(r.replica_keys) for r in res) > 64


def test_long_prefix_router_seeds_oracle():
    """derive_router_seed (base.py:63-65) for prefixes of every length class:
    host midstate (lower.sha256_midstate) + oracle tail hash == hashlib."""
    from oracle import oracle
    for n in (10, 63, 64, 65, 127, 128, 191, 192, 193, 250, 600, 1000):
        pre = "7:" + "c" * n + "/3:"
        for mb, step, layer in ((0, 5, 2), (3, 12345, 60), (1, 0, 0)):
            msg = pre + (f"{mb}:" if mb > 0 else "") + f"{step}:{layer}"
            want = int.from_bytes(hashlib.sha256(msg.encode()).digest()[:4], "big")
            assert oracle.router_seed(pre, mb, step, layer) == want, (n, mb)


@pytest.mark.gpu
def test_device_past_engine_limits(engine, golden_capacity):
    _check(engine, golden_capacity)


@pytest.mark.gpu
def test_long_prefix_router_seeds_device(engine):
    prefixes, want, steps, layers, mbs = [], [], [], [], []
    for n in (10, 63, 64, 65, 191, 192, 193, 250, 600, 1000):
        for mb, step, layer in ((0, 5, 2), (3, 12345, 60)):
            pre = "7:" + "c" * n + "/3:"
            msg = pre + (f"{mb}:" if mb > 0 else "") + f"{step}:{layer}"
            prefixes.append(pre)
            mbs.append(mb)
            steps.append(step)
            layers.append(layer)
            want.append(int.from_bytes(hashlib.sha256(msg.encode()).digest()[:4], "big"))
    got = engine.router_seeds(prefixes, list(range(len(prefixes))), mbs, steps, layers)
    assert got.tolist() == want


# ---- top_k > 16 (tests/golden/largek.json.gz, make_golden.py --only largek) ----------------

@pytest.fixture(scope="module")
def golden_largek():
    return load_golden("largek")["data"]


def test_oracle_large_topk(golden_largek):
    from oracle import oracle
    for T, E, k, seed, policy, alpha, counts in golden_largek["route_calls"]:
        got, st = oracle.route(T, E, k, policy, seed, alpha)
        assert st == 0 and list(got) == counts, (T, E, k, seed, policy)
    sc = golden_largek["scenarios"]
    res = run_backend("oracle", [g["config"] for g in sc.values()], routes=True)
    bad = {n: compare_to_golden(r, g) for (n, g), r in zip(sc.items(), res)}
    assert {n: b for n, b in bad.items() if b} == {}


@pytest.mark.gpu
def test_device_large_topk(engine, golden_largek):
    import numpy as np
    for T, E, k, seed, policy, alpha, counts in golden_largek["route_calls"]:
        got, st = engine.route_tokens(np.array([T]), np.array([seed], dtype=np.uint64), E, k,
                                      policy, alpha)
        assert st[0] == 0 and got[0].tolist() == counts, (T, E, k, seed, policy)
    sc = golden_largek["scenarios"]
    res = run_backend(engine, [g["config"] for g in sc.values()], routes=True)
    bad = {n: compare_to_golden(r, g) for (n, g), r in zip(sc.items(), res)}
    assert {n: b for n, b in bad.items() if b} == {}
