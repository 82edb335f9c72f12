"""dirichlet_skew routing (reference costmodel/routing.py:99-106).

CPU: the C oracle's restatement of numpy's Generator.dirichlet / exponential
(ziggurat tables read from numpy's own libnpyrandom.a) against vectors the
reference produced (tests/golden/dirichlet.json.gz, numpy 2.3.5): raw stream
bits, route_tokens counts and whole simulations. GPU: the device router and the
simulation engine against the same fixtures and the oracle.
"""

import numpy as np
import pytest

from conftest import load_golden
from parity import compare_to_golden, run_backend


@pytest.fixture(scope="module")
def golden_dirichlet():
    return load_golden("dirichlet")["data"]


def test_oracle_dirichlet_stream_bits(golden_dirichlet):
    from oracle import oracle
    for E, alpha, seed, pop_bits, key_bits in golden_dirichlet["dirichlet_stream"]:
        pop, keys = oracle.dirichlet_row(E, alpha, seed)
        assert pop.view(np.uint64).tolist() == pop_bits, (E, alpha, seed)
        assert keys.view(np.uint64).tolist() == key_bits, (E, alpha, seed)


def test_oracle_route_dirichlet_counts(golden_dirichlet):
    from oracle import oracle
    for T, E, k, alpha, seed, counts in golden_dirichlet["route_dirichlet"]:
        c, st = oracle.route(T, E, k, "dirichlet_skew", seed, alpha)
        assert st == 0 and c == counts, (T, E, k, alpha, seed)


def test_oracle_dirichlet_live_numpy():
    """Beyond the fixture: the restatement against numpy itself, many seeds."""
    from oracle import oracle

    def rng(seed):  # routing.py:59-62
        return np.random.Generator(np.random.Philox(
            np.random.SeedSequence([seed, 0xE0]).generate_state(2, np.uint64)))

    for seed in range(25):
        for E, alpha in ((8, 0.3), (32, 0.07), (16, 1.7)):
            g = rng(seed)
            pop = np.maximum(g.dirichlet(np.full(E, alpha)), 1e-12)
            keys = g.exponential(1.0, (1, E))[0] / pop
            p2, k2 = oracle.dirichlet_row(E, alpha, seed)
            assert np.array_equal(p2.view(np.uint64), pop.view(np.uint64))
            assert np.array_equal(k2.view(np.uint64), keys.view(np.uint64))


def test_oracle_dirichlet_scenarios(golden_dirichlet):
    sc = golden_dirichlet["scenarios"]
    names = list(sc)
    res = run_backend("oracle", [sc[n]["config"] for n in names], routes=True)
    bad = {n: compare_to_golden(r, sc[n]) for n, r in zip(names, res)}
    assert {n: b for n, b in bad.items() if b} == {}


def test_oracle_dirichlet_bad_alpha():
    from oracle import oracle
    _, st = oracle.route(10, 8, 2, "dirichlet_skew", 1, 0.0)
    assert st == 5  # FS_ERR_ROUTING: "dirichlet_skew needs alpha > 0"
    c, st = oracle.route(0, 8, 2, "dirichlet_skew", 1, 0.0)  # T == 0 shortcut wins
    assert st == 0 and c == [0] * 8


@pytest.mark.gpu
def test_device_route_dirichlet_counts(engine, golden_dirichlet):
    groups = {}
    for T, E, k, alpha, seed, counts in golden_dirichlet["route_dirichlet"]:
        groups.setdefault((E, k, alpha), []).append((T, seed, counts))
    for (E, k, alpha), calls in groups.items():
        counts, st = engine.route_tokens([c[0] for c in calls], [c[1] for c in calls], E, k,
                                         "dirichlet_skew", alpha)
        assert (st == 0).all(), (E, k, alpha, st)
        assert counts.tolist() == [c[2] for c in calls], (E, k, alpha)


@pytest.mark.gpu
def test_device_route_dirichlet_vs_oracle(engine):
    """Many more calls than the fixture: device counts == oracle counts."""
    from oracle import oracle
    rs = np.random.default_rng(99)
    for E, k, alpha in ((8, 2, 0.3), (256, 8, 0.3), (64, 6, 0.05), (16, 3, 2.0)):
        T = rs.integers(1, 200, size=64)
        seeds = rs.integers(0, 2**32, size=64, dtype=np.uint64)
        counts, st = engine.route_tokens(T, seeds, E, k, "dirichlet_skew", alpha)
        for i in range(64):
            c, s = oracle.route(int(T[i]), E, k, "dirichlet_skew", int(seeds[i]), alpha)
            assert st[i] == s and counts[i].tolist() == c, (E, k, alpha, i)


@pytest.mark.gpu
def test_device_dirichlet_scenarios(engine, golden_dirichlet):
    sc = golden_dirichlet["scenarios"]
    names = list(sc)
    res = run_backend(engine, [sc[n]["config"] for n in names], routes=True)
    bad = {n: compare_to_golden(r, sc[n]) for n, r in zip(names, res)}
    assert {n: b for n, b in bad.items() if b} == {}
