"""Pin the C oracle against golden vectors produced by the reference itself.

These are the parity anchors: the CUDA engine is then checked against the
oracle (and against these same fixtures) in test_gpu_parity.py.
"""

import copy
import math

import numpy as np
import pytest

from parity import compare_to_golden, run_backend
from paper_2508_03148_b200 import workloads as W


def test_scenarios_bit_exact(golden_scenarios):
    names = list(golden_scenarios)
    res = run_backend("oracle", [golden_scenarios[n]["config"] for n in names], routes=True)
    failures = {n: compare_to_golden(r, golden_scenarios[n]) for n, r in zip(names, res)}
    assert {n: b for n, b in failures.items() if b} == {}


@pytest.mark.parametrize("name", ["C1_colocated_llama7b_1000", "C3_pd_70b_tight_300",
                                  "C3_pd_70b_roomy_300", "C4_af_dsv3_10", "C4_colocated_ep8_10"])
def test_baseline_configs_bit_exact(golden_baseline, name):
    g = golden_baseline[name]
    r = run_backend("oracle", [g["config"]], routes=name.startswith("C4"))[0]
    assert compare_to_golden(r, g) == []


def test_c5_design_points_bit_exact(golden_c5):
    base = W.c5_sweep_configs(64)
    docs = []
    for ci in range(64):
        d = copy.deepcopy(base[ci])
        d["seed"] = 1000 + 64 * ci
        docs.append(d)
    res = run_backend("oracle", docs, threads=8)
    bad = {ci: compare_to_golden(r, golden_c5[str(ci)]) for ci, r in enumerate(res)}
    assert {k: v for k, v in bad.items() if v} == {}


def test_router_seed_vectors(golden_pure):
    from oracle import oracle
    for master, scope, step, layer, want in golden_pure["router_seed"]:
        pre = f"{master}:{scope}:"
        assert oracle.router_seed(pre, 0, step, layer) == want, (master, scope, step, layer)


def test_af_microbatch_seed_prefix(golden_pure):
    # "{seed}:{key}:mb{i}:{step}:{layer}" built from the mb prefix + tail ints
    from oracle import oracle
    for master, scope, step, layer, want in golden_pure["router_seed"]:
        if ":mb" in scope:
            key, mb = scope.rsplit(":mb", 1)
            assert oracle.router_seed(f"{master}:{key}:mb", int(mb), step, layer) == want


def test_philox_keys(golden_pure):
    from oracle import oracle
    for seed, _state, key in golden_pure["philox_keys"]:
        assert list(oracle.routing_key(seed)) == key


def test_route_uniform_counts(golden_pure):
    from oracle import oracle
    for T, E, k, seed, counts in golden_pure["route_uniform"]:
        got, st = oracle.route_uniform(T, E, k, seed)
        assert st == 0 and got == counts, (T, E, k, seed)


def test_attention_analytic(golden_pure):
    from oracle import oracle
    for phase, q, kv, hq, hkv, hd, us, _vec in golden_pure["attention"]:
        got = oracle.attention_us(phase == "decode", q, kv, hq, hkv, hd, 2.25e15, 8e12)
        assert got == us


def test_python_sum_emulation(golden_pure):
    from oracle import oracle
    for xs, want in golden_pure["py_sum"]:
        got = oracle.pysum(xs)
        assert got == want or (math.isnan(got) and math.isnan(want))


def _budget_specs(golden_scenarios, names):
    import dataclasses
    from parity import specs_for
    specs = []
    for n in names:
        g = golden_scenarios[n]
        (sp,) = specs_for([g["config"]])
        specs.append(dataclasses.replace(sp, max_events=g["events"]))      # exactly enough
        specs.append(dataclasses.replace(sp, max_events=g["events"] - 1))  # one short
    return specs


BUDGET_CASES = ("co_llama_40", "pd_2_3_paged_tight", "af_tiny_moe_m3_dp2", "co_moe_mixtral_ep2")


def test_event_budget_boundary_oracle(golden_scenarios):
    """core.py:186-191: EventBudgetExceeded once processed > max_events."""
    from oracle import oracle
    from paper_2508_03148_b200.lower import lower
    raw = oracle.run(lower(_budget_specs(golden_scenarios, BUDGET_CASES)))
    assert raw.rows["status"].tolist() == [0, 3] * len(BUDGET_CASES)
