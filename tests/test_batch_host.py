"""The batched host path (parse_many, template-based lower) against the
one-config-at-a-time path: a sweep's seed points share one parse, one
validation and one descriptor template, and must produce exactly what parsing
and lowering each document on its own produces -- configs, config hashes
(pinned to the reference's in test_host.py), lowered byte arrays, and per-point
failures."""

import copy

import numpy as np

from paper_2508_03148_b200 import workloads as W
from paper_2508_03148_b200.api import Failure, instance_spec, parse_all
from paper_2508_03148_b200.config import parse_config, parse_many
from paper_2508_03148_b200.lower import lower


def _docs(golden_scenarios):
    docs = W.c5_sweep(n_seeds=3, n_requests=12, configs=list(range(0, 64, 3)))
    for g in golden_scenarios.values():  # every mode / policy; seeds varied below
        for s in (0, 11, 12345):
            d = copy.deepcopy(g["config"])
            d["seed"] = s
            docs.append(d)
            d2 = copy.deepcopy(d)
            if isinstance(d2.get("workload"), dict) and "arrival" in d2["workload"]:
                d2["workload"]["seed"] = s + 7  # explicit workload seed
                docs.append(d2)
    return docs


def test_parse_many_equals_parse_config(golden_scenarios):
    docs = _docs(golden_scenarios)
    one = [parse_config(copy.deepcopy(d)) for d in docs]
    many = parse_many(copy.deepcopy(docs))
    assert len(one) == len(many)
    for a, b in zip(one, many):
        assert a == b
        assert a.to_document() == b.to_document()
        assert a.config_hash() == b.config_hash()
        assert a.deployment() == b.deployment()
        assert a.workload == b.workload
    # seed points of one config share their parse (and validation) ...
    shared = {id(c.__dict__.get("_shared")) for c in many}
    assert len(shared) < len(many)
    # ... but every point carries its own seeds
    assert len({(c.seed, c.workload.seed if c.workload else None) for c in many}) > len(shared)


def test_template_lower_equals_per_instance_lower(golden_scenarios):
    docs = [d for d in _docs(golden_scenarios)
            if "trace_path" not in d.get("workload", {})]
    solo = [instance_spec(parse_config(copy.deepcopy(d))) for d in docs]
    shared = [instance_spec(c) for c in parse_many(copy.deepcopy(docs))]
    a = lower(solo)
    b = lower(shared)
    for f in ("descs", "replicas", "prefixes", "trace_counts", "arrival", "prompt", "output",
              "id_rank"):
        x, y = getattr(a, f), getattr(b, f)
        assert x.dtype == y.dtype and x.tobytes() == y.tobytes(), f
    assert a.replica_keys == b.replica_keys
    assert a.request_ids == b.request_ids
    # and per-instance lowering agrees with the batch
    for i in (0, 5, len(docs) - 1):
        one = lower([solo[i]])
        d = a.descs[i].copy()
        d["req_offset"] = 0
        d["replica_offset"] = 0
        d["trace_offset"] = 0
        assert one.descs[0].tobytes() == d.tobytes()


def test_parse_all_failures_per_point():
    good = W.c1_colocated(4)
    bad_model = copy.deepcopy(good)
    bad_model["model"] = {"name": "broken"}
    bad_seed = copy.deepcopy(good)
    bad_seed["seed"] = "seven"  # takes the full parse and its error message
    neg = copy.deepcopy(good)
    neg["workload"]["num_requests"] = 0
    out = parse_all([good, bad_model, bad_seed, neg, copy.deepcopy(bad_model)])
    assert not isinstance(out[0], Failure)
    for i in (1, 2, 4):
        assert isinstance(out[i], Failure), i
    assert "seed" in out[2].status
    assert out[1].status == out[4].status
    ref = []
    for d in (bad_model, bad_seed, neg):
        try:
            parse_config(copy.deepcopy(d))
            ref.append(None)
        except Exception as exc:  # the one-at-a-time path's verdict
            ref.append(f"failed: {type(exc).__name__}: {exc}")
    got = [o.status if isinstance(o, Failure) else None for o in out[1:4]]
    assert got == ref


def test_shared_request_ids_are_ranked_like_python_strings():
    from paper_2508_03148_b200.lower import _id_ranks, shared_ids
    for n in (1, 9, 10, 11, 64, 1000):
        ids = shared_ids(n)
        assert ids is shared_ids(n) and ids == [f"r{k}" for k in range(n)]
        order = sorted(range(n), key=ids.__getitem__)
        rank = np.empty(n, np.int64)
        rank[order] = np.arange(n)
        assert (_id_ranks(ids) == rank).all()


def test_metrics_many_equals_compute_metrics(golden_scenarios):
    """api.metrics_many (row fields read once per batch) builds exactly the bundles
    (or failures) compute_metrics builds instance by instance."""
    from oracle.oracle import OracleEngine
    from paper_2508_03148_b200.api import _metrics_or_failure, metrics_many, run_specs
    docs = [copy.deepcopy(g["config"]) for g in golden_scenarios.values()]
    docs += W.c5_sweep(n_seeds=1, n_requests=8, configs=list(range(0, 64, 9)))
    specs = []
    for d in docs:
        try:
            specs.append(instance_spec(parse_config(d)))
        except Exception:
            continue
    run = run_specs(specs, OracleEngine(threads=4))
    got = metrics_many(run)  # from the batch columns: no InstanceResult built
    assert run._results is None
    want = [_metrics_or_failure(r) for r in run.results]
    again = metrics_many(run)  # and through the InstanceResults

    def key(b):
        return b.status if isinstance(b, Failure) else b.to_dict()
    assert [key(b) for b in again] == [key(b) for b in got]
    assert len(got) == len(want)
    for a, b in zip(got, want):
        if isinstance(b, Failure):
            assert isinstance(a, Failure) and a.status == b.status
        else:
            assert a.to_dict() == b.to_dict()
    assert any(isinstance(b, Failure) for b in want) and not all(isinstance(b, Failure) for b in want)
