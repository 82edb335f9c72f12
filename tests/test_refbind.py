"""The reference-side binding (paper_2508_03148_b200/refbind.py) run on
the reference's OWN config objects (frontier_sim.config.parse_config) and compared
with the reference's own run_one: trace hash, metrics.to_dict() (expert_imbalance
included) and exception types.

Build container only (the reference is not on the GPU box). The engine slot is
filled by the oracle behind the Engine interface (oracle.OracleEngine, test
infrastructure), so the binding's conversion path -- reference Deployment /
Request / SchedulerPolicy / RoutingPolicySpec / LearnedOperatorModel objects into
the engine's lowering -- is what is under test here; the CUDA engine is pinned to
the oracle by the GPU tests.
"""

import copy
import os
import sys

import pytest

REF_SRC = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present")

CASES = ["co_llama_40", "co_2rep_paged_skip", "co_moe_mixtral_ep2", "pd_2_3_paged_tight",
         "af_tiny_moe_m3_dp2", "af_dense_m4", "err_colocated_cannot_fit",
         "err_trace_routing_sum"]


_CACHE = {}


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, REF_SRC)
    try:
        from frontier_sim.cli import run_one
        from frontier_sim.config import parse_config
    finally:
        sys.path.remove(REF_SRC)
    return parse_config, run_one


def _engine():
    from oracle.oracle import OracleEngine
    return OracleEngine(threads=4)


def _ref_result(ref, doc, base_dir="."):
    import json
    key = (json.dumps(doc, sort_keys=True), base_dir)
    if key in _CACHE:
        return _CACHE[key]
    parse_config, run_one = ref
    cfg = parse_config(copy.deepcopy(doc), base_dir=base_dir)
    try:
        out = run_one(cfg)
        r = cfg, out["trace"].hash, out["metrics"].to_dict()
    except Exception as exc:
        r = cfg, type(exc).__name__, None
    _CACHE[key] = r
    return r


def test_run_one_on_reference_objects(ref, golden_scenarios):
    from paper_2508_03148_b200 import refbind
    for name in CASES:
        cfg, want_hash, want = _ref_result(ref, golden_scenarios[name]["config"])
        if want is None:
            with pytest.raises(Exception) as ei:
                refbind.run_one(cfg, engine=_engine())
            assert type(ei.value).__name__ == want_hash, name
            continue
        out = refbind.run_one(cfg, engine=_engine())
        assert out["trace"].hash == want_hash, name
        assert out["metrics"].to_dict() == want, name
        assert out["config_hash"] == cfg.config_hash()


def test_run_batch_on_reference_objects(ref, golden_scenarios):
    from paper_2508_03148_b200 import refbind
    refs = [_ref_result(ref, golden_scenarios[n]["config"]) for n in CASES]
    got = refbind.run_batch([r[0] for r in refs], engine=_engine())
    for name, (cfg, want_hash, want), g in zip(CASES, refs, got):
        if want is None:
            assert isinstance(g, Exception) and type(g).__name__ == want_hash, name
        else:
            assert g.to_dict() == want, name   # expert_imbalance too (second pass)


def test_learned_models_from_reference_objects(ref, golden_learned, model_dir):
    """LearnedOperatorModel objects the reference loaded are converted via their
    portable document (costmodel/model.py:140-152). learned_af_tiny_moe is re-run in
    the reference (1 s); the others take the reference 1-5 minutes, so they are
    compared with the fixtures it recorded."""
    from paper_2508_03148_b200 import refbind
    parse_config, _ = ref
    cfg, want_hash, want = _ref_result(ref, golden_learned["learned_af_tiny_moe"]["config"],
                                       model_dir)
    out = refbind.run_one(cfg, engine=_engine())
    assert out["trace"].hash == want_hash
    assert out["metrics"].to_dict() == want
    for name in ("learned_co_llama_40", "learned_both_pd_70b_30"):
        g = golden_learned[name]
        cfg = parse_config(copy.deepcopy(g["config"]), base_dir=model_dir)
        out = refbind.run_one(cfg, engine=_engine())
        assert out["trace"].hash == g["trace_hash"], name
        assert out["metrics"].to_dict()["aggregates"] == g["metrics"]["aggregates"], name
