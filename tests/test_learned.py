"""Learned operator models (costmodel/model.py, forest.py, features.py).

CPU: model-file loading (format / hash / schema checks) and the oracle's
forest inference pinned against predictions made by the reference itself.
GPU: the batched forest kernel and learned-mode simulations, bit-exact
against the same fixtures (tolerance 0).
"""

import copy
import gzip
import json
import os

import numpy as np
import pytest

from parity import compare_to_golden, run_backend, specs_for
from paper_2508_03148_b200 import costmodel
from paper_2508_03148_b200.errors import ModelFileError, SchemaMismatch

RUNNABLE = ("learned_co_llama_40", "learned_pd_70b_tight_30", "learned_af_tiny_moe",
            "learned_gg_co_llama_40", "learned_both_pd_70b_30",
            "learned_gg_mode_analytic_still_loads", "learned_err_attention_schema")


def _csr(preds):
    q, kv, off, dec = [], [], [0], []
    for phase, qq, kk, _ in preds:
        q += qq
        kv += kk
        off.append(len(q))
        dec.append(1 if phase == "decode" else 0)
    return (np.array(q, np.int32), np.array(kv, np.int32), np.array(off, np.int64),
            np.array(dec, np.uint8), np.array([p[3] for p in preds]))


def test_model_files_load(model_dir):
    m = costmodel.load_model_file(os.path.join(model_dir, "forest_c2.json"))
    assert (m.operator, m.schema, m.n_trees, m.n_features) == ("attention", "attention_v1", 100, 17)
    g = costmodel.load_model_file(os.path.join(model_dir, "forest_gg_small.json"))
    assert (g.operator, g.schema, g.n_features) == ("grouped_gemm", "grouped_gemm_v1", 12)
    # every internal node's children lie inside its own tree
    assert (m.left[m.feature >= 0] > 0).all() and (m.feature < 17).all()


def test_model_file_tamper_detected(model_dir, tmp_path):
    doc = json.load(open(os.path.join(model_dir, "forest_small.json")))
    doc["trees"][0]["nodes"][0]["threshold"] = 1.0 + doc["trees"][0]["nodes"][0].get("threshold", 0)
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps(doc))
    with pytest.raises(ModelFileError):
        costmodel.load_model_file(str(bad))
    doc["format"] = "something-else"
    bad.write_text(json.dumps(doc))
    with pytest.raises(ModelFileError):
        costmodel.load_model_file(str(bad))


def test_model_slot_operator_check(model_dir):
    gg = costmodel.load_model_file(os.path.join(model_dir, "forest_gg_small.json"))
    with pytest.raises(SchemaMismatch):
        costmodel.check_model_slots(gg, None)
    att = costmodel.load_model_file(os.path.join(model_dir, "forest_small.json"))
    with pytest.raises(SchemaMismatch):
        costmodel.check_model_slots(None, att)


@pytest.mark.parametrize("name", ["forest_small", "forest_c2"])
def test_oracle_forest_predictions(model_dir, golden_forest_predictions, name):
    from oracle import oracle
    fs = costmodel.ForestSet()
    fs.add(costmodel.load_model_file(os.path.join(model_dir, f"{name}.json")))
    preds = golden_forest_predictions[name]
    got = [oracle.attention_forest(fs, 0, ph == "decode", q, kv, 32, 8, 128)[0]
           for ph, q, kv, _ in preds]
    want = [p[3] for p in preds]
    assert got == want


def test_oracle_learned_scenarios(model_dir, golden_learned):
    res = run_backend("oracle", [golden_learned[n]["config"] for n in RUNNABLE], routes=True,
                      base_dir=model_dir)
    bad = {n: compare_to_golden(r, golden_learned[n]) for n, r in zip(RUNNABLE, res)}
    assert {n: b for n, b in bad.items() if b} == {}


def test_operator_slot_mismatch_is_config_time(model_dir, golden_learned):
    g = golden_learned["learned_err_operator_slot"]
    assert g["error"]["type"] == "SchemaMismatch"
    with pytest.raises(SchemaMismatch):
        specs_for([g["config"]], model_dir)


# -- device ---------------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("name", ["forest_small", "forest_c2"])
def test_gpu_forest_predictions(engine, model_dir, golden_forest_predictions, name):
    from types import SimpleNamespace
    model = costmodel.load_model_file(os.path.join(model_dir, f"{name}.json"))
    q, kv, off, dec, want = _csr(golden_forest_predictions[name])
    hw = SimpleNamespace(peak_flops=2.25e15, mem_bw=8.0e12, kernel_overhead_us=5.0)
    got = costmodel.attention_cost_batches(q, kv, off, dec, 32, 8, 128, hw, model=model,
                                           engine=engine)
    assert engine.last_launch_count >= 1
    assert got.tolist() == want.tolist()


@pytest.mark.gpu
def test_gpu_learned_scenarios(engine, model_dir, golden_learned):
    res = run_backend(engine, [golden_learned[n]["config"] for n in RUNNABLE], routes=True,
                      base_dir=model_dir)
    bad = {n: compare_to_golden(r, golden_learned[n]) for n, r in zip(RUNNABLE, res)}
    assert {n: b for n, b in bad.items() if b} == {}


@pytest.mark.gpu
def test_gpu_learned_mixed_batch_matches_oracle(engine, model_dir, golden_learned):
    """Analytic and learned instances in one launch (the learned kernel variant
    runs the analytic instances too) equal the oracle field by field."""
    from paper_2508_03148_b200 import workloads as W
    from test_gpu_parity import assert_same_raw
    from paper_2508_03148_b200.lower import lower
    from oracle import oracle
    docs = [golden_learned[n]["config"] for n in RUNNABLE if "error" not in golden_learned[n]] + \
        [W.c1_colocated(30, seed=s) for s in range(3)]
    low = lower(specs_for(docs, model_dir))
    assert_same_raw(engine.run(low), oracle.run(low, threads=4))


@pytest.mark.gpu
def test_gpu_simulate_learned_failures(engine, model_dir, golden_learned):
    from paper_2508_03148_b200.api import Failure, simulate
    names = list(golden_learned)
    out = simulate([copy.deepcopy(golden_learned[n]["config"]) for n in names], engine=engine,
                   base_dir=model_dir)
    for n, o in zip(names, out):
        if "error" in golden_learned[n]:
            assert isinstance(o, Failure) and type(o.exception).__name__ == "SchemaMismatch", n
        else:
            assert not isinstance(o, Failure), (n, o)


# -- learned grouped-GEMM model on MoE layers (moe.py:95-106, model.py:323-326) --------------

@pytest.fixture(scope="module")
def golden_learned_moe():
    from conftest import load_golden
    return load_golden("learned_moe")["data"]


def test_oracle_gg_local_feature_vectors(model_dir, golden_learned_moe):
    """GroupedGemmFeatures(..., "local").vector() bits and predictions (400 rank loads)."""
    from oracle import oracle
    fs = costmodel.ForestSet()
    fs.add(costmodel.load_model_file(os.path.join(model_dir, "forest_gg_small.json")))
    for counts, dm, dff, k, bits, pred in golden_learned_moe["gg_vectors"]:
        x, v = oracle.gg_features(counts, dm, dff, k, fs, 0)
        assert x.view(np.uint64).tolist() == bits, counts
        assert v == pred, counts


def test_oracle_learned_moe_scenarios(model_dir, golden_learned_moe):
    sc = golden_learned_moe["scenarios"]
    names = list(sc)
    res = run_backend("oracle", [sc[n]["config"] for n in names], routes=True, threads=4,
                      base_dir=model_dir)
    bad = {n: compare_to_golden(r, sc[n]) for n, r in zip(names, res)}
    assert {n: b for n, b in bad.items() if b} == {}


@pytest.mark.gpu
def test_gpu_learned_moe_scenarios(engine, model_dir, golden_learned_moe):
    sc = golden_learned_moe["scenarios"]
    names = list(sc)
    res = run_backend(engine, [sc[n]["config"] for n in names], routes=True, base_dir=model_dir)
    bad = {n: compare_to_golden(r, sc[n]) for n, r in zip(names, res)}
    assert {n: b for n, b in bad.items() if b} == {}
