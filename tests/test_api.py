"""Host API semantics of simulate() / run_sweep (api.py, sweep.py) on CPU.

The engine slot is filled by the oracle behind the Engine interface
(oracle.OracleEngine, test infrastructure): these tests pin the host logic --
per-point failure capture, expert_imbalance, the rows-only sweep path -- not the
device arithmetic (tests marked gpu do that).
"""

import copy
import csv
import json

import pytest

from oracle.oracle import OracleEngine
from paper_2508_03148_b200 import workloads as W
from paper_2508_03148_b200.api import Failure, simulate, simulate_rows
from paper_2508_03148_b200.metrics import MetricsBundle


@pytest.fixture(scope="module")
def eng():
    return OracleEngine(threads=4)


def test_per_point_failures_do_not_sink_the_batch(eng, tmp_path, golden_scenarios):
    good = golden_scenarios["co_llama_40"]["config"]
    empty_trace = tmp_path / "empty.csv"
    empty_trace.write_text("request_id,arrival_ns,prompt_tokens,output_tokens\n")
    no_requests = copy.deepcopy(good)
    no_requests["workload"] = {"trace_path": str(empty_trace)}
    af_two = copy.deepcopy(golden_scenarios["af_dense_m4"]["config"])
    af_two["clusters"][0]["num_replicas"] = 2        # AF takes a single pipeline
    dup_cap = copy.deepcopy(good)
    dup_cap["model"]["moe"] = {"num_experts": 4096, "top_k": 2, "expert_d_ff": 64}
    out = simulate([good, no_requests, af_two, dup_cap, good], engine=eng)
    assert isinstance(out[0], MetricsBundle) and isinstance(out[4], MetricsBundle)
    assert out[0].to_dict() == out[4].to_dict()
    assert isinstance(out[1], Failure) and type(out[1].exception).__name__ == "IncompleteTrace"
    assert isinstance(out[2], Failure) and type(out[2].exception).__name__ == "ValueError"
    assert isinstance(out[3], Failure)


def test_expert_imbalance_filled_by_simulate(eng, golden_scenarios):
    names = ["co_moe_mixtral_ep2", "pd_moe_mixtral", "co_llama_40", "af_tiny_moe_m3_dp2"]
    out = simulate([golden_scenarios[n]["config"] for n in names], engine=eng)
    for n, m in zip(names, out):
        assert m.expert_imbalance == golden_scenarios[n]["metrics"]["expert_imbalance"], n
    off = simulate([golden_scenarios[names[0]]["config"]], engine=eng, expert_imbalance=False)
    assert off[0].expert_imbalance is None


def test_rows_path_matches_bundles(eng):
    docs = W.c5_sweep(n_seeds=1, n_requests=12, configs=[0, 17, 40, 63])
    bundles = simulate(docs, engine=eng, expert_imbalance=False)
    sr = simulate_rows(docs, engine=eng)
    for i, b in enumerate(bundles):
        r = sr.bundle(i)
        assert (r.ttft, r.tpot, r.e2e, r.makespan_s, r.throughput_tokens_per_s_per_gpu) == \
            (b.ttft, b.tpot, b.e2e, b.makespan_s, b.throughput_tokens_per_s_per_gpu)


def test_sweep_override_failure_is_a_row(eng, tmp_path):
    from paper_2508_03148_b200.config import parse_config
    from paper_2508_03148_b200.sweep import run_sweep
    cfg = parse_config(W.c1_colocated(8))
    grid = {"policies.max_num_seqs": [4, 8], "workload.arrival.kind.sub": [1]}
    run_sweep(cfg, grid, str(tmp_path), engine=eng)
    rows = list(csv.reader(open(tmp_path / "sweep.csv")))
    assert len(rows) == 3 and all(r[2].startswith("failed: ") for r in rows[1:])
    grid = {"policies.max_num_seqs": [4, 8, 0]}
    summary = run_sweep(cfg, grid, str(tmp_path), engine=eng)
    rows = list(csv.reader(open(tmp_path / "sweep.csv")))
    assert [r[2].split(":")[0] for r in rows[1:]] == ["ok", "ok", "failed"]
    assert summary["ok"] == 2
    assert json.load(open(tmp_path / "frontier.json"))


def test_pipelined_batches_equal_one_batch(eng, golden_scenarios, monkeypatch):
    """simulate() splits a large mixed input into a MoE batch and a dense batch on two
    engines (api._pipeline_groups); every bundle and failure equals the one-batch run."""
    import paper_2508_03148_b200.api as api
    names = ["co_moe_mixtral_ep2", "co_llama_40", "pd_moe_mixtral", "af_dense_m4",
             "af_tiny_moe_m3_dp2"]
    docs = [golden_scenarios[n]["config"] for n in names]
    bad = copy.deepcopy(docs[1])
    bad["clusters"][0]["num_replicas"] = 0
    docs.insert(2, bad)
    one = simulate(copy.deepcopy(docs), engine=eng)
    monkeypatch.setattr(api, "PIPELINE_MIN", 2)
    groups = api._pipeline_groups(
        [api.parse_config(copy.deepcopy(d)) if i != 2 else None for i, d in enumerate(docs)],
        [None] * len(docs))
    assert groups == [[0, 3, 5], [1, 4]]
    two = simulate(copy.deepcopy(docs), engine=eng)
    for a, b in zip(one, two):
        if isinstance(a, Failure):
            assert isinstance(b, Failure) and a.status == b.status
        else:
            assert a.to_dict() == b.to_dict()
