"""Host-side logic: config parsing, workload generation, lowering, report helpers.

Pinned against the golden fixtures recorded from the reference (config
hashes, generated requests) and against the reference's documented rules
(unknown keys rejected, defaults, error classes).
"""

import copy
import math

import numpy as np
import pytest

from paper_2508_03148_b200 import abi
from paper_2508_03148_b200 import workloads as W
from paper_2508_03148_b200.api import instance_spec
from paper_2508_03148_b200.config import ParseError, ValidationError, parse_config
from paper_2508_03148_b200.lower import lower, replica_layout
from paper_2508_03148_b200.metrics import (MetricsBundle, pareto_frontier, summary_csv_row,
                                           SUMMARY_CSV_HEADER)
from paper_2508_03148_b200.topology import kv_bytes_per_token


def test_config_hash_matches_reference(golden_scenarios):
    for name, g in golden_scenarios.items():
        assert parse_config(copy.deepcopy(g["config"])).config_hash() == g["config_hash"], name


def test_generated_requests_match_reference(golden_scenarios, golden_baseline):
    for g in list(golden_scenarios.values()) + list(golden_baseline.values()):
        arr = parse_config(copy.deepcopy(g["config"])).request_arrays()
        assert arr.ids == g["requests"]["ids"]
        assert arr.arrival_ns.tolist() == g["requests"]["arrival_ns"]
        assert arr.prompt.tolist() == g["requests"]["prompt"]
        assert arr.output.tolist() == g["requests"]["output"]


def test_unknown_key_rejected():
    d = W.c1_colocated(4)
    d["policies"] = {"max_num_seqs": 8, "typo_key": 1}
    with pytest.raises(ParseError, match="unknown key"):
        parse_config(d)
    d = W.c1_colocated(4)
    d["extra"] = 1
    with pytest.raises(ParseError):
        parse_config(d)


def test_missing_and_mistyped_keys():
    d = W.c1_colocated(4)
    del d["model"]["d_ff"]
    with pytest.raises(ParseError, match="required key missing"):
        parse_config(d)
    d = W.c1_colocated(4)
    d["model"]["num_layers"] = 32.0
    with pytest.raises(ParseError, match="integer"):
        parse_config(d)
    d = W.c1_colocated(4)
    d["clusters"][0]["hardware"]["mem_bw"] = True
    with pytest.raises(ParseError, match="number"):
        parse_config(d)


def test_semantic_validation_errors():
    d = W.c1_colocated(4)
    d["mode"] = "split"
    with pytest.raises(ValidationError):
        parse_config(d)
    d = W.c1_colocated(4)
    d["clusters"][0]["gpus_per_replica"] = 2      # tp*pp*ep == 1
    with pytest.raises(ValidationError, match="gpus_per_replica"):
        parse_config(d)
    d = W.c1_colocated(4)
    d["policies"] = {"admission": "lifo"}
    with pytest.raises(ValidationError):
        parse_config(d)
    d = W.c4_af(4)
    d["clusters"][0]["parallelism"]["attn_dp"] = 2   # attn_dp*attn_tp != moe_tp*moe_ep
    with pytest.raises(ValidationError):
        parse_config(d)


def test_defaults_follow_reference():
    cfg = parse_config(W.c1_colocated(4))
    assert cfg.policy.admission == "fcfs" and cfg.policy.max_num_seqs == 256
    assert cfg.policy.max_batch_tokens == 8192 and cfg.policy.memory_mode == "exact"
    assert cfg.routing.policy == "uniform" and cfg.routing.alpha == 0.3
    assert cfg.activation_reserve_fraction == 0.1
    assert cfg.workload.seed == cfg.seed  # workload seed defaults to the master seed
    af = parse_config(W.c4_af(4))
    assert af.af.micro_batches == 2


def test_kv_pool_and_kv_bytes():
    dep = parse_config(W.c3_pd(4, tight=True)).deployment()
    assert kv_bytes_per_token(dep.model) == 327_680
    assert [c.kv_pool_tokens for c in dep.clusters][1] == 26_485  # tight pool


def test_replica_layout_and_key_ranks():
    d = W.c5_sweep_configs(8)[16 + 5]  # PD 2:3
    d["seed"] = 5
    d["clusters"][1]["num_replicas"] = 12   # keys d0/0 .. d0/11: "d0/10" < "d0/2"
    d["clusters"][1]["gpus_per_replica"] = 2
    spec = instance_spec(parse_config(d))
    layout = replica_layout(spec.deployment)
    assert [r.key for r in layout][:3] == ["p0/0", "p0/1", "d0/0"]
    low = lower([spec])
    ranks = {k: int(r["key_rank"]) for k, r in zip(low.replica_keys[0], low.replicas)}
    assert ranks["d0/10"] < ranks["d0/2"] and ranks["d0/11"] < ranks["d0/2"]
    assert ranks["d0/0"] < ranks["d0/1"] < ranks["d0/10"]


def test_lowering_prefixes_and_ids():
    spec = instance_spec(parse_config(W.c4_af(12, seed=77)))
    low = lower([spec])
    pf = low.prefixes
    assert bytes(pf[0]["bytes"][: pf[0]["len"]]) == b"77:attn/0:"
    assert bytes(pf[1]["bytes"][: pf[1]["len"]]) == b"77:attn/0:mb"
    assert int(low.replicas[0]["prefix_mb"]) == 1
    ids = low.request_ids[0]
    ranks = low.id_rank.tolist()
    assert sorted(range(len(ids)), key=lambda i: ids[i]) == sorted(range(len(ids)), key=lambda i: ranks[i])
    d = low.descs[0]
    assert d["af_attn"]["tp"] == 8 and d["af_ffn"]["ep"] == 8 and d["af_micro_batches"] == 2


def test_struct_layouts_are_c_layouts():
    assert abi.COST_CTX.itemsize == 40
    assert abi.SEED_PREFIX.itemsize == 232
    assert abi.REPLICA_DESC.itemsize == 64
    assert abi.BATCH_REC.itemsize == 64
    assert abi.EVENT_REC.itemsize == 40
    assert abi.ROUTE_REC.itemsize == 32


def _bundle(thr, p90):
    agg = None if p90 is None else {"mean": p90, "p50": p90, "p90": p90, "p99": p90}
    return MetricsBundle({}, agg, agg, agg, 0, 1.0, 1, thr, {}, None, [], {})


def test_pareto_frontier_bruteforce():
    rng = np.random.default_rng(3)
    pts = [(i, _bundle(float(rng.integers(0, 20)), float(rng.integers(0, 20)))) for i in range(60)]
    pts.append((60, _bundle(5.0, None)))
    front = {t for t, _ in pareto_frontier(pts)}
    for t, b in pts:
        dominated = any(
            o.throughput_tokens_per_s_per_gpu >= b.throughput_tokens_per_s_per_gpu
            and (o.tpot["p90"] if o.tpot else math.inf) <= (b.tpot["p90"] if b.tpot else math.inf)
            and (o.throughput_tokens_per_s_per_gpu > b.throughput_tokens_per_s_per_gpu
                 or (o.tpot["p90"] if o.tpot else math.inf) < (b.tpot["p90"] if b.tpot else math.inf))
            for s, o in pts if s != t)
        assert (t in front) == (not dominated)


def test_summary_csv_row_format():
    row = summary_csv_row(_bundle(1.5, 0.25), "abc")
    assert len(row) == len(SUMMARY_CSV_HEADER)
    assert row[0] == "abc" and row[1] == repr(1.5) and row[5] == repr(0.25)
    assert summary_csv_row(_bundle(1.0, None), "x")[5] == ""
