"""Sweep driver: grid expansion, overrides (incl. list indices), point seeds."""

import copy
import hashlib
import json

import pytest

from paper_2508_03148_b200 import workloads as W
from paper_2508_03148_b200.config import ParseError, parse_config
from paper_2508_03148_b200.sweep import apply_overrides, grid_points, point_documents, point_seed


def test_grid_is_sorted_cartesian_product():
    pts = grid_points({"b": [1, 2], "a": ["x", "y", "z"]})
    assert len(pts) == 6
    assert pts[0] == {"a": "x", "b": 1} and pts[1] == {"a": "x", "b": 2}
    with pytest.raises(ParseError):
        grid_points({"a": []})


def test_point_seed_formula():
    ov = {"policies.max_num_seqs": 64}
    want = int.from_bytes(hashlib.sha256(
        f"7:{json.dumps(ov, sort_keys=True, separators=(',', ':'))}".encode()).digest()[:4], "big")
    assert point_seed(7, ov) == want


def test_dict_overrides_match_reference_semantics():
    doc = W.c1_colocated(8)
    out = apply_overrides(doc, {"policies.max_num_seqs": 32, "model.num_layers": 4})
    assert out["policies"]["max_num_seqs"] == 32 and out["model"]["num_layers"] == 4
    assert doc.get("policies") is None  # deep copy
    parse_config(out)


def test_list_index_overrides_address_clusters():
    doc = W.c5_sweep_configs(8)[16]  # PD
    doc["seed"] = 3
    out = apply_overrides(doc, {"clusters.1.num_replicas": 3, "clusters.0.parallelism.tp": 4,
                                "clusters.0.gpus_per_replica": 4})
    assert out["clusters"][1]["num_replicas"] == 3
    assert out["clusters"][0]["parallelism"]["tp"] == 4
    cfg = parse_config(out)
    assert cfg.clusters[0].parallelism.tp == 4


def test_workload_seed_follows_point_seed():
    doc = W.c1_colocated(8, seed=5)
    doc["workload"]["seed"] = 5
    docs = point_documents(doc, [{"policies.max_num_seqs": 16}], 5)
    assert "seed" not in docs[0]["workload"]
    assert docs[0]["seed"] == point_seed(5, {"policies.max_num_seqs": 16})
