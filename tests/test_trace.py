"""EventTrace parity: the reference's trace (core.py:85-129) rendered from the
engine's / oracle's event log.

CPU tests pin the renderer with the C oracle's event log against the trace
hashes the reference produced (tests/golden), and -- where /root/reference is
importable (the build container) -- line by line against the reference's own
trace. GPU tests run the public drop-in path (make_simulation -> run() ->
EventTrace, run_one, the `run` CLI) and compare device records with the oracle's.
"""

import copy
import os
import sys

import numpy as np
import pytest

from parity import run_backend, specs_for
from paper_2508_03148_b200 import workloads as W
from paper_2508_03148_b200.metrics import compute_metrics
from paper_2508_03148_b200.trace import EventKind

REF_SRC = "/root/reference/pkg/src"


def _ok_names(golden):
    return [n for n in golden if "error" not in golden[n]]


def test_oracle_trace_hashes_match_reference(golden_scenarios):
    names = _ok_names(golden_scenarios)
    res = run_backend("oracle", [golden_scenarios[n]["config"] for n in names])
    got = {n: r.trace().hash for n, r in zip(names, res)}
    assert got == {n: golden_scenarios[n]["trace_hash"] for n in names}


def test_trace_api(golden_scenarios, tmp_path):
    g = golden_scenarios["pd_2_3_paged_tight"]
    (r,) = run_backend("oracle", [g["config"]])
    tr = r.trace()
    assert len(tr) == r.events == g["events"]
    lines = tr.lines()
    assert lines[0].split(",", 3)[2] == "REQUEST_ARRIVAL"
    assert [ (e.timestamp, e.seq) for e in tr] == sorted((e.timestamp, e.seq) for e in tr)
    assert len(tr.events_of_kind(EventKind.BATCH_COMPLETE)) == r.iterations
    assert len(tr.events_of_kind(EventKind.KV_CACHE_TRANSFER_START)) == \
        len(tr.events_of_kind(EventKind.KV_CACHE_TRANSFER_DONE))
    path = tmp_path / "trace.log"
    tr.export(str(path))
    data = path.read_bytes()
    assert data.endswith(f"#hash={g['trace_hash']}\n".encode())
    assert data[: -len(f"#hash={g['trace_hash']}\n")] == tr.body_bytes()
    # compute_metrics accepts the trace, as in the reference
    assert compute_metrics(tr).to_dict()["aggregates"] == g["metrics"]["aggregates"]


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present (GPU box)")
@pytest.mark.parametrize("name", ["co_2rep_paged_skip", "pd_2_3_paged_tight",
                                  "af_tiny_moe_m3_dp2", "co_moe_mixtral_ep2"])
def test_trace_lines_equal_reference(golden_scenarios, name):
    """Line-by-line against the reference's own EventTrace (build container only)."""
    sys.path.insert(0, REF_SRC)
    try:
        from frontier_sim.cli import run_one as ref_run_one
        from frontier_sim.config import parse_config as ref_parse
    finally:
        sys.path.remove(REF_SRC)
    doc = golden_scenarios[name]["config"]
    ref = ref_run_one(ref_parse(copy.deepcopy(doc)))["trace"].lines()
    (r,) = run_backend("oracle", [doc])
    mine = r.trace().lines()
    assert len(mine) == len(ref)
    bad = [i for i, (a, b) in enumerate(zip(mine, ref)) if a != b]
    assert bad == [], (mine[bad[0]], ref[bad[0]]) if bad else None


# ---- device --------------------------------------------------------------------------------

@pytest.mark.gpu
def test_run_one_trace_hash(engine, golden_scenarios, golden_baseline):
    from paper_2508_03148_b200.api import run_one
    from paper_2508_03148_b200.config import parse_config
    cases = {n: golden_scenarios[n] for n in _ok_names(golden_scenarios)}
    cases.update(golden_baseline)
    bad = {}
    for n, g in cases.items():
        out = run_one(parse_config(copy.deepcopy(g["config"])), engine=engine)
        if out["trace"].hash != g["trace_hash"]:
            bad[n] = out["trace"].hash
        m = out["metrics"].to_dict()
        if m["aggregates"] != g["metrics"]["aggregates"]:
            bad[n] = "metrics"
    assert bad == {}


@pytest.mark.gpu
def test_cli_run_writes_trace_artifacts(golden_scenarios, tmp_path):
    import json
    from paper_2508_03148_b200.cli import main
    g = golden_scenarios["co_llama_40"]
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps(g["config"]))
    assert main(["run", str(cfg), "--out", str(tmp_path / "out")]) == 0
    body = (tmp_path / "out" / "trace.log").read_bytes()
    assert body.endswith(f"#hash={g['trace_hash']}\n".encode())
    assert (tmp_path / "out" / "summary.csv").read_text().startswith("config_hash,")
    assert json.loads((tmp_path / "out" / "metrics.json").read_text())["config_hash"] == \
        g["config_hash"]


@pytest.mark.gpu
def test_event_log_device_equals_oracle(engine):
    """Raw event records (payload fields included) of 96 C5 instances and 4 AF / EP
    instances: device == oracle, record for record."""
    from oracle import oracle
    from paper_2508_03148_b200.engine import LogSpec
    from paper_2508_03148_b200.lower import lower
    from paper_2508_03148_b200.orchestrator import detail_log_spec
    docs = W.c5_sweep(n_seeds=2)[::4] + [W.c4_af(12), W.c4_colocated_ep(12)]
    for i, d in enumerate(docs[-2:]):
        d["seed"] = 31 + i
    specs = specs_for(docs)
    logs = [detail_log_spec(s, events=True) for s in specs]
    log = LogSpec(*(max(getattr(l, f) for l in logs) for f in
                    ("batch_cap", "member_cap", "moe_cap", "route_cap", "counts_cap",
                     "event_cap")))
    low = lower(specs)
    dev = engine.run(low, log=log)
    ref = oracle.run(low, log=log, threads=8)
    assert (dev.rows["status"] == 0).all()
    assert np.array_equal(dev.log.event_count, ref.log.event_count)
    assert np.array_equal(dev.log.event_count, dev.rows["events"])
    for i in range(low.n_instances):
        a, b = dev.log.instance_events(i), ref.log.instance_events(i)
        assert a.tobytes() == b.tobytes(), i
