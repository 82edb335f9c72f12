"""Shared comparison helpers for golden / oracle / device parity tests."""

from __future__ import annotations

import copy

from paper_2508_03148_b200.api import instance_spec
from paper_2508_03148_b200.config import parse_config
from paper_2508_03148_b200.lower import lower
from paper_2508_03148_b200.metrics import compute_metrics, split_results
from paper_2508_03148_b200.orchestrator import detail_log_spec

PHASE = {"prefill": "prefill", "decode": "decode", "af_decode": "af_decode"}


def specs_for(docs, base_dir="."):
    return [instance_spec(parse_config(copy.deepcopy(d), base_dir=base_dir)) for d in docs]


def run_backend(backend, docs, routes=False, threads=1, base_dir=".", events=True):
    """backend: 'oracle' or an Engine. events: also record the event trace."""
    specs = specs_for(docs, base_dir)
    low = lower(specs)
    logs = [detail_log_spec(s, routes=routes, events=events) for s in specs]
    from paper_2508_03148_b200.engine import LogSpec
    log = LogSpec(*(max(getattr(l, f) for l in logs) for f in
                    ("batch_cap", "member_cap", "moe_cap", "route_cap", "counts_cap",
                     "event_cap")))
    if backend == "oracle":
        from oracle import oracle
        raw = oracle.run(low, log=log, threads=threads)
    else:
        raw = backend.run(low, log=log)
    return split_results(low, raw, [s.deployment.mode for s in specs])


def compare_to_golden(res, g, check_routes=True):
    """Return a list of mismatch descriptions (empty == bit-exact parity)."""
    bad = []
    if "error" in g:
        if res.ok:
            bad.append(f"expected {g['error']['type']}, run succeeded")
        elif type(res.error()).__name__ != g["error"]["type"]:
            bad.append(f"error type {type(res.error()).__name__} != {g['error']['type']}")
        return bad
    if not res.ok:
        return [f"run failed: {res.error()!r}"]
    if res.request_ids != g["requests"]["ids"]:
        bad.append("request ids differ")
    if res.arrival_ns.tolist() != g["requests"]["arrival_ns"]:
        bad.append("arrivals differ")
    if res.first_token_ns.tolist() != g["first_token_ns"]:
        diff = [i for i, (a, b) in enumerate(zip(res.first_token_ns.tolist(), g["first_token_ns"])) if a != b]
        bad.append(f"first_token_ns differ at {diff[:5]}")
    if res.done_ns.tolist() != g["done_ns"]:
        diff = [i for i, (a, b) in enumerate(zip(res.done_ns.tolist(), g["done_ns"])) if a != b]
        bad.append(f"done_ns differ at {diff[:5]}")
    if res.completion_order() != g["completion_order"]:
        bad.append("completion order differs")
    if res.iterations != g["iterations"]:
        bad.append(f"iterations {res.iterations} != {g['iterations']}")
    if res.events != g["events"]:
        bad.append(f"events {res.events} != {g['events']}")
    if "trace_hash" in g and res.event_log is not None:
        if len(res.event_log) != res.events:
            bad.append(f"event log has {len(res.event_log)} records, {res.events} events")
        elif res.trace().hash != g["trace_hash"]:
            bad.append("trace hash differs")
    if "batches" in g and res.batches is not None:
        gb = g["batches"]
        if len(res.batches) != len(gb):
            bad.append(f"batch count {len(res.batches)} != {len(gb)}")
        for j, (mb, rb) in enumerate(zip(res.batches, gb)):
            rkey, phase, t, dur, ids, moe = rb
            mine_ids = [res.request_ids[m] for m in mb["members"]]
            if (res.replica_keys[mb["replica"]] != rkey or mb["phase"] != phase
                    or mb["t_complete"] != t or mb["duration_ns"] != dur or mine_ids != ids):
                bad.append(f"batch {j}: {(res.replica_keys[mb['replica']], mb['phase'], mb['t_complete'], mb['duration_ns'], mine_ids[:4])} != {(rkey, phase, t, dur, ids[:4])}")
                break
            mine_moe = [round(x, 6) for x in mb["moe_ratio"]] if mb["moe_ratio"] is not None else None
            if mine_moe != moe:
                bad.append(f"batch {j}: moe_imbalance differs")
                break
    if check_routes and "routes" in g and res.routes is not None:
        gr = g["routes"]
        if len(res.routes) != len(gr):
            bad.append(f"route count {len(res.routes)} != {len(gr)}")
        for j, (mr, rr) in enumerate(zip(res.routes, gr)):
            scope, step, layer, T, counts = rr
            key = res.replica_keys[mr["replica"]]
            mscope = key if mr["micro_batch"] == 0 else f"{key}:mb{mr['micro_batch']}"
            if (mscope, mr["step"], mr["layer"], mr["tokens"], mr["counts"]) != (scope, step, layer, T, counts):
                bad.append(f"route {j}: {(mscope, mr['step'], mr['layer'], mr['tokens'])} != {(scope, step, layer, T)}")
                break
    m = compute_metrics(res).to_dict()
    gm = g["metrics"]
    for key in ("aggregates", "total_tokens", "makespan_s", "total_gpus",
                "throughput_tokens_per_s_per_gpu", "busy_fraction", "bubble_fraction",
                "workload_summary", "per_request"):
        if key in gm and m[key] != gm[key]:
            bad.append(f"metrics.{key}: {str(m[key])[:200]} != {str(gm[key])[:200]}")
    if res.batches is not None and m["expert_imbalance"] != gm["expert_imbalance"]:
        bad.append("metrics.expert_imbalance differs")
    return bad
