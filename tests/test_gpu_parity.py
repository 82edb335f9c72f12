"""Device engine parity: CUDA path vs golden fixtures and vs the C oracle.

Bit-exact for integer state (batch composition, expert counts, completion
order, event counts) and for every fp64 latency/percentile (the engine
reproduces Python's operation order; tolerance 0).
"""

import copy

import numpy as np
import pytest

from parity import compare_to_golden, run_backend
from paper_2508_03148_b200 import workloads as W
from paper_2508_03148_b200.api import instance_spec
from paper_2508_03148_b200.config import parse_config
from paper_2508_03148_b200.lower import lower

pytestmark = pytest.mark.gpu

ROW_FIELDS = ("status", "iterations", "events", "total_tokens", "makespan_ns", "prefill_batches",
              "decode_batches", "af_steps", "n_tpot", "makespan_s",
              "throughput_tokens_per_s_per_gpu", "ttft", "tpot", "e2e", "avg_input_tokens",
              "avg_output_tokens", "af_busy_ns", "af_busy_fraction", "routing_calls",
              "routing_draws")


def assert_same_raw(dev, ref):
    assert (dev.first_ns == ref.first_ns).all()
    assert (dev.done_ns == ref.done_ns).all()
    assert (dev.done_rank == ref.done_rank).all()
    for f in ROW_FIELDS:
        a, b = dev.rows[f], ref.rows[f]
        same = (a == b) | (np.isnan(a) & np.isnan(b)) if a.dtype.kind == "f" else (a == b)
        assert np.all(same), f
    bf_a, bf_b = dev.rows["bubble_fraction"], ref.rows["bubble_fraction"]
    assert np.all((bf_a == bf_b) | (np.isnan(bf_a) & np.isnan(bf_b)))
    assert (dev.replica_out["busy_ns"] == ref.replica_out["busy_ns"]).all()
    assert (dev.replica_out["steps_executed"] == ref.replica_out["steps_executed"]).all()


def test_scenarios_vs_golden(engine, golden_scenarios):
    names = list(golden_scenarios)
    res = run_backend(engine, [golden_scenarios[n]["config"] for n in names], routes=True)
    failures = {n: compare_to_golden(r, golden_scenarios[n]) for n, r in zip(names, res)}
    assert {n: b for n, b in failures.items() if b} == {}


@pytest.mark.parametrize("name", ["C1_colocated_llama7b_1000", "C3_pd_70b_tight_300",
                                  "C3_pd_70b_roomy_300", "C4_af_dsv3_10", "C4_colocated_ep8_10"])
def test_baseline_configs_vs_golden(engine, golden_baseline, name):
    g = golden_baseline[name]
    r = run_backend(engine, [g["config"]], routes=name.startswith("C4"))[0]
    assert compare_to_golden(r, g) == []


def test_c5_design_points_vs_golden(engine, golden_c5):
    base = W.c5_sweep_configs(64)
    docs = []
    for ci in range(64):
        d = copy.deepcopy(base[ci])
        d["seed"] = 1000 + 64 * ci
        docs.append(d)
    res = run_backend(engine, docs)
    bad = {ci: compare_to_golden(r, golden_c5[str(ci)]) for ci, r in enumerate(res)}
    assert {k: v for k, v in bad.items() if v} == {}


def test_full_c5_sweep_vs_oracle(engine):
    """All 64 configs x 8 seeds: device == oracle on every output array."""
    from oracle import oracle
    docs = W.c5_sweep(n_seeds=8)
    low = lower([instance_spec(parse_config(d)) for d in docs])
    dev = engine.run(low)
    ref = oracle.run(low, threads=8)
    assert_same_raw(dev, ref)


def test_route_uniform_vectors(engine, golden_pure):
    groups = {}
    for T, E, k, seed, counts in golden_pure["route_uniform"]:
        groups.setdefault((E, k), []).append((T, seed, counts))
    for (E, k), calls in groups.items():
        counts, st = engine.route_uniform([c[0] for c in calls], [c[1] for c in calls], E, k)
        assert (st == 0).all()
        assert counts.tolist() == [c[2] for c in calls]


def test_router_seed_vectors(engine, golden_pure):
    rows = golden_pure["router_seed"]
    prefixes = [f"{m}:{s}:" for m, s, _, _, _ in rows]
    got = engine.router_seeds(prefixes, list(range(len(rows))), [0] * len(rows),
                              [r[2] for r in rows], [r[3] for r in rows])
    assert got.tolist() == [r[4] for r in rows]


def test_attention_cost_vectors(engine, golden_pure):
    from paper_2508_03148_b200.engine import attn_params
    for phase, q, kv, hq, hkv, hd, us, vec in golden_pure["attention"]:
        off = np.array([0, len(q)], dtype=np.int64)
        p = attn_params(hq, hkv, hd, 2, 2.25e15, 8e12, 5.0)
        out, st = engine.attention_cost(q, kv, off, [phase == "decode"], p)
        assert st[0] == 0 and out[0] == us
        feats = engine.attention_features(q, kv, off, [phase == "decode"], p)
        assert feats[0].tolist() == vec


def test_attention_cost_bulk_vs_oracle(engine):
    from oracle import oracle
    from paper_2508_03148_b200.engine import attn_params
    q, kv, off, dec = W.attention_batches(4096)
    p = attn_params(32, 8, 128, 2, 2.25e15, 8e12, 5.0)
    out, st = engine.attention_cost(q, kv, off, dec, p)
    assert (st == 0).all()
    for b in range(0, 4096, 97):
        s, e = off[b], off[b + 1]
        assert out[b] == oracle.attention_us(bool(dec[b]), q[s:e], kv[s:e], 32, 8, 128, 2.25e15, 8e12)


@pytest.mark.parametrize("mode", ["tpb", "tma", "warp", "g4a"])
def test_attention_cost_kernel_variants_agree(engine, mode, monkeypatch):
    """Every C2 kernel variant (FS_C2) gives the default's bits, incl. ragged,
    empty and invalid batches and an unaligned CSR start."""
    from paper_2508_03148_b200.engine import attn_params
    rs = np.random.default_rng(5)
    lens = rs.integers(0, 300, size=3000)
    lens[::97] = 0                                   # empty batches
    off = np.concatenate([[3], 3 + np.cumsum(lens)]).astype(np.int64)  # unaligned start
    n = int(off[-1])
    kv = np.clip(rs.lognormal(6.5, 1.4, size=n), 1, 32768).astype(np.int32)
    dec = (np.arange(3000) % 2).astype(np.uint8)
    q = np.maximum(1, kv - rs.integers(0, 3, size=n)).astype(np.int32)  # c == l and c > l
    for b in range(3000):
        if dec[b]:
            q[off[b]:off[b + 1]] = 1
    q[off[500]] = 0                                   # invalid members: l < 1,
    kv[off[900]] = np.iinfo(np.int32).min             # c < 0 (c - l wraps in int32),
    q[off[701]] = 2                                   # a decode member with l != 1,
    kv[off[703]] = 0                                  # a decode member with c < 1,
    kv[off[902]] = q[off[902]] - 1                    # a prefill member with c < l
    for b in (500, 900, 701, 703, 902):
        assert off[b + 1] > off[b] and bool(dec[b]) == (b % 2 == 1)
    q[off[1000]:off[1001]] = kv[off[1000]:off[1001]] = 2 ** 30  # past the exact-integer guard
    p = attn_params(32, 8, 128, 2, 2.25e15, 8e12, 5.0)
    monkeypatch.delenv("FS_C2", raising=False)
    want, wst = engine.attention_cost(q, kv, off, dec, p)
    monkeypatch.setenv("FS_C2", mode)
    got, gst = engine.attention_cost(q, kv, off, dec, p)
    assert (gst == wst).all()
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    assert all(wst[b] != 0 for b in (500, 900, 701, 703, 902)) and wst[1000] == 0
    assert (wst == 0).sum() > 2500


def test_sweep_driver_end_to_end(engine, tmp_path):
    """run_sweep on the GPU: ok rows equal the oracle's metrics, failures become rows."""
    import csv

    from oracle import oracle
    from paper_2508_03148_b200.sweep import grid_points, point_documents, run_sweep
    doc = W.c1_colocated(24, seed=11)
    cfg = parse_config(copy.deepcopy(doc))
    grid = {"policies.max_num_seqs": [4, 32], "clusters.0.hardware.hbm_capacity_bytes": [11.2e9, 180e9]}
    summary = run_sweep(cfg, grid, str(tmp_path), engine=engine)
    assert summary["points"] == 4
    with open(tmp_path / "sweep.csv") as fh:
        rows = list(csv.DictReader(fh))
    docs = point_documents(cfg.to_document(), grid_points(grid), cfg.seed)
    low = lower([instance_spec(parse_config(d)) for d in docs])
    ref = oracle.run(low)
    for r, st, thr in zip(rows, ref.rows["status"], ref.rows["throughput_tokens_per_s_per_gpu"]):
        if st == 0:
            assert r["status"] == "ok" and float(r["throughput_tokens_per_s_per_gpu"]) == thr
        else:
            assert r["status"].startswith("failed: RequestCannotFit")
    assert (tmp_path / "frontier.json").exists()


def test_event_budget_boundary_device(engine, golden_scenarios):
    """core.py:186-191 on the device: exactly enough events passes, one short fails."""
    from test_oracle_golden import BUDGET_CASES, _budget_specs
    raw = engine.run(lower(_budget_specs(golden_scenarios, BUDGET_CASES)))
    assert raw.rows["status"].tolist() == [0, 3] * len(BUDGET_CASES)


def test_baseline_full_sizes_vs_oracle_with_invariants(engine):
    """BASELINE C1 (1,000 requests) and C4 (AF m=2 and EP=8, DeepSeek-V3 shape) at the
    GPU's 64-request instance size: device == oracle on every output, plus
    size-independent properties -- every request completes after its first token,
    every router call tallies exactly T * top_k expert slots, iterations add up."""
    from oracle import oracle
    from parity import run_backend
    docs = [W.c1_colocated(1000, seed=7), W.c4_af(64, seed=5), W.c4_colocated_ep(64, seed=6)]
    low = lower([instance_spec(parse_config(copy.deepcopy(d))) for d in docs])
    dev = engine.run(low)
    assert (dev.rows["status"] == 0).all()
    assert_same_raw(dev, oracle.run(low, threads=3))
    res = run_backend(engine, docs, routes=True)
    for r, d in zip(res, docs):
        assert r.ok
        assert (r.first_token_ns >= r.arrival_ns).all() and (r.done_ns >= r.first_token_ns).all()
        assert sorted(r.completion_order()) == sorted(r.request_ids)
        k = d["model"].get("moe", {}).get("top_k", 0)
        for rt in (r.routes or []):
            assert sum(rt["counts"]) == rt["tokens"] * k
        assert r.iterations == len(r.batches)


@pytest.mark.parametrize("env", [{"FS_SPLIT_FAMILIES": "0"}, {"FS_DENSE_VARIANT": "0"}, {"FS_COMOE_VARIANT": "0"},
                                 {"FS_CHUNK_BLOCKS": "16"}, {"FS_NO_LONGROW": "1"}])
def test_dispatch_knobs_do_not_change_results(engine, env, monkeypatch):
    """Wave split, kernel-variant choice and chunk geometry are scheduling only:
    a mixed batch (dense, Mixtral, DeepSeek-V3, PD) gives the same bytes."""
    from paper_2508_03148_b200.engine import Engine
    docs = W.c5_sweep(n_seeds=1)[::3] + [W.c4_colocated_ep(8, seed=3), W.c3_pd(20, seed=4)]
    low = lower([instance_spec(parse_config(copy.deepcopy(d))) for d in docs])
    want = engine.run(low)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    other = Engine(0)  # knobs are read when the engine is created
    got = other.run(low)
    assert got.rows.tobytes() == want.rows.tobytes()
    assert np.array_equal(got.first_ns, want.first_ns) and np.array_equal(got.done_ns, want.done_ns)


def test_per_variant_waves_match_solo_runs(engine):
    """A heterogeneous batch runs as one wave per kernel variant (learned /
    dirichlet, long-row, sweep, dense; fs_stage): every instance's outputs equal
    its own single-instance run and the oracle's."""
    from oracle import oracle
    dsv3_dir = W.c4_colocated_ep(12, seed=5)
    dsv3_dir["routing"] = {"policy": "dirichlet_skew", "alpha": 0.3}
    mix_dir = W.c5_sweep_configs(4)[48 + 2]
    mix_dir = copy.deepcopy(mix_dir)
    mix_dir["routing"] = {"policy": "dirichlet_skew", "alpha": 1.0}
    docs = (W.c5_sweep(n_seeds=1, n_requests=16)[::5]
            + [W.c4_colocated_ep(10, seed=3), dsv3_dir, mix_dir, W.c3_pd(12, seed=4)])
    specs = [instance_spec(parse_config(copy.deepcopy(d))) for d in docs]
    batch = engine.run(lower(specs))
    ref = oracle.run(lower(specs))
    assert_same_raw(batch, ref)
    for i in (0, len(docs) - 4, len(docs) - 3, len(docs) - 2, len(docs) - 1):
        solo = engine.run(lower([specs[i]]))
        o = int(lower(specs).descs[i]["req_offset"])
        n = len(specs[i].requests)
        assert solo.rows.tobytes() == batch.rows[i:i + 1].tobytes(), i
        assert np.array_equal(solo.first_ns, batch.first_ns[o:o + n]), i
        assert np.array_equal(solo.done_ns, batch.done_ns[o:o + n]), i


def test_simulate_pipeline_on_two_engines(engine, monkeypatch):
    """simulate() on a mixed C5 slice: the MoE batch on the engine and the dense batch on
    its peer, launched back to back (the second staged while the first runs), give the
    same bundles as one batch, and the same as the C oracle."""
    import paper_2508_03148_b200.api as api
    from oracle.oracle import OracleEngine
    from paper_2508_03148_b200.api import simulate
    docs = W.c5_sweep(n_seeds=2, n_requests=24, configs=list(range(0, 64, 3)))
    one = simulate(copy.deepcopy(docs), engine=engine, device_workload=True)
    monkeypatch.setattr(api, "PIPELINE_MIN", 2)
    two = simulate(copy.deepcopy(docs), engine=engine, device_workload=True)
    ref = simulate(copy.deepcopy(docs), engine=OracleEngine(threads=8))
    assert any(d["model"].get("moe") for d in docs) and any(not d["model"].get("moe") for d in docs)
    for a, b, c in zip(one, two, ref):
        assert a.to_dict() == b.to_dict() == c.to_dict()


@pytest.mark.parametrize("experts,top_k", [(8, 1), (8, 3), (12, 2), (16, 3), (32, 8), (10, 2),
                                           (64, 1), (64, 3), (128, 8)])
def test_routing_shapes_vs_oracle(engine, experts, top_k):
    """Router shapes around the whole-row pass (process_rows: nseg == 1, E % 4 == 0,
    top_k 1-3 and 8) and outside it (E % 4 != 0), on the sweep, analytic and long-row
    kernels: device == oracle on every output (statuses included), and every router
    call of a completed instance tallies exactly T * top_k expert slots."""
    from oracle import oracle
    from parity import run_backend
    base = [d for d in W.c5_sweep(n_seeds=1, n_requests=24) if d["model"].get("moe")]
    docs = []
    for j, d in enumerate(base[::3]):
        d = copy.deepcopy(d)
        d["model"]["moe"]["num_experts"] = experts
        d["model"]["moe"]["top_k"] = top_k
        cl = d["clusters"][0]
        ep0 = ep = cl.get("parallelism", {}).get("ep", 1)
        while experts % ep:
            ep //= 2
        cl.setdefault("parallelism", {})["ep"] = ep
        cl["gpus_per_replica"] = cl["gpus_per_replica"] // ep0 * ep  # = tp * pp * ep
        d["seed"] = 31 + j
        docs.append(d)
    low = lower([instance_spec(parse_config(copy.deepcopy(d))) for d in docs])
    dev = engine.run(low)
    # large expert counts at ep 1-2 leave no KV room (RequestCannotFit, as the reference)
    assert (dev.rows["status"] == 0).sum() >= 2, dev.rows["status"]
    ref = oracle.run(low, threads=8)
    assert (dev.rows["status"] == ref.rows["status"]).all()
    ok = dev.rows["status"] == 0  # a failed instance's row carries no metrics
    assert (dev.first_ns == ref.first_ns).all() and (dev.done_ns == ref.done_ns).all()
    for f in ROW_FIELDS:
        a, b = dev.rows[f][ok], ref.rows[f][ok]
        assert np.all((a == b) | (np.isnan(a) & np.isnan(b)) if a.dtype.kind == "f" else a == b), f
    for r in run_backend(engine, docs, routes=True):
        for rt in (r.routes or []) if r.ok else []:
            assert sum(rt["counts"]) == rt["tokens"] * top_k
