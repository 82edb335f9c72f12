"""Generate golden vectors by running the REFERENCE simulator in this container.

Usage (container only; /root/reference does not exist on the GPU box):

    python tests/golden/make_golden.py [--skip-c5]

Writes `tests/golden/*.json.gz`. Every fixture records the numpy version
it was generated under (routing and workload draws are numpy Philox
streams; numpy 2.3.5 here). Nothing in the test suite imports the reference:
the fixtures are the pin.

What is recorded per scenario (reference call sites in brackets):
  - requests as generated  [workload.py:204-220]
  - per request: first TOKEN_EMITTED ns, REQUEST_COMPLETE ns, completion rank
                                                  [metrics.py:93-116]
  - per BATCH_COMPLETE: replica, phase, request ids, duration_ns, timestamp,
    moe_imbalance                                  [base.py:233-255, af.py:489-503]
  - per router call (small MoE scenarios): scope, step, layer, T, counts
                                                  [base.py:128-147, af.py:289-301]
  - metrics.to_dict(), event count, trace sha256  [metrics.py:81-178, core.py:116-118]
  - or the exception type/message for failing scenarios
"""

from __future__ import annotations

import argparse
import copy
import gzip
import json
import os
import sys
import time

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))  # repo root
sys.path.insert(0, REF_SRC)

import numpy as np  # noqa: E402

from frontier_sim import cli as ref_cli  # noqa: E402
from frontier_sim.config import parse_config  # noqa: E402
from frontier_sim.core import EventKind  # noqa: E402
from frontier_sim.orchestrator import af as ref_af  # noqa: E402
from frontier_sim.orchestrator import base as ref_base  # noqa: E402

from paper_2508_03148_b200 import workloads as W  # noqa: E402


# -- scenario documents -------------------------------------------------------

def _tight_hw(hbm):
    hw = dict(W.B200_HW)
    hw["hbm_capacity_bytes"] = hbm
    return hw


def _pool_hw(model_doc, gpus, pool_tokens, role="colocated", attn_dp=1):
    """Back-solve per-GPU HBM for a KV pool of ~pool_tokens [topology.py:289-302]."""
    from frontier_sim.config import _parse_model, _Node
    from frontier_sim.topology import kv_bytes_per_token, weight_bytes_total
    model = _parse_model(_Node(copy.deepcopy(model_doc), "m"))
    weights = weight_bytes_total(model) * (attn_dp if role == "attention" else 1)
    need = pool_tokens * kv_bytes_per_token(model) + weights
    return _tight_hw((need / 0.9 + 4096) / gpus)


TINY_MOE_MODEL = {"num_layers": 3, "d_model": 512, "d_ff": 2048, "num_query_heads": 8,
                  "num_kv_heads": 2, "head_dim": 64,
                  "moe": {"num_experts": 16, "top_k": 3, "expert_d_ff": 1024, "gated": True}}
SMALL_DENSE = {"num_layers": 4, "d_model": 1024, "d_ff": 4096, "num_query_heads": 8,
               "num_kv_heads": 4, "head_dim": 128}


def scenarios() -> dict[str, dict]:
    s: dict[str, dict] = {}
    s["co_llama_40"] = W.c1_colocated(40, seed=3)

    d = W.c1_colocated(30, seed=4)
    d["clusters"][0].update(gpus_per_replica=4, parallelism={"tp": 2, "pp": 2})
    s["co_tp2_pp2"] = d

    # Small pool (weights 13.0e9 of 7B shape; pool ~ 3000 tokens): HOL blocking, paged.
    d = W.c1_colocated(40, seed=5)
    d["clusters"][0].update(num_replicas=2, hardware=_pool_hw(W.LLAMA2_7B, 1, 7000))
    d["policies"] = {"admission": "fcfs_skip", "memory_mode": "paged", "block_tokens": 16,
                     "max_num_seqs": 8, "max_batch_tokens": 4096}
    s["co_2rep_paged_skip"] = d

    d = W.c1_colocated(40, seed=6)
    d["clusters"][0].update(hardware=_pool_hw(W.LLAMA2_7B, 1, 9000))
    d["policies"] = {"admission": "priority", "priority_key": "prompt_tokens", "max_num_seqs": 6}
    s["co_priority_prompt"] = d

    d = W.c1_colocated(40, seed=7)
    d["clusters"][0].update(num_replicas=3, hardware=_pool_hw(W.LLAMA2_7B, 1, 8000))
    d["policies"] = {"admission": "priority", "priority_key": "arrival_time",
                     "memory_mode": "paged", "block_tokens": 64}
    d["workload"]["arrival"] = {"kind": "batch_at_zero"}
    s["co_priority_arrival_batch0"] = d

    d = W.c1_colocated(24, seed=8)
    d["workload"]["arrival"] = {"kind": "fixed_interval", "gap_ns": 2_000_000}
    d["workload"]["prompt_tokens"] = {"kind": "uniform", "lo": 1, "hi": 300}
    d["workload"]["output_tokens"] = {"kind": "fixed", "value": 7}
    s["co_fixed_interval_uniform"] = d

    d = copy.deepcopy(W.c5_sweep_configs(12)[48 + 5])  # ep=2, mns=64
    d["seed"] = 9
    s["co_moe_mixtral_ep2"] = d

    d = {"mode": "colocated", "seed": 10, "model": copy.deepcopy(TINY_MOE_MODEL),
         "clusters": [{"id": "c0", "role": "colocated", "gpus_per_replica": 4,
                       "hardware": dict(W.B200_HW), "parallelism": {"tp": 1, "ep": 4}},
                      ],
         "network": copy.deepcopy(W.NETWORK), "routing": {"policy": "uniform"},
         "workload": W.poisson_workload(16, 40.0, prompt_mu=4.0, output_mu=2.5)}
    s["co_tiny_moe_gated_ep4"] = d

    d = W.c3_pd(40, seed=11, tight=True)
    s["pd_70b_tight_40"] = d

    d = W.c5_sweep_configs(40)[16 + 5]   # PD tp=2, mns=64, P:D=2:3
    d = copy.deepcopy(d)
    d["seed"] = 12
    d["policies"].update(memory_mode="paged", block_tokens=32)
    d["clusters"][1]["hardware"] = _pool_hw(W.LLAMA2_7B, 2, 6000)
    s["pd_2_3_paged_tight"] = d

    d = {"mode": "pd", "seed": 13, "model": copy.deepcopy(W.MIXTRAL_8X7B),
         "clusters": [
             {"id": "pre", "role": "prefill", "num_replicas": 2, "gpus_per_replica": 2,
              "hardware": dict(W.B200_HW), "parallelism": {"ep": 2}},
             {"id": "dec", "role": "decode", "num_replicas": 1, "gpus_per_replica": 4,
              "hardware": dict(W.B200_HW), "parallelism": {"ep": 4}}],
         "network": copy.deepcopy(W.NETWORK), "routing": {"policy": "uniform"},
         "workload": W.poisson_workload(12, 20.0)}
    s["pd_moe_mixtral"] = d

    d = W.c4_af(10, seed=1)
    s["af_dsv3_m2_10"] = d

    d = {"mode": "af", "seed": 14, "model": copy.deepcopy(TINY_MOE_MODEL),
         "clusters": [
             {"id": "A", "role": "attention", "gpus_per_replica": 4, "hardware": dict(W.B200_HW),
              "parallelism": {"attn_tp": 2, "attn_dp": 2, "moe_tp": 2, "moe_ep": 2}},
             {"id": "F", "role": "ffn", "gpus_per_replica": 4, "hardware": dict(W.B200_HW),
              "parallelism": {"attn_tp": 2, "attn_dp": 2, "moe_tp": 2, "moe_ep": 2}}],
         "network": copy.deepcopy(W.NETWORK), "af": {"micro_batches": 3},
         "routing": {"policy": "uniform"},
         "workload": W.poisson_workload(14, 30.0, prompt_mu=4.5, output_mu=2.5)}
    s["af_tiny_moe_m3_dp2"] = d

    d = {"mode": "af", "seed": 15, "model": copy.deepcopy(SMALL_DENSE),
         "clusters": [
             {"id": "attn", "role": "attention", "gpus_per_replica": 2, "hardware": dict(W.B200_HW),
              "parallelism": {"attn_tp": 2, "attn_dp": 1, "moe_tp": 2, "moe_ep": 1}},
             {"id": "ffn", "role": "ffn", "gpus_per_replica": 2, "hardware": dict(W.B200_HW),
              "parallelism": {"attn_tp": 2, "attn_dp": 1, "moe_tp": 2, "moe_ep": 1}}],
         "network": copy.deepcopy(W.NETWORK), "af": {"micro_batches": 4},
         "workload": W.poisson_workload(20, 30.0, prompt_mu=5.0, output_mu=3.0)}
    s["af_dense_m4"] = d

    # -- failure scenarios ------------------------------------------------------
    d = W.c1_colocated(8, seed=16)
    d["clusters"][0]["hardware"] = _pool_hw(W.LLAMA2_7B, 1, 900)
    s["err_colocated_cannot_fit"] = d

    d = copy.deepcopy(s["co_tiny_moe_gated_ep4"])
    d["routing"] = {"policy": "trace", "trace_counts": [1] * 16}
    s["err_trace_routing_sum"] = d

    d = W.c3_pd(10, seed=17, tight=True)
    d["clusters"][0]["hardware"] = _pool_hw(W.DENSE_70B, 4, 1200)
    s["err_pd_prefill_cannot_fit"] = d
    return s


def baseline_scenarios() -> dict[str, dict]:
    return {
        "C1_colocated_llama7b_1000": W.c1_colocated(1000, seed=1),
        "C3_pd_70b_tight_300": W.c3_pd(300, seed=1, tight=True),
        "C3_pd_70b_roomy_300": W.c3_pd(300, seed=1, tight=False),
        "C4_af_dsv3_10": W.c4_af(10, seed=1),
        "C4_colocated_ep8_10": W.c4_colocated_ep(10, seed=1),
    }


# -- recording ----------------------------------------------------------------

class RouterRecorder:
    """Wraps derive_router_seed / route_tokens in the orchestrator modules."""

    def __init__(self) -> None:
        self.calls: list[list] = []
        self._pending: list | None = None
        self._orig_seed = ref_base.derive_router_seed
        self._orig_route_base = ref_base.route_tokens
        self._orig_route_af = ref_af.route_tokens

    def __enter__(self):
        rec = self

        def seed_fn(master, scope, step, layer):
            rec._pending = [scope, step, layer]
            return rec._orig_seed(master, scope, step, layer)

        def route_fn(orig):
            def wrapped(total_tokens, num_experts, top_k, *args, **kwargs):
                a = orig(total_tokens, num_experts, top_k, *args, **kwargs)
                scope, step, layer = rec._pending if rec._pending else (None, None, None)
                rec.calls.append([scope, step, layer, total_tokens, list(a.counts)])
                rec._pending = None
                return a
            return wrapped

        ref_base.derive_router_seed = seed_fn
        ref_af.derive_router_seed = seed_fn
        ref_base.route_tokens = route_fn(self._orig_route_base)
        ref_af.route_tokens = route_fn(self._orig_route_af)
        return self

    def __exit__(self, *exc):
        ref_base.derive_router_seed = self._orig_seed
        ref_af.derive_router_seed = self._orig_seed
        ref_base.route_tokens = self._orig_route_base
        ref_af.route_tokens = self._orig_route_af
        return False


def record(doc: dict, with_batches: bool = True, with_routes: bool = False, base_dir: str = ".") -> dict:
    out: dict = {"config": doc}
    config = parse_config(copy.deepcopy(doc), base_dir=base_dir)
    reqs = config.requests()
    out["requests"] = {
        "ids": [r.id for r in reqs],
        "arrival_ns": [r.arrival_time for r in reqs],
        "prompt": [r.prompt_tokens for r in reqs],
        "output": [r.output_tokens for r in reqs],
    }
    out["config_hash"] = config.config_hash()
    t0 = time.perf_counter()
    try:
        if with_routes:
            with RouterRecorder() as rr:
                result = ref_cli.run_one(config)
            out["routes"] = rr.calls
        else:
            result = ref_cli.run_one(config)
    except Exception as exc:  # failure scenarios record the exception
        out["error"] = {"type": type(exc).__name__, "message": str(exc)}
        out["wall_s"] = time.perf_counter() - t0
        return out
    out["wall_s"] = time.perf_counter() - t0
    trace = result["trace"]
    first: dict[str, int] = {}
    done: dict[str, int] = {}
    order: list[str] = []
    batches = []
    for ev in trace:
        p = ev.payload
        if ev.kind is EventKind.TOKEN_EMITTED:
            for rid in p["request_ids"]:
                first.setdefault(rid, ev.timestamp)
        elif ev.kind is EventKind.REQUEST_COMPLETE:
            done[p["request_id"]] = ev.timestamp
            order.append(p["request_id"])
        elif ev.kind is EventKind.BATCH_COMPLETE:
            batches.append([p["replica"], p["phase"], ev.timestamp, p["duration_ns"],
                            p["request_ids"], p.get("moe_imbalance")])
    ids = out["requests"]["ids"]
    out["first_token_ns"] = [first[i] for i in ids]
    out["done_ns"] = [done[i] for i in ids]
    out["completion_order"] = order
    out["iterations"] = len(batches)
    if with_batches:
        out["batches"] = batches
    out["events"] = len(trace)
    out["trace_hash"] = trace.hash
    out["metrics"] = result["metrics"].to_dict()
    return out


def pure_function_vectors() -> dict:
    """Golden vectors for the pure functions on the path."""
    from frontier_sim.costmodel import analytic
    from frontier_sim.costmodel.features import AttentionFeatures, GroupedGemmFeatures
    from frontier_sim.costmodel.model import CostModel
    from frontier_sim.costmodel.moe import MoeExecutionTopology, moe_layer_latency
    from frontier_sim.costmodel.routing import route_tokens
    from frontier_sim.orchestrator.base import derive_router_seed
    from frontier_sim.topology import (HardwareSpec, LinkSpec, ModelConfig, MoeConfig,
                                       collective_time, transfer_time)

    rng = np.random.default_rng(2508)
    vec: dict = {}

    # Router seeds [base.py:63-65]
    seeds = []
    for master in (0, 1, 7, 1000, 4294967295, 4294967296, 2**40 + 3):
        for scope in ("c0/0", "d0/12", "attn/0:mb1", "a-much-longer-cluster-identifier-x/3:mb2",
                      "x" * 70 + "/1"):
            for step in (0, 1, 9, 10, 12345):
                for layer in (0, 5, 60):
                    seeds.append([master, scope, step, layer,
                                  derive_router_seed(master, scope, step, layer)])
    vec["router_seed"] = seeds

    # SeedSequence-derived Philox keys [routing.py:59-62]
    keys = []
    for s in [0, 1, 2, 7, 224, 123456789, 2**32 - 1, 2**32, 2**33 + 5, 2**63 + 11, 2**64 - 1]:
        ss_state = np.random.SeedSequence([s, 0xE0]).generate_state(2, np.uint64)
        bitgen = np.random.Philox(ss_state)
        k = bitgen.state["state"]["key"]
        keys.append([s, [int(x) for x in ss_state], [int(x) for x in k]])
    vec["philox_keys"] = keys

    # route_tokens counts [routing.py:65-113]
    routes = []
    cases = [(1, 8, 2), (5, 8, 2), (17, 8, 2), (64, 8, 2), (300, 8, 2), (3, 256, 8),
             (40, 256, 8), (1000, 16, 3), (7, 16, 1), (33, 16, 15), (10, 4, 4), (0, 8, 2),
             (2048, 8, 2), (5, 1, 1), (9, 60, 6)]
    for T, E, k in cases:
        for seed in (0, 1, 3735928559, int(rng.integers(0, 2**32))):
            a = route_tokens(T, E, k, policy="uniform", seed=seed)
            routes.append([T, E, k, seed, list(a.counts)])
    vec["route_uniform"] = routes

    # Analytic attention on skewed batches [analytic.py:32-53]; features [features.py:101-115]
    hw = HardwareSpec(peak_flops=2.25e15, mem_bw=8e12, hbm_capacity_bytes=180e9)
    attn = []
    for b in range(64):
        n = int(rng.integers(1, 200)) if b % 8 else 72
        kv = np.clip(np.rint(rng.lognormal(6.5, 1.4, size=n)), 16, 32768).astype(int)
        phase = "decode" if b % 2 == 0 else "prefill"
        q = [1] * n if phase == "decode" else [int(x) for x in kv]
        if phase == "prefill" and b % 4 == 1:  # prefill with prior context c > l
            q = [max(1, int(x) // 3) for x in kv]
        hq, hkv, hd = [(32, 8, 128), (8, 1, 64), (64, 8, 128), (3, 3, 80)][b % 4]
        f = AttentionFeatures(phase, tuple(q), tuple(int(x) for x in kv), hq, hkv, hd)
        us = analytic.attention_us(f, hw, 2)
        attn.append([phase, q, [int(x) for x in kv], hq, hkv, hd, us,
                     [float(x) for x in f.vector()]])
    vec["attention"] = attn

    # linear / grouped GEMM / collectives / transfers [analytic.py:23-71, topology.py:360-394]
    lin = []
    for _ in range(200):
        m, n, k = (int(x) for x in rng.integers(1, 20000, size=3))
        lin.append([m, n, k, analytic.linear_us(m, n, k, hw, 2)])
    vec["linear"] = lin
    gg = []
    for _ in range(200):
        E = int(rng.integers(1, 40))
        counts = [int(x) if rng.random() > 0.3 else 0 for x in rng.integers(0, 500, size=E)]
        if sum(counts) == 0:
            counts[0] = 1
        d, dff, nm = int(rng.integers(64, 8192)), int(rng.integers(64, 30000)), int(rng.integers(2, 4))
        f = GroupedGemmFeatures(sum(counts), tuple(counts), d, dff, 1, mode="local")
        gg.append([counts, d, dff, nm, analytic.grouped_gemm_us(f, hw, 2, nm)])
    vec["grouped_gemm"] = gg
    coll = []
    link = LinkSpec(latency_s=5e-6, bandwidth_bps=900e9)
    for kind in ("all_to_all", "all_reduce", "all_gather"):
        for n in (1, 2, 3, 4, 8, 16):
            for b in (0, 1, 12345, 7.5e6, 3 * 2**30, 1.0 / 3.0):
                coll.append([kind, b, n, collective_time(kind, b, n, link)])
    vec["collective"] = coll
    vec["transfer"] = [[b, transfer_time(b, LinkSpec(20e-6, 50e9))]
                       for b in (0, 1, 327680, 327680 * 4000, 1748992 * 77)]

    # moe_layer_latency breakdowns over real uniform routing [moe.py:69-128]
    moe = []
    for (E, k, ep, mtp, gated, T) in [(8, 2, 1, 1, False, 12), (8, 2, 2, 1, False, 300),
                                      (256, 8, 8, 1, False, 5), (256, 8, 8, 1, False, 64),
                                      (16, 3, 4, 2, True, 9), (64, 6, 16, 1, False, 3)]:
        model = ModelConfig(num_layers=2, d_model=4096, d_ff=14336, num_query_heads=32,
                            num_kv_heads=8, head_dim=128,
                            moe=MoeConfig(E, k, 14336 if E == 8 else 2048, gated))
        cm = CostModel(hardware=hw, dtype_bytes=2, ffn_matrices=model.ffn_matrices)
        topo = MoeExecutionTopology(ep_ranks=ep, moe_tp=mtp, link=link)
        for seed in (1, 99):
            a = route_tokens(T, E, k, seed=seed)
            total, br = moe_layer_latency(a, model, topo, cm)
            moe.append([E, k, ep, mtp, gated, T, seed, list(a.counts), total, br.to_dict()])
    vec["moe_layer"] = moe

    # Python sum() (Neumaier in CPython 3.12) over float lists, as used at
    # cluster.py:345 and metrics.py:36
    sums = []
    for _ in range(300):
        n = int(rng.integers(1, 100))
        xs = [float(x) for x in rng.lognormal(0, 4, size=n) * rng.choice([-1.0, 1.0], size=n)]
        sums.append([xs, sum(xs)])
    for x in (0.1, 1.7e-3, 123.456789, 3.3333333333333335e4):
        for L in (1, 2, 3, 32, 61, 80, 127):
            sums.append([[x] * L, sum([x] * L)])
    vec["py_sum"] = sums
    return vec


def _save_model(name: str, model) -> str:
    """Write `model` as tests/golden/{name}.json.gz and a plain copy under /tmp."""
    path = os.path.join(HERE, f"{name}.json.gz")
    with gzip.open(path, "wt", encoding="utf-8") as fh:
        json.dump(model.to_document(), fh, sort_keys=True, separators=(",", ":"))
        fh.write("\n")
    raw = os.path.join("/tmp", f"{name}.json")
    with gzip.open(path, "rt", encoding="utf-8") as fh, open(raw, "w", encoding="utf-8") as g:
        g.write(fh.read())
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")
    return raw


def forest_fixtures() -> dict:
    """Learned operator models in the reference's model-file format
    (model.py:140-182) plus reference predictions on C2-style batches."""
    from frontier_sim.costmodel.features import AttentionFeatures
    from frontier_sim.costmodel.forest import ForestHyperparams
    from frontier_sim.costmodel.model import fit_model, load_model_file
    from frontier_sim.costmodel.synthetic import (make_attention_suite, make_grouped_gemm_suite,
                                                  sqrt_proxy_dataset)

    out = {}
    specs = {"forest_c2": (5000, None),                       # C2: 100 trees, depth 12
             "forest_small": (1000, ForestHyperparams(n_trees=12, max_depth=8))}
    for name, (n, hp) in specs.items():
        suite, feats = make_attention_suite(n, seed=11, noise=0.03)
        model, _ = fit_model(suite, hp, seed=7)
        loaded = load_model_file(_save_model(name, model))
        rng = np.random.default_rng(404)
        preds = []
        for b in range(512):
            nreq = 72 if b % 5 else int(rng.integers(1, 300))
            kv = np.clip(np.rint(rng.lognormal(6.5, 1.4, size=nreq)), 16, 32768).astype(int)
            phase = "decode" if b % 2 == 0 else "prefill"
            q = [1] * nreq if phase == "decode" else [int(x) for x in kv]
            f = AttentionFeatures(phase, tuple(q), tuple(int(x) for x in kv), 32, 8, 128)
            preds.append([phase, q, [int(x) for x in kv], loaded.predict_us(f.vector())])
        out[name] = preds
        if name == "forest_small":
            # an attention-operator model on the wrong schema (SchemaMismatch at predict)
            proxy, _ = fit_model(sqrt_proxy_dataset(suite, feats),
                                 ForestHyperparams(n_trees=4, max_depth=4), seed=7)
            _save_model("forest_sqrt_proxy", proxy)
    # grouped-GEMM model (dense FFNs call it with one local expert, cluster.py:286-296)
    suite, _ = make_grouped_gemm_suite(1500, seed=12, noise=0.02)
    gg, _ = fit_model(suite, ForestHyperparams(n_trees=16, max_depth=10), seed=5)
    _save_model("forest_gg_small", gg)
    return out


def learned_scenarios() -> dict[str, dict]:
    """Scenarios whose operator costs come from the small learned forests."""
    att = {"mode": "learned", "attention_model": "forest_small.json"}
    gg = {"mode": "learned", "grouped_gemm_model": "forest_gg_small.json"}
    both = {"mode": "learned", "attention_model": "forest_small.json",
            "grouped_gemm_model": "forest_gg_small.json"}
    s = {}
    d = W.c1_colocated(40, seed=21)
    d["cost_model"] = dict(att)
    s["learned_co_llama_40"] = d
    d = W.c3_pd(30, seed=22, tight=True)
    d["cost_model"] = dict(att)
    s["learned_pd_70b_tight_30"] = d
    d = copy.deepcopy(scenarios()["af_tiny_moe_m3_dp2"])
    d["seed"] = 23
    d["cost_model"] = dict(att)
    s["learned_af_tiny_moe"] = d
    d = W.c1_colocated(40, seed=24)
    d["cost_model"] = dict(gg)
    s["learned_gg_co_llama_40"] = d
    d = W.c3_pd(30, seed=25, tight=False)
    d["cost_model"] = dict(both)
    s["learned_both_pd_70b_30"] = d
    d = W.c1_colocated(12, seed=26)
    d["cost_model"] = {"mode": "learned", "attention_model": "forest_sqrt_proxy.json"}
    s["learned_err_attention_schema"] = d
    d = W.c1_colocated(12, seed=27)
    d["cost_model"] = {"mode": "learned", "attention_model": "forest_gg_small.json"}
    s["learned_err_operator_slot"] = d
    d = W.c1_colocated(12, seed=28)
    d["cost_model"] = {"mode": "analytic", "grouped_gemm_model": "forest_gg_small.json"}
    s["learned_gg_mode_analytic_still_loads"] = d
    return s


def learned_moe_fixtures() -> dict:
    """Learned grouped-GEMM model on MoE layers (moe.py:95-106 -> model.py:323-327):
    GroupedGemmFeatures(mode="local").vector() bits and predictions for per-rank
    expert loads, plus whole MoE simulations costed with the model."""
    from frontier_sim.costmodel.features import GroupedGemmFeatures
    from frontier_sim.costmodel.model import load_model_file

    gg_path = os.path.join("/tmp", "forest_gg_small.json")
    with gzip.open(os.path.join(HERE, "forest_gg_small.json.gz"), "rt") as fh, \
            open(gg_path, "w") as g:
        g.write(fh.read())
    model = load_model_file(gg_path)
    rng = np.random.default_rng(77)
    vecs = []
    for i in range(400):
        per = int(rng.choice([1, 2, 4, 7, 8, 16, 32, 33, 64, 128, 256]))
        k = int(rng.integers(1, 9))
        if i % 7 == 0:
            counts = [0] * per
            counts[int(rng.integers(0, per))] = int(rng.integers(1, 5000))
        else:
            lam = float(rng.choice([0.3, 2.0, 40.0, 900.0]))
            counts = [int(x) for x in rng.poisson(lam, size=per)]
        if sum(counts) == 0:
            counts[0] = 1
        dm = int(rng.choice([1024, 4096, 7168])); dff = int(rng.choice([256, 2048, 14336]))
        f = GroupedGemmFeatures(total_tokens=sum(counts), expert_token_counts=tuple(counts),
                                d_model=dm, d_ff=dff, top_k=k, mode="local")
        v = f.vector()
        vecs.append([counts, dm, dff, k, [int(x) for x in v.view(np.uint64)],
                     model.predict_us(v)])
    sims = {}
    gg = {"mode": "learned", "grouped_gemm_model": "forest_gg_small.json"}
    both = {"mode": "learned", "attention_model": "forest_small.json",
            "grouped_gemm_model": "forest_gg_small.json"}
    d = copy.deepcopy(W.c5_sweep_configs(24)[48 + 5])  # Mixtral ep=2
    d["seed"] = 31
    d["cost_model"] = dict(gg)
    sims["learned_gg_mixtral_ep2"] = d
    d = copy.deepcopy(scenarios()["af_tiny_moe_m3_dp2"])
    d["seed"] = 32
    d["cost_model"] = dict(both)
    sims["learned_both_af_tiny_moe"] = d
    d = W.c4_colocated_ep(6, seed=33)
    d["cost_model"] = dict(gg)
    sims["learned_gg_dsv3_ep8"] = d
    d = copy.deepcopy(scenarios()["co_tiny_moe_gated_ep4"])
    d["seed"] = 34
    d["cost_model"] = dict(gg)
    sims["learned_gg_tiny_moe_gated"] = d
    out = {"gg_vectors": vecs,
           "scenarios": {n: record(doc, with_batches=True, with_routes=True, base_dir="/tmp")
                         for n, doc in sims.items()}}
    for name, r in out["scenarios"].items():
        print(name, r.get("iterations"), r.get("error"), f"{r['wall_s']:.2f}s")
    return out


def dirichlet_fixtures() -> dict:
    """dirichlet_skew routing (routing.py:99-106): route_tokens counts from the
    reference, the raw stream (popularity + first key row) from the reference's
    own _rng, and whole simulations that route with the policy."""
    from frontier_sim.costmodel.routing import _rng, route_tokens

    out: dict = {}
    routes = []
    cases = [(1, 8, 2), (37, 8, 2), (300, 8, 2), (5, 256, 8), (40, 256, 8), (100, 64, 6),
             (20, 16, 3), (9, 60, 6), (3, 1024, 16), (64, 8, 7), (0, 8, 2), (12, 4, 4)]
    for T, E, k in cases:
        for alpha in (0.3, 0.05, 1.0, 2.5):
            for seed in (0, 1, 3735928559, 2**32 - 1):
                try:
                    c = list(route_tokens(T, E, k, "dirichlet_skew", seed, alpha).counts)
                except Exception as exc:  # pragma: no cover - none expected
                    c = f"{type(exc).__name__}: {exc}"
                routes.append([T, E, k, alpha, seed, c])
    out["route_dirichlet"] = routes
    streams = []
    for E in (8, 64, 256):
        for alpha in (0.3, 0.05, 2.5):
            for seed in (0, 7, 123456789):
                g = _rng(seed)
                pop = np.maximum(g.dirichlet(np.full(E, alpha)), 1e-12)
                keys = g.exponential(1.0, (2, E)) / pop
                streams.append([E, alpha, seed, [int(x) for x in pop.view(np.uint64)],
                                [int(x) for x in keys[0].view(np.uint64)]])
    out["dirichlet_stream"] = streams
    sims = {}
    d = copy.deepcopy(W.c5_sweep_configs(24)[48 + 5])  # Mixtral ep=2
    d["seed"] = 21
    d["routing"] = {"policy": "dirichlet_skew", "alpha": 0.3}
    sims["co_mixtral_dirichlet"] = d
    d = copy.deepcopy(W.c5_sweep_configs(16)[48 + 2])
    d["seed"] = 22
    d["routing"] = {"policy": "dirichlet_skew", "alpha": 0.05}
    sims["co_mixtral_dirichlet_small_alpha"] = d
    d = W.c4_colocated_ep(6, seed=23)
    d["routing"] = {"policy": "dirichlet_skew", "alpha": 0.3}
    sims["co_dsv3_ep8_dirichlet"] = d
    d = W.c4_af(6, seed=24)
    d["routing"] = {"policy": "dirichlet_skew", "alpha": 2.0}
    sims["af_dsv3_dirichlet"] = d
    out["scenarios"] = {name: record(doc, with_batches=True, with_routes=True)
                        for name, doc in sims.items()}
    for name, r in out["scenarios"].items():
        print(name, r.get("iterations"), r.get("error"), f"{r['wall_s']:.2f}s")
    return out


def capacity_scenarios() -> dict[str, dict]:
    """Past the round-1 engine limits: > 64 replicas per instance (PD with many
    prefill and decode replicas, co-located MoE), and cluster ids long enough that
    the router-seed prefix "{seed}:{id}/{i}:mb" exceeds 192 bytes."""
    from paper_2508_03148_b200 import workloads as W
    out = {}
    d = W.c3_pd(160, seed=3, tight=True)
    d["clusters"][0]["num_replicas"] = 40
    d["clusters"][1]["num_replicas"] = 60
    d["workload"]["arrival"]["rate_rps"] = 200.0
    out["pd_40x60_replicas"] = d
    d = W.c5_sweep_configs(8)[48 + 5]  # Mixtral co-located EP, 8 requests per seed
    d = copy.deepcopy(d)
    d["clusters"][0]["num_replicas"] = 80
    d["workload"]["num_requests"] = 120
    d["workload"]["arrival"]["rate_rps"] = 400.0
    d["seed"] = 11
    out["moe_colocated_80_replicas"] = d
    d = W.c3_pd(40, seed=5, tight=False)
    d["clusters"][0]["id"] = "prefill-" + "p" * 230
    d["clusters"][1]["id"] = "decode-" + "d" * 300
    d["clusters"][1]["num_replicas"] = 3
    out["pd_long_cluster_ids"] = d
    d = W.c4_af(12, seed=9)
    d["clusters"][0]["id"] = "attention-" + "a" * 260
    out["af_long_cluster_id"] = d
    return out


def largek_fixtures() -> dict:
    """top_k above the round-1 engine bound of 16: route_tokens counts (uniform and
    dirichlet_skew) and two whole simulations of a 64-expert model with top_k 20 / 24."""
    from frontier_sim.costmodel.routing import route_tokens
    calls = []
    for (T, E, k) in [(3, 32, 17), (40, 64, 20), (7, 64, 40), (5, 256, 100), (2, 256, 255),
                      (9, 1024, 300)]:
        for seed in (0, 5, 3735928559):
            for policy, alpha in (("uniform", 0.3), ("dirichlet_skew", 0.3), ("dirichlet_skew", 2.0)):
                a = route_tokens(T, E, k, policy=policy, seed=seed, alpha=alpha)
                calls.append([T, E, k, seed, policy, alpha, list(a.counts)])
    sims = {}
    base = W.c5_sweep_configs(12)[48 + 1]
    for name, k, routing in (("moe64_k20_uniform", 20, None),
                             ("moe64_k24_dirichlet", 24, {"policy": "dirichlet_skew", "alpha": 0.5})):
        d = copy.deepcopy(base)
        d["model"]["moe"] = {"num_experts": 64, "top_k": k, "expert_d_ff": 2048}
        d["model"]["num_layers"] = 6
        d["seed"] = 21
        if routing:
            d["routing"] = routing
        sims[name] = record(d, with_batches=True, with_routes=True)
        print(name, sims[name].get("iterations"), sims[name].get("error"))
    return {"route_calls": calls, "scenarios": sims}


def write(name: str, payload) -> None:
    payload = {"numpy": np.__version__, "python": sys.version.split()[0], "data": payload}
    path = os.path.join(HERE, f"{name}.json.gz")
    with gzip.open(path, "wt", encoding="utf-8") as fh:
        json.dump(payload, fh, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-c5", action="store_true")
    ap.add_argument("--skip-baseline", action="store_true")
    ap.add_argument("--only", default=None, help="comma-separated fixture names")
    args = ap.parse_args()
    only = set(args.only.split(",")) if args.only else None

    if only is None or "pure" in only:
        write("pure", pure_function_vectors())
    if only is None or "scenarios" in only:
        sc = {}
        for name, doc in scenarios().items():
            moe = "moe" in doc["model"]
            sc[name] = record(doc, with_batches=True, with_routes=moe)
            print(name, sc[name].get("iterations"), sc[name].get("error"),
                  f"{sc[name]['wall_s']:.2f}s")
        write("scenarios", sc)
    if only is not None and "largek" in only:
        write("largek", largek_fixtures())
    if only is not None and "capacity" in only:
        cap = {}
        for name, doc in capacity_scenarios().items():
            moe = "moe" in doc["model"]
            cap[name] = record(doc, with_batches=True, with_routes=moe and name.startswith("af"))
            print(name, cap[name].get("iterations"), cap[name].get("error"),
                  f"{cap[name]['wall_s']:.2f}s")
        write("capacity", cap)
    if only is None or "learned_moe" in only:
        write("learned_moe", learned_moe_fixtures())
    if only is None or "dirichlet" in only:
        write("dirichlet", dirichlet_fixtures())
    if only is None or "forest" in only:
        write("forest_predictions", forest_fixtures())
        sc = {}
        for name, doc in learned_scenarios().items():
            sc[name] = record(doc, with_batches=True, with_routes="moe" in doc["model"],
                              base_dir="/tmp")
            print(name, sc[name].get("iterations"), sc[name].get("error"))
        write("learned_scenarios", sc)
    if not args.skip_baseline and (only is None or "baseline" in only):
        bl = {}
        for name, doc in baseline_scenarios().items():
            bl[name] = record(doc, with_batches=name.startswith("C4"),
                              with_routes=name.startswith("C4"))
            print(name, bl[name].get("iterations"), f"{bl[name]['wall_s']:.2f}s")
        write("baseline", bl)
    if not args.skip_c5 and (only is None or "c5" in only):
        rows = {}
        base = W.c5_sweep_configs(64)
        t0 = time.perf_counter()
        for ci, doc in enumerate(base):
            d = copy.deepcopy(doc)
            d["seed"] = 1000 + 64 * ci  # s = 0 of the C5 seed grid
            r = record(d, with_batches=False)
            r.pop("config")
            r["metrics"].pop("per_request")
            rows[str(ci)] = r
            print("c5", ci, r.get("iterations"), f"{r['wall_s']:.1f}s",
                  f"total {time.perf_counter() - t0:.0f}s", flush=True)
        write("c5_seed0", rows)


if __name__ == "__main__":
    main()
