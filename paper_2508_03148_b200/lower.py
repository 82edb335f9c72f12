"""Lowering: simulation instances -> packed descriptors for the device engine.

One `InstanceSpec` is what the reference builds inside `make_simulation`
(orchestrator/base.py:71-111 and the mode subclasses): a validated
deployment, the request list, the scheduler policy, AF and routing settings
and the master seed. `lower` packs a list of them into the flat arrays of
the C ABI (include/frontier_b200.h): one instance descriptor each, a replica
table, a router-seed prefix table, the trace-count table and the request
struct-of-arrays. Everything here is host-side bookkeeping done once per
instance; no simulation arithmetic happens on the host.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import abi
from .cluster import SchedulerPolicy
from .costmodel import ForestSet, forest_slot
from .errors import EngineCapacityError, SimulationError
from .specs import AfPipelineConfig, RoutingPolicySpec
from .topology import ClusterSpec, Deployment, kv_bytes_per_token
from .workload import RequestArrays


@dataclass
class InstanceSpec:
    deployment: Deployment
    requests: RequestArrays
    policy: SchedulerPolicy
    af: AfPipelineConfig | None = None
    routing: RoutingPolicySpec = field(default_factory=RoutingPolicySpec)
    seed: int = 0
    attention_model: object = None      # costmodel.LearnedModel | None
    grouped_gemm_model: object = None   # costmodel.LearnedModel | None
    max_events: int = abi.DEFAULT_MAX_EVENTS
    tag: object = None


    @property
    def learned(self) -> bool:
        return self.attention_model is not None or self.grouped_gemm_model is not None


@dataclass
class ReplicaInfo:
    key: str
    role: str
    cluster: ClusterSpec


def replica_layout(dep: Deployment) -> list[ReplicaInfo]:
    """Replica order of the reference's constructors (colocated.py:24-28,
    pd.py:26-33, af.py:382-400)."""
    if dep.mode == "colocated":
        roles = ("colocated",)
    elif dep.mode == "pd":
        roles = ("prefill", "decode")
    else:
        roles = ("attention",)
    out = []
    for role in roles:
        for c in dep.clusters_with_role(role):
            for i in range(c.num_replicas):
                out.append(ReplicaInfo(f"{c.id}/{i}", role, c))
    return out


def _cost(hw, tp, ep, moe_tp, pp) -> tuple:
    return (float(hw.peak_flops), float(hw.mem_bw), float(hw.kernel_overhead_us),
            int(tp), int(ep), int(moe_tp), int(pp))


def _prefix(text: str) -> np.void:
    b = text.encode("utf-8")
    if len(b) > abi.MAX_PREFIX_BYTES:
        raise EngineCapacityError(
            f"router-seed prefix of {len(b)} bytes exceeds {abi.MAX_PREFIX_BYTES}: {text[:40]}...")
    rec = np.zeros((), dtype=abi.SEED_PREFIX)
    rec["bytes"][: len(b)] = np.frombuffer(b, dtype=np.uint8)
    rec["len"] = len(b)
    rec["mid_blocks"] = len(b) // 64
    return rec


def _id_ranks(ids: list[str]) -> np.ndarray:
    """Rank of each id in Python str order ("r10" < "r2"), cluster.py:153-157."""
    order = sorted(range(len(ids)), key=ids.__getitem__)
    rank = np.empty(len(ids), dtype=np.int32)
    rank[order] = np.arange(len(ids), dtype=np.int32)
    return rank


def _estimate_cost(spec: InstanceSpec) -> int:
    m = spec.deployment.model
    out_tokens = int(spec.requests.output.sum()) + len(spec.requests)
    prompt_tokens = int(spec.requests.prompt.sum())
    moe = m.moe
    work = out_tokens * m.num_layers
    if moe is not None:
        work += (out_tokens + prompt_tokens) * m.num_layers * moe.num_experts // 4
    return int(work)


@dataclass
class Lowered:
    descs: np.ndarray
    replicas: np.ndarray
    prefixes: np.ndarray
    trace_counts: np.ndarray
    arrival: np.ndarray
    prompt: np.ndarray
    output: np.ndarray
    id_rank: np.ndarray
    replica_keys: list[list[str]]
    request_ids: list[list[str]]
    forests: object = None  # costmodel.ForestSet | None (learned operator models)

    @property
    def n_instances(self) -> int:
        return len(self.descs)

    @property
    def n_requests(self) -> int:
        return len(self.arrival)


def check_spec(sp: InstanceSpec) -> None:
    """The per-instance checks the reference makes inside make_simulation
    (base.py:71-111, af.py:381-392, cluster.py:108-118) plus the engine's
    capacity limits. simulate() runs this per point, so a bad point becomes a
    Failure row (cli.py:229-233) and lower() cannot raise for the others."""
    dep, model = sp.deployment, sp.deployment.model
    sp.policy.validate()
    if len(set(sp.requests.ids)) != len(sp.requests.ids):
        raise SimulationError("duplicate request id")
    layout = replica_layout(dep)
    if not layout:
        raise SimulationError(f"{dep.mode} deployment has no serving replicas")
    if len(layout) > abi.MAX_REPLICAS:
        raise EngineCapacityError(f"{len(layout)} replicas exceed {abi.MAX_REPLICAS}")
    if model.moe is not None and model.moe.num_experts > abi.MAX_EXPERTS:
        raise EngineCapacityError(f"{model.moe.num_experts} experts exceed {abi.MAX_EXPERTS}")
    for ri in layout:
        _prefix(f"{sp.seed}:{ri.key}:mb")  # router-seed prefix length
    if dep.mode == "af":
        (sp.af or AfPipelineConfig()).validate()
        attn = dep.clusters_with_role("attention")
        ffn = dep.clusters_with_role("ffn")
        if len(attn) != 1 or len(ffn) != 1:
            raise ValueError("af mode takes exactly one attention and one ffn cluster")
        if attn[0].num_replicas != 1 or ffn[0].num_replicas != 1:
            raise ValueError("af mode models a single pipeline: num_replicas must be 1")
    for m, schema in ((sp.attention_model, "attention_v1"),
                      (sp.grouped_gemm_model, "grouped_gemm_v1")):
        if m is not None and m.schema == schema and m.n_trees > abi.MAX_FOREST_TREES:
            raise EngineCapacityError(f"{m.path}: {m.n_trees} trees exceed {abi.MAX_FOREST_TREES}")


def lower(specs: list[InstanceSpec]) -> Lowered:
    n = len(specs)
    descs = np.zeros(n, dtype=abi.INSTANCE_DESC)
    reps: list[tuple] = []
    prefixes: list[np.void] = []
    trace: list[int] = []
    arr_parts, p_parts, o_parts, rank_parts = [], [], [], []
    replica_keys, request_ids = [], []
    req_off = 0
    forests = ForestSet()
    for i, sp in enumerate(specs):
        dep, model, pol = sp.deployment, sp.deployment.model, sp.policy
        check_spec(sp)
        layout = replica_layout(dep)
        d = descs[i]
        d["mode"] = abi.MODE[dep.mode]
        d["n_requests"] = len(sp.requests)
        d["req_offset"] = req_off
        d["n_replicas"] = len(layout)
        d["replica_offset"] = len(reps)
        for f in ("num_layers", "d_model", "d_ff", "num_query_heads", "num_kv_heads", "head_dim",
                  "dtype_bytes"):
            d[f] = getattr(model, f)
        d["ffn_matrices"] = model.ffn_matrices
        if model.moe is not None:
            d["has_moe"] = 1
            d["num_experts"] = model.moe.num_experts
            d["top_k"] = model.moe.top_k
            d["expert_d_ff"] = model.moe.expert_d_ff
            if model.moe.num_experts > abi.MAX_EXPERTS:
                raise EngineCapacityError(f"{model.moe.num_experts} experts exceed {abi.MAX_EXPERTS}")
        d["admission"] = abi.ADMISSION[pol.admission]
        d["priority_key"] = abi.PRIORITY_KEY[pol.priority_key]
        d["max_num_seqs"] = pol.max_num_seqs
        d["max_batch_tokens"] = pol.max_batch_tokens
        d["paged"] = 1 if pol.memory_mode == "paged" else 0
        d["block_tokens"] = pol.block_tokens
        rt = sp.routing
        d["routing_policy"] = abi.ROUTING[rt.policy]
        d["routing_alpha"] = rt.alpha
        d["trace_offset"] = len(trace)
        if rt.trace_counts:
            d["n_trace_counts"] = len(rt.trace_counts)
            trace.extend(int(c) for c in rt.trace_counts)
        net = dep.network
        d["intra_latency_s"] = net.intra_replica.latency_s
        d["intra_bandwidth_bps"] = net.intra_replica.bandwidth_bps
        d["inter_latency_s"] = net.inter_cluster.latency_s
        d["inter_bandwidth_bps"] = net.inter_cluster.bandwidth_bps
        d["kv_bytes_per_token"] = kv_bytes_per_token(model)
        d["max_events"] = sp.max_events
        d["total_gpus"] = dep.total_gpus
        for slot, model, schema in (("attn_forest", sp.attention_model, "attention_v1"),
                                    ("gg_forest", sp.grouped_gemm_model, "grouped_gemm_v1")):
            if model is not None and model.schema == schema and model.n_trees > abi.MAX_FOREST_TREES:
                raise EngineCapacityError(
                    f"{model.path}: {model.n_trees} trees exceed {abi.MAX_FOREST_TREES}")
            d[slot] = forest_slot(forests, model, schema)
        d["est_cost"] = _estimate_cost(sp)
        keys = [ri.key for ri in layout]
        key_rank = {k: r for r, k in enumerate(sorted(keys))}
        for ri in layout:
            c = ri.cluster
            p = c.parallelism
            pidx = len(prefixes)
            prefixes.append(_prefix(f"{sp.seed}:{ri.key}:"))
            pmb = -1
            if dep.mode == "af":
                cost = _cost(c.hardware, p.attn_tp, 1, 1, p.pp)
                pmb = len(prefixes)
                prefixes.append(_prefix(f"{sp.seed}:{ri.key}:mb"))
            else:
                cost = _cost(c.hardware, p.tp, p.ep, p.tp, p.pp)
            reps.append((abi.ROLE[ri.role], key_rank[ri.key], c.kv_pool_tokens, cost, pidx, pmb))
        if dep.mode == "af":
            af = sp.af or AfPipelineConfig()
            af.validate()
            attn = dep.clusters_with_role("attention")
            ffn = dep.clusters_with_role("ffn")
            if len(attn) != 1 or len(ffn) != 1:
                raise ValueError("af mode takes exactly one attention and one ffn cluster")
            if attn[0].num_replicas != 1 or ffn[0].num_replicas != 1:
                raise ValueError("af mode models a single pipeline: num_replicas must be 1")
            pa, pf = attn[0].parallelism, ffn[0].parallelism
            d["af_micro_batches"] = af.micro_batches
            d["af_attn_dp"] = pa.attn_dp
            d["af_attn"] = _cost(attn[0].hardware, pa.attn_tp, 1, 1, pa.pp)
            d["af_ffn"] = _cost(ffn[0].hardware, pf.moe_tp, pf.moe_ep, pf.moe_tp, pf.pp)
        r = sp.requests
        arr_parts.append(np.asarray(r.arrival_ns, dtype=np.int64))
        p_parts.append(np.asarray(r.prompt, dtype=np.int32))
        o_parts.append(np.asarray(r.output, dtype=np.int32))
        rank_parts.append(_id_ranks(r.ids))
        replica_keys.append(keys)
        request_ids.append(r.ids)
        req_off += len(r)
    replicas = np.array(reps, dtype=abi.REPLICA_DESC) if reps else np.zeros(0, abi.REPLICA_DESC)
    pref = np.array(prefixes, dtype=abi.SEED_PREFIX) if prefixes else np.zeros(0, abi.SEED_PREFIX)
    cat = lambda parts, dt: np.concatenate(parts).astype(dt) if parts else np.zeros(0, dt)  # noqa: E731
    return Lowered(
        descs=descs, replicas=replicas, prefixes=pref,
        trace_counts=np.asarray(trace if trace else [0], dtype=np.int64),
        arrival=cat(arr_parts, np.int64), prompt=cat(p_parts, np.int32),
        output=cat(o_parts, np.int32), id_rank=cat(rank_parts, np.int32),
        replica_keys=replica_keys, request_ids=request_ids,
        forests=forests if forests.models else None)
