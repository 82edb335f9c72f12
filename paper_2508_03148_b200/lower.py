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


_SHA256_K = (
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2)
_SHA256_IV = (0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
              0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19)


def sha256_midstate(data: bytes) -> tuple[int, ...]:
    """SHA-256 state after compressing the complete 64-byte blocks of `data` (FIPS
    180-4 compression function; hashlib does not expose midstates)."""
    m32 = 0xFFFFFFFF

    def rotr(x: int, n: int) -> int:
        return ((x >> n) | (x << (32 - n))) & m32

    h = list(_SHA256_IV)
    for b in range(len(data) // 64):
        w = list(int.from_bytes(data[64 * b + 4 * i: 64 * b + 4 * i + 4], "big") for i in range(16))
        for i in range(16, 64):
            s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3)
            s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10)
            w.append((w[i - 16] + s0 + w[i - 7] + s1) & m32)
        a, bb, c, d, e, f, g, hh = h
        for i in range(64):
            t1 = (hh + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g))
                  + _SHA256_K[i] + w[i]) & m32
            t2 = ((rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & bb) ^ (a & c) ^ (bb & c))) & m32
            hh, g, f, e, d, c, bb, a = g, f, e, (d + t1) & m32, c, bb, a, (t1 + t2) & m32
        h = [(x + y) & m32 for x, y in zip(h, (a, bb, c, d, e, f, g, hh))]
    return tuple(h)


def _fill_prefix(rec, b: bytes) -> None:
    """fs_seed_prefix for the text `b` (include/frontier_b200.h): short texts whole,
    long ones as their tail and the midstate of their leading 64-byte blocks."""
    rec["len"] = len(b)
    rec["mid_blocks"] = len(b) // 64
    if len(b) <= abi.MAX_PREFIX_BYTES:
        rec["bytes"][: len(b)] = np.frombuffer(b, dtype=np.uint8)
        return
    skip = 64 * (len(b) // 64)
    tail = b[skip:]
    if tail:
        rec["bytes"][: len(tail)] = np.frombuffer(tail, dtype=np.uint8)
    rec["mid"] = sha256_midstate(b[:skip])


def _prefix(text: str) -> np.void:
    rec = np.zeros((), dtype=abi.SEED_PREFIX)
    _fill_prefix(rec, text.encode("utf-8"))
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


def _check_static(sp: InstanceSpec) -> int:
    """The seed- and request-independent checks of check_spec; returns the longest
    replica key (for the router-seed prefix bound)."""
    dep, model = sp.deployment, sp.deployment.model
    sp.policy.validate()
    layout = replica_layout(dep)
    if not layout:
        raise SimulationError(f"{dep.mode} deployment has no serving replicas")
    if len(layout) > abi.MAX_REPLICAS:
        raise EngineCapacityError(f"{len(layout)} replicas exceed {abi.MAX_REPLICAS}")
    if model.moe is not None and model.moe.num_experts > abi.MAX_EXPERTS:
        raise EngineCapacityError(f"{model.moe.num_experts} experts exceed {abi.MAX_EXPERTS}")
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
    return max(len(ri.key.encode("utf-8")) for ri in layout)


def check_spec(sp: InstanceSpec) -> None:
    """The per-instance checks the reference makes inside make_simulation
    (base.py:71-111, af.py:381-392, cluster.py:108-118) plus the engine's
    capacity limits. simulate() runs this per point, so a bad point becomes a
    Failure row (cli.py:229-233) and lower() cannot raise for the others.
    The seed-independent part is memoised on the Deployment (sweep points of one
    config share it; the memo keeps the objects it keys on alive)."""
    memo = sp.deployment.__dict__.setdefault("_spec_checks", {})
    key = (sp.policy, sp.af, id(sp.attention_model), id(sp.grouped_gemm_model))
    hit = memo.get(key)
    if hit is None:
        try:
            longest = _check_static(sp)
        except Exception as exc:
            longest = exc
        hit = memo[key] = (sp.attention_model, sp.grouped_gemm_model, longest)
    if isinstance(hit[2], Exception):
        raise hit[2]
    ids = sp.requests.ids
    if ids is not _RANKS_CACHE.get(len(ids), (None,))[0] and len(set(ids)) != len(ids):
        raise SimulationError("duplicate request id")
    sp.__dict__["_checked"] = True


class _Template:
    """Everything `lower` derives from an instance that does not depend on its seed
    or its requests: the descriptor row, the replica rows (prefix indices relative
    to the instance's first prefix), the replica keys and trace counts. A sweep's
    config x seed points share one per config (parse_many shares the objects)."""

    __slots__ = ("desc", "reps", "keys", "prefix_suffix", "trace", "af")

    def __init__(self, sp: InstanceSpec, forests: ForestSet) -> None:
        dep, model, pol = sp.deployment, sp.deployment.model, sp.policy
        layout = replica_layout(dep)
        d = np.zeros((), dtype=abi.INSTANCE_DESC)
        d["mode"] = abi.MODE[dep.mode]
        d["n_replicas"] = len(layout)
        for f in ("num_layers", "d_model", "d_ff", "num_query_heads", "num_kv_heads", "head_dim",
                  "dtype_bytes"):
            d[f] = getattr(model, f)
        d["ffn_matrices"] = model.ffn_matrices
        if model.moe is not None:
            if model.moe.num_experts > abi.MAX_EXPERTS:
                raise EngineCapacityError(f"{model.moe.num_experts} experts exceed {abi.MAX_EXPERTS}")
            d["has_moe"] = 1
            d["num_experts"] = model.moe.num_experts
            d["top_k"] = model.moe.top_k
            d["expert_d_ff"] = model.moe.expert_d_ff
        d["admission"] = abi.ADMISSION[pol.admission]
        d["priority_key"] = abi.PRIORITY_KEY[pol.priority_key]
        d["max_num_seqs"] = pol.max_num_seqs
        d["max_batch_tokens"] = pol.max_batch_tokens
        d["paged"] = 1 if pol.memory_mode == "paged" else 0
        d["block_tokens"] = pol.block_tokens
        rt = sp.routing
        d["routing_policy"] = abi.ROUTING[rt.policy]
        d["routing_alpha"] = rt.alpha
        self.trace = [int(c) for c in rt.trace_counts] if rt.trace_counts else []
        d["n_trace_counts"] = len(self.trace)
        net = dep.network
        d["intra_latency_s"] = net.intra_replica.latency_s
        d["intra_bandwidth_bps"] = net.intra_replica.bandwidth_bps
        d["inter_latency_s"] = net.inter_cluster.latency_s
        d["inter_bandwidth_bps"] = net.inter_cluster.bandwidth_bps
        d["kv_bytes_per_token"] = kv_bytes_per_token(model)
        d["max_events"] = sp.max_events
        d["total_gpus"] = dep.total_gpus
        for slot, m, schema in (("attn_forest", sp.attention_model, "attention_v1"),
                                ("gg_forest", sp.grouped_gemm_model, "grouped_gemm_v1")):
            if m is not None and m.schema == schema and m.n_trees > abi.MAX_FOREST_TREES:
                raise EngineCapacityError(
                    f"{m.path}: {m.n_trees} trees exceed {abi.MAX_FOREST_TREES}")
            d[slot] = forest_slot(forests, m, schema)
        self.af = dep.mode == "af"
        if self.af:
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
        self.desc = d
        self.keys = [ri.key for ri in layout]
        key_rank = {k: r for r, k in enumerate(sorted(self.keys))}
        reps, suffix = [], []
        for ri in layout:
            c, p = ri.cluster, ri.cluster.parallelism
            pidx = len(suffix)
            suffix.append(f":{ri.key}:")
            pmb = -1
            if self.af:
                cost = _cost(c.hardware, p.attn_tp, 1, 1, p.pp)
                pmb = len(suffix)
                suffix.append(f":{ri.key}:mb")
            else:
                cost = _cost(c.hardware, p.tp, p.ep, p.tp, p.pp)
            reps.append((abi.ROLE[ri.role], key_rank[ri.key], c.kv_pool_tokens, cost, pidx, pmb))
        self.reps = np.array(reps, dtype=abi.REPLICA_DESC)
        self.prefix_suffix = suffix  # prefix text = f"{seed}{suffix}"


def _template_key(sp: InstanceSpec) -> tuple:
    return (id(sp.deployment), id(sp.policy), id(sp.routing), id(sp.af),
            id(sp.attention_model), id(sp.grouped_gemm_model), sp.max_events)


_RANKS_CACHE: dict[int, tuple[list[str], np.ndarray]] = {}


def shared_ids(n: int) -> list[str]:
    """The id list ["r0", ..., "r{n-1}"] of a generated workload, one shared list per
    n (treated as immutable), with its str-order ranks computed once."""
    hit = _RANKS_CACHE.get(n)
    if hit is None:
        ids = [f"r{k}" for k in range(n)]
        hit = _RANKS_CACHE[n] = (ids, _id_ranks(ids))
    return hit[0]


def _ranks_of(ids: list[str]) -> np.ndarray:
    """_id_ranks, cached for the generated id lists r0..r{n-1} (shared lists)."""
    hit = _RANKS_CACHE.get(len(ids))
    if hit is not None and hit[0] is ids:
        return hit[1]
    return _id_ranks(ids)


def lower(specs: list[InstanceSpec]) -> Lowered:
    """Pack instances for fs_run_batch. Seed-independent parts are built once per
    template (_Template); per instance only offsets, seeds' router-seed prefixes
    and the request arrays are added, mostly as whole-array numpy operations."""
    n = len(specs)
    forests = ForestSet()
    templates: dict[tuple, _Template] = {}
    tmpl_of: list[_Template] = []
    for sp in specs:
        if not getattr(sp, "_checked", False):
            check_spec(sp)
        key = _template_key(sp)
        t = templates.get(key)
        if t is None:
            t = templates[key] = _Template(sp, forests)
        tmpl_of.append(t)
    descs = np.zeros(n, dtype=abi.INSTANCE_DESC)
    uniq = list({id(t): t for t in tmpl_of}.values())
    pos = {id(t): j for j, t in enumerate(uniq)}
    which = np.fromiter((pos[id(t)] for t in tmpl_of), dtype=np.int64, count=n)
    if n:
        tdesc = np.zeros(len(uniq), dtype=abi.INSTANCE_DESC)
        for j, t in enumerate(uniq):
            tdesc[j] = t.desc
        descs[:] = tdesc[which]
    n_req = np.fromiter((len(sp.requests) for sp in specs), dtype=np.int64, count=n)
    n_rep = descs["n_replicas"].astype(np.int64)
    req_off = np.concatenate([[0], np.cumsum(n_req)[:-1]]) if n else n_req
    rep_off = np.concatenate([[0], np.cumsum(n_rep)[:-1]]) if n else n_rep
    descs["n_requests"] = n_req
    descs["req_offset"] = req_off
    descs["replica_offset"] = rep_off
    n_pref = np.fromiter((len(t.prefix_suffix) for t in tmpl_of), dtype=np.int64, count=n)
    pref_off = np.concatenate([[0], np.cumsum(n_pref)[:-1]]) if n else n_pref
    n_tr = np.fromiter((len(t.trace) for t in tmpl_of), dtype=np.int64, count=n)
    if n:
        descs["trace_offset"] = np.concatenate([[0], np.cumsum(n_tr)[:-1]])
    trace: list[int] = [c for t in tmpl_of for c in t.trace]
    # replicas: template rows with prefix indices made global
    if n:
        # gather template rows: row j of instance i = template row (tbase[which[i]] + j)
        tsize = np.array([len(t.reps) for t in uniq], dtype=np.int64)
        tbase = np.concatenate([[0], np.cumsum(tsize)[:-1]])
        trows = np.zeros(int(tsize.sum()), dtype=abi.REPLICA_DESC)
        for j, t in enumerate(uniq):
            trows[tbase[j]: tbase[j] + tsize[j]] = t.reps
        within = np.arange(int(n_rep.sum()), dtype=np.int64) - np.repeat(rep_off, n_rep)
        replicas = trows[np.repeat(tbase[which], n_rep) + within]
        shift = np.repeat(pref_off, n_rep)
        replicas["prefix"] += shift.astype(np.int32)
        mb = replicas["prefix_mb"] >= 0
        replicas["prefix_mb"][mb] += shift[mb].astype(np.int32)
    else:
        replicas = np.zeros(0, abi.REPLICA_DESC)
    # router-seed prefixes "{seed}:{key}:" (and ":mb") for every replica
    texts = [f"{sp.seed}{suf}".encode("utf-8") for sp, t in zip(specs, tmpl_of)
             for suf in t.prefix_suffix]
    pref = np.zeros(len(texts), dtype=abi.SEED_PREFIX)
    if texts:
        lens = np.fromiter((len(b) for b in texts), dtype=np.int64, count=len(texts))
        long_ = np.flatnonzero(lens > abi.MAX_PREFIX_BYTES).tolist()
        for j in long_:  # tail + host midstate (rare: cluster ids of ~180+ characters)
            texts[j] = b""
        buf = b"".join(b.ljust(abi.MAX_PREFIX_BYTES, b"\0") for b in texts)
        pref["bytes"] = np.frombuffer(buf, dtype=np.uint8).reshape(len(texts), abi.MAX_PREFIX_BYTES)
        pref["len"] = lens
        pref["mid_blocks"] = lens // 64
        if long_:
            full = [f"{sp.seed}{suf}".encode("utf-8") for sp, t in zip(specs, tmpl_of)
                    for suf in t.prefix_suffix]
            for j in long_:
                _fill_prefix(pref[j], full[j])
    # request struct-of-arrays
    cat = lambda parts, dt: np.concatenate(parts).astype(dt, copy=False) if parts else np.zeros(0, dt)  # noqa: E731
    arrival = cat([sp.requests.arrival_ns for sp in specs], np.int64)
    prompt = cat([sp.requests.prompt for sp in specs], np.int32)
    output = cat([sp.requests.output for sp in specs], np.int32)
    id_rank = cat([sp.requests.id_rank if getattr(sp.requests, "id_rank", None) is not None
                   else _ranks_of(sp.requests.ids) for sp in specs], np.int32)
    # est_cost (_estimate_cost) over the concatenated arrays
    if n:
        nz = n_req > 0
        starts = req_off[nz]
        out_tok = np.zeros(n, np.int64)
        pr_tok = np.zeros(n, np.int64)
        if len(starts):
            out_tok[nz] = np.add.reduceat(output.astype(np.int64), starts)
            pr_tok[nz] = np.add.reduceat(prompt.astype(np.int64), starts)
        out_tok += n_req
        L = descs["num_layers"].astype(np.int64)
        work = out_tok * L
        moe = descs["has_moe"] != 0
        work[moe] += (out_tok + pr_tok)[moe] * L[moe] * descs["num_experts"][moe] // 4
        descs["est_cost"] = work
    return Lowered(
        descs=descs, replicas=replicas, prefixes=pref,
        trace_counts=np.asarray(trace if trace else [0], dtype=np.int64),
        arrival=arrival, prompt=prompt, output=output, id_rank=id_rank,
        replica_keys=[t.keys for t in tmpl_of],
        request_ids=[sp.requests.ids for sp in specs],
        forests=forests if forests.models else None)
