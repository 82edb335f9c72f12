"""ctypes binding of libfrontier_b200.so (include/frontier_b200.h).

The engine library is the only compute path: if it cannot be loaded or no
CUDA device is present, `Engine()` raises `EngineUnavailable`. There is no
CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import abi
from .lower import Lowered

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
LIB_PATH = os.environ.get("FS_ENGINE_LIB", os.path.join(LIB_DIR, "libfrontier_b200.so"))


class EngineUnavailable(RuntimeError):
    """The CUDA engine library is missing or no B200 is visible."""


class EngineError(RuntimeError):
    """A call-level engine failure (CUDA error, bad arguments)."""


_lib = None


def load_library(path: str = LIB_PATH):
    """Load and type the engine library (safe without a GPU: no CUDA call is made)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise EngineUnavailable(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    sig = {
        "fs_abi_version": (ctypes.c_int, []),
        "fs_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(vp)]),
        "fs_destroy": (None, [vp]),
        "fs_last_error": (ctypes.c_char_p, [vp]),
        "fs_last_launch_count": (ctypes.c_int, [vp]),
        "fs_run_batch": (ctypes.c_int, [vp, vp, i32, vp, i32, vp, i32, vp, i64, abi.RequestSoA,
                                        i64, vp, vp, abi.RequestOut, vp]),
        "fs_stage": (ctypes.c_int, [vp, vp, i32, vp, i32, vp, i32, vp, i64, abi.RequestSoA, i64]),
        "fs_launch_async": (ctypes.c_int, [vp, vp]),
        "fs_fetch": (ctypes.c_int, [vp, vp, vp, abi.RequestOut]),
        "fs_attention_cost": (ctypes.c_int, [vp, vp, vp, vp, vp, i64, _AttnParamsC, vp, vp]),
        "fs_attention_cost_dev": (ctypes.c_int, [vp, vp, vp, vp, vp, i64, _AttnParamsC, vp, vp, vp]),
        "fs_attention_features": (ctypes.c_int, [vp, vp, vp, vp, vp, i64, _AttnParamsC, vp]),
        "fs_attention_features_dev": (ctypes.c_int, [vp, vp, vp, vp, vp, i64, _AttnParamsC, vp, vp]),
        "fs_route_uniform": (ctypes.c_int, [vp, vp, vp, i32, i32, i32, vp, vp]),
        "fs_route_tokens": (ctypes.c_int, [vp, vp, vp, i32, i32, i32, i32, ctypes.c_double, vp,
                                           vp]),
        "fs_generate_workload": (ctypes.c_int, [vp, vp, i32, vp, vp, vp, vp, vp]),
        "fs_router_seeds": (ctypes.c_int, [vp, vp, vp, vp, vp, vp, i32, vp]),
        "fs_eval": (ctypes.c_int, [vp, i32, vp, i32, i64, vp, i32, vp]),
        "fs_set_forests": (ctypes.c_int, [vp, abi.ForestSetC]),
        "fs_attention_forest": (ctypes.c_int, [vp, i32, vp, vp, vp, vp, i64, _AttnParamsC, vp]),
        "fs_attention_forest_dev": (ctypes.c_int, [vp, i32, vp, vp, vp, vp, i64, _AttnParamsC,
                                                   vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    abi.check_sizes(lib, "fs_struct_sizes")
    if lib.fs_abi_version() != 2:
        raise EngineUnavailable("ABI version mismatch")
    _lib = lib
    return lib


class _AttnParamsC(ctypes.Structure):
    _fields_ = [("num_query_heads", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("dtype_bytes", ctypes.c_int32),
                ("peak_flops", ctypes.c_double), ("mem_bw", ctypes.c_double),
                ("kernel_overhead_us", ctypes.c_double)]


def attn_params(num_query_heads, num_kv_heads, head_dim, dtype_bytes, peak_flops, mem_bw,
                kernel_overhead_us=5.0) -> _AttnParamsC:
    return _AttnParamsC(num_query_heads, num_kv_heads, head_dim, dtype_bytes, peak_flops, mem_bw,
                        kernel_overhead_us)


@dataclass
class LogSpec:
    """Per-instance capacities of the optional batch / routing / event-trace log."""

    batch_cap: int = 0
    member_cap: int = 0
    moe_cap: int = 0
    route_cap: int = 0
    counts_cap: int = 0
    event_cap: int = 0


@dataclass
class RawLog:
    spec: LogSpec
    batches: np.ndarray
    members: np.ndarray
    moe: np.ndarray
    routes: np.ndarray
    counts: np.ndarray
    batch_count: np.ndarray
    route_count: np.ndarray
    truncated: np.ndarray
    c_struct: abi.LogC
    events: np.ndarray | None = None
    event_count: np.ndarray | None = None
    bases: dict | None = None

    def instance_batches(self, i: int) -> list[dict]:
        """Batch records of instance i in BATCH_COMPLETE dispatch order (t_complete, seq);
        the engine records them when they start. `index` = position in the raw log."""
        n = int(self.batch_count[i])
        bb, mb, eb = self.bases["batch"][i], self.bases["member"][i], self.bases["moe"][i]
        raw = self.batches[bb: bb + n]
        order = np.lexsort((raw["seq"], raw["t_complete"])) if n else []
        out = []
        for j in order:
            b = raw[j]
            mo = int(b["member_offset"])
            mem = self.members[mb + mo: mb + mo + int(b["n_members"])]
            moe = None
            if b["n_moe"] > 0:
                eo = eb + int(b["moe_offset"])
                moe = self.moe[eo: eo + int(b["n_moe"])].tolist()
            out.append({"replica": int(b["replica"]), "phase": abi.PHASES[int(b["phase"])],
                        "t_complete": int(b["t_complete"]), "duration_ns": int(b["duration_ns"]),
                        "members": mem.tolist(), "moe_ratio": moe, "seq": int(b["seq"]),
                        "pool_used": int(b["pool_used"]), "af_step": int(b["af_step"]),
                        "index": int(j)})
        return out

    def instance_events(self, i: int) -> np.ndarray:
        """Event records of instance i indexed by seq (fs_event_rec)."""
        cap = self.spec.event_cap
        n = int(self.event_count[i])
        if n > cap:
            raise RuntimeError(f"event log of instance {i} truncated ({n} events, cap {cap})")
        b = self.bases["event"][i]
        return self.events[b: b + n].copy()

    def moe_imbalance(self, i: int) -> list[float]:
        """expert_imbalance of instance i (metrics.py:105-109): the per-layer values of
        its prefill/decode batches in BATCH_COMPLETE order (already round(x, 6))."""
        n = int(self.batch_count[i])
        if n == 0:
            return []
        bb, eb = self.bases["batch"][i], self.bases["moe"][i]
        raw = self.batches[bb: bb + n]
        raw = raw[np.lexsort((raw["seq"], raw["t_complete"]))]
        raw = raw[raw["n_moe"] > 0]
        if len(raw) == 0:
            return []
        L = int(raw["n_moe"][0])
        idx = eb + raw["moe_offset"].astype(np.int64)[:, None] + np.arange(L)[None, :]
        return self.moe[idx.ravel()].tolist()

    def instance_routes(self, i: int) -> list[dict]:
        out = []
        rb, cb = self.bases["route"][i], self.bases["counts"][i]
        for j in range(int(self.route_count[i])):
            r = self.routes[rb + j]
            co = cb + int(r["counts_offset"])
            out.append({"replica": int(r["replica"]), "micro_batch": int(r["micro_batch"]),
                        "step": int(r["step"]), "layer": int(r["layer"]),
                        "tokens": int(r["tokens"]),
                        "counts": self.counts[co: co + int(r["n_experts"])].tolist()})
        return out


_LOG_FIELDS = ("batch", "member", "moe", "route", "counts", "event")


def make_log(n_instances: int, spec: LogSpec, sizes: dict | None = None) -> RawLog:
    """Log buffers: instance i owns [base_i, base_i + cap) of each array. `sizes`
    (field -> per-instance int array) packs regions of exactly those sizes instead
    of `cap` each -- for a re-run whose record counts are known, since a run
    never writes more records than it produces (the caps stay the maxima)."""
    sizes = sizes or {}
    bases, total = {}, {}
    for f in _LOG_FIELDS:
        cap = getattr(spec, f + "_cap")
        sz = np.asarray(sizes[f], dtype=np.int64) if f in sizes else np.full(n_instances, cap, np.int64)
        bases[f] = np.concatenate([[0], np.cumsum(sz)[:-1]]).astype(np.int64) if n_instances \
            else np.zeros(0, np.int64)
        # fs_run_batch copies max_i(base_i + cap) records back (include/frontier_b200.h,
        # fs_log): with packed regions the last one still needs `cap` slots of room
        total[f] = int((bases[f] + cap).max()) if cap and n_instances else 0
    log = RawLog(
        spec=spec,
        batches=np.zeros(max(1, total["batch"]), dtype=abi.BATCH_REC),
        members=np.zeros(max(1, total["member"]), dtype=np.int32),
        moe=np.zeros(max(1, total["moe"]), dtype=np.float64),
        routes=np.zeros(max(1, total["route"]), dtype=abi.ROUTE_REC),
        counts=np.zeros(max(1, total["counts"]), dtype=np.int32),
        batch_count=np.zeros(n_instances, dtype=np.int32),
        route_count=np.zeros(n_instances, dtype=np.int32),
        truncated=np.zeros(n_instances, dtype=np.int32),
        c_struct=abi.LogC(),
        events=np.zeros(max(1, total["event"]), dtype=abi.EVENT_REC),
        event_count=np.zeros(n_instances, dtype=np.int64))
    log.bases = bases
    c = log.c_struct
    log._keep = [bases[f] for f in _LOG_FIELDS]
    c.event_base = abi.ptr(log._keep[5])
    c.event_cap = spec.event_cap
    c.events = abi.ptr(log.events) if spec.event_cap else None
    c.event_count = abi.ptr(log.event_count)
    c.batch_base, c.member_base, c.moe_base, c.route_base, c.counts_base = [
        abi.ptr(b) for b in log._keep[:5]]
    c.batch_cap, c.member_cap, c.moe_cap = spec.batch_cap, spec.member_cap, spec.moe_cap
    c.route_cap, c.counts_cap = spec.route_cap, spec.counts_cap
    c.batches = abi.ptr(log.batches) if spec.batch_cap else None
    c.members = abi.ptr(log.members) if spec.member_cap else None
    c.moe_ratio = abi.ptr(log.moe) if spec.moe_cap else None
    c.routes = abi.ptr(log.routes) if spec.route_cap else None
    c.counts = abi.ptr(log.counts) if spec.counts_cap else None
    c.batch_count = abi.ptr(log.batch_count)
    c.route_count = abi.ptr(log.route_count)
    c.truncated = abi.ptr(log.truncated)
    return log


@dataclass
class RawResults:
    rows: np.ndarray
    replica_out: np.ndarray
    first_ns: np.ndarray
    done_ns: np.ndarray
    done_rank: np.ndarray
    log: RawLog | None = None


def alloc_results(low: Lowered) -> RawResults:
    n = low.n_requests
    return RawResults(rows=np.zeros(low.n_instances, dtype=abi.METRIC_ROW),
                      replica_out=np.zeros(max(1, len(low.replicas)), dtype=abi.REPLICA_OUT),
                      first_ns=np.zeros(max(1, n), dtype=np.int64),
                      done_ns=np.zeros(max(1, n), dtype=np.int64),
                      done_rank=np.zeros(max(1, n), dtype=np.int32))


def soa(low: Lowered) -> abi.RequestSoA:
    return abi.RequestSoA(abi.ptr(low.arrival), abi.ptr(low.prompt), abi.ptr(low.output),
                          abi.ptr(low.id_rank))


class Engine:
    """One engine handle on one CUDA device."""

    def __init__(self, device: int = 0) -> None:
        self.lib = load_library()
        h = ctypes.c_void_p()
        rc = self.lib.fs_create(device, ctypes.byref(h))
        if rc != 0:
            raise EngineUnavailable(f"fs_create(device={device}) failed with code {rc} "
                                    "(no CUDA device visible?)")
        self.h = h
        self.device = device
        self._forests = None
        self._staged = None

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.fs_destroy(self.h)
            self.h = None

    def __del__(self) -> None:
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int, what: str) -> None:
        if rc != 0:
            msg = self.lib.fs_last_error(self.h)
            raise EngineError(f"{what} failed ({rc}): {msg.decode() if msg else ''}")

    @property
    def last_launch_count(self) -> int:
        return int(self.lib.fs_last_launch_count(self.h))

    # -- batched simulation -------------------------------------------------------------
    def set_forests(self, forests) -> None:
        """Stage learned operator models (costmodel.ForestSet) in HBM; kept until replaced."""
        from .costmodel import forest_set_struct
        if forests is None or forests is self._forests:
            return
        self._check(self.lib.fs_set_forests(self.h, forest_set_struct(forests)), "fs_set_forests")
        self._forests = forests

    def run(self, low: Lowered, log: LogSpec | None = None,
            log_sizes: dict | None = None) -> RawResults:
        self.set_forests(low.forests)
        res = alloc_results(low)
        if log is not None:
            res.log = make_log(low.n_instances, log, log_sizes)
        pr = abi.RequestOut(abi.ptr(res.first_ns), abi.ptr(res.done_ns), abi.ptr(res.done_rank))
        rc = self.lib.fs_run_batch(
            self.h, abi.ptr(low.descs), low.n_instances, abi.ptr(low.replicas), len(low.replicas),
            abi.ptr(low.prefixes), len(low.prefixes), abi.ptr(low.trace_counts),
            len(low.trace_counts), soa(low), low.n_requests, abi.ptr(res.rows),
            abi.ptr(res.replica_out), pr,
            ctypes.byref(res.log.c_struct) if res.log is not None else None)
        self._check(rc, "fs_run_batch")
        return res

    def stage(self, low: Lowered) -> None:
        self.set_forests(low.forests)
        rc = self.lib.fs_stage(
            self.h, abi.ptr(low.descs), low.n_instances, abi.ptr(low.replicas), len(low.replicas),
            abi.ptr(low.prefixes), len(low.prefixes), abi.ptr(low.trace_counts),
            len(low.trace_counts), soa(low), low.n_requests)
        self._check(rc, "fs_stage")
        self._staged = low

    def peer(self) -> "Engine":
        """A second engine on the same device (own staging buffers and stream), kept
        for the life of this one: lets a caller stage and launch the next batch while
        this engine's batch is still on the device (api.simulate's pipeline)."""
        p = getattr(self, "_peer", None)
        if p is None:
            p = self._peer = Engine(self.device)
        return p

    def launch(self, stream_ptr: int | None = None) -> None:
        self._check(self.lib.fs_launch_async(self.h, stream_ptr), "fs_launch_async")

    def fetch(self, low: Lowered | None = None, per_request: bool = True) -> RawResults:
        low = low or self._staged
        res = alloc_results(low)
        pr = abi.RequestOut(abi.ptr(res.first_ns) if per_request else None,
                            abi.ptr(res.done_ns) if per_request else None,
                            abi.ptr(res.done_rank) if per_request else None)
        self._check(self.lib.fs_fetch(self.h, abi.ptr(res.rows), abi.ptr(res.replica_out), pr),
                    "fs_fetch")
        return res

    # -- cost-model kernels ----------------------------------------------------------------
    def attention_cost(self, q, kv, offsets, is_decode, params) -> tuple[np.ndarray, np.ndarray]:
        q = np.ascontiguousarray(q, dtype=np.int32)
        kv = np.ascontiguousarray(kv, dtype=np.int32)
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        is_decode = np.ascontiguousarray(is_decode, dtype=np.uint8)
        nb = len(offsets) - 1
        out = np.zeros(max(nb, 1), dtype=np.float64)
        st = np.zeros(max(nb, 1), dtype=np.int32)
        self._check(self.lib.fs_attention_cost(self.h, abi.ptr(q), abi.ptr(kv), abi.ptr(offsets),
                                               abi.ptr(is_decode), nb, params, abi.ptr(out),
                                               abi.ptr(st)), "fs_attention_cost")
        return out[:nb], st[:nb]

    def attention_cost_dev(self, q_ptr, kv_ptr, off_ptr, dec_ptr, nb, params, out_ptr,
                           status_ptr, stream_ptr) -> None:
        self._check(self.lib.fs_attention_cost_dev(self.h, q_ptr, kv_ptr, off_ptr, dec_ptr, nb,
                                                   params, out_ptr, status_ptr, stream_ptr),
                    "fs_attention_cost_dev")

    def attention_features(self, q, kv, offsets, is_decode, params) -> np.ndarray:
        q = np.ascontiguousarray(q, dtype=np.int32)
        kv = np.ascontiguousarray(kv, dtype=np.int32)
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        is_decode = np.ascontiguousarray(is_decode, dtype=np.uint8)
        nb = len(offsets) - 1
        out = np.zeros((max(nb, 1), 17), dtype=np.float64)
        self._check(self.lib.fs_attention_features(self.h, abi.ptr(q), abi.ptr(kv),
                                                   abi.ptr(offsets), abi.ptr(is_decode), nb,
                                                   params, abi.ptr(out)), "fs_attention_features")
        return out[:nb]

    def attention_forest(self, forests, forest: int, q, kv, offsets, is_decode,
                         params) -> np.ndarray:
        """LearnedOperatorModel.predict_us(AttentionFeatures(...).vector()) per CSR batch."""
        self.set_forests(forests)
        q = np.ascontiguousarray(q, dtype=np.int32)
        kv = np.ascontiguousarray(kv, dtype=np.int32)
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        is_decode = np.ascontiguousarray(is_decode, dtype=np.uint8)
        nb = len(offsets) - 1
        out = np.zeros(max(nb, 1), dtype=np.float64)
        self._check(self.lib.fs_attention_forest(self.h, forest, abi.ptr(q), abi.ptr(kv),
                                                 abi.ptr(offsets), abi.ptr(is_decode), nb,
                                                 params, abi.ptr(out)), "fs_attention_forest")
        return out[:nb]

    def attention_forest_dev(self, forest: int, q_ptr, kv_ptr, off_ptr, dec_ptr, nb, params,
                             out_ptr, stream_ptr) -> None:
        """Device-pointer form of attention_forest (models staged with set_forests)."""
        self._check(self.lib.fs_attention_forest_dev(self.h, forest, q_ptr, kv_ptr, off_ptr,
                                                     dec_ptr, nb, params, out_ptr, stream_ptr),
                    "fs_attention_forest_dev")

    def route_uniform(self, tokens, seeds, num_experts: int, top_k: int):
        tokens = np.ascontiguousarray(tokens, dtype=np.int64)
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        n = len(tokens)
        counts = np.zeros((max(n, 1), num_experts), dtype=np.int32)
        st = np.zeros(max(n, 1), dtype=np.int32)
        self._check(self.lib.fs_route_uniform(self.h, abi.ptr(tokens), abi.ptr(seeds), n,
                                              num_experts, top_k, abi.ptr(counts), abi.ptr(st)),
                    "fs_route_uniform")
        return counts[:n], st[:n]

    def route_tokens(self, tokens, seeds, num_experts: int, top_k: int, policy: str = "uniform",
                     alpha: float = 0.3):
        """route_tokens(T, E, k, policy, seed, alpha).counts per call (routing.py:65-113)
        for the uniform and dirichlet_skew policies; returns (counts, status)."""
        tokens = np.ascontiguousarray(tokens, dtype=np.int64)
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        n = len(tokens)
        counts = np.zeros((max(n, 1), num_experts), dtype=np.int32)
        st = np.zeros(max(n, 1), dtype=np.int32)
        self._check(self.lib.fs_route_tokens(self.h, abi.ptr(tokens), abi.ptr(seeds), n,
                                             num_experts, top_k, abi.ROUTING[policy], alpha,
                                             abi.ptr(counts), abi.ptr(st)), "fs_route_tokens")
        return counts[:n], st[:n]

    def generate_workload(self, descs):
        """generate(spec) for fs_workload_desc rows on the device (workload.py:193-216):
        (arrival_ns int64, prompt int32, output int32, id_rank int32, status per row)."""
        descs = np.ascontiguousarray(descs, dtype=abi.WORKLOAD_DESC)
        n = len(descs)
        total = int((descs["out_offset"] + descs["n_requests"]).max()) if n else 0
        arr = np.zeros(max(total, 1), np.int64)
        pr = np.zeros(max(total, 1), np.int32)
        out = np.zeros(max(total, 1), np.int32)
        rk = np.zeros(max(total, 1), np.int32)
        st = np.zeros(max(n, 1), np.int32)
        self._check(self.lib.fs_generate_workload(self.h, abi.ptr(descs), n, abi.ptr(arr),
                                                  abi.ptr(pr), abi.ptr(out), abi.ptr(rk),
                                                  abi.ptr(st)), "fs_generate_workload")
        return arr[:total], pr[:total], out[:total], rk[:total], st[:n]

    def router_seeds(self, prefixes: list[str], prefix_idx, micro_batch, steps, layers):
        from .lower import _prefix
        pf = np.array([_prefix(p) for p in prefixes], dtype=abi.SEED_PREFIX)
        pidx = np.ascontiguousarray(prefix_idx, dtype=np.int32)
        mb = np.ascontiguousarray(micro_batch, dtype=np.int32)
        st = np.ascontiguousarray(steps, dtype=np.int64)
        ly = np.ascontiguousarray(layers, dtype=np.int32)
        out = np.zeros(max(len(pidx), 1), dtype=np.uint32)
        self._check(self.lib.fs_router_seeds(self.h, abi.ptr(pf), abi.ptr(pidx), abi.ptr(mb),
                                             abi.ptr(st), abi.ptr(ly), len(pidx), abi.ptr(out)),
                    "fs_router_seeds")
        return out[: len(pidx)]

    EVAL_FNS = {"exp": 1, "log": 2, "log1p": 3, "pow": 4, "linear": 5, "grouped_gemm": 6,
                "collective_int": 7, "collective_flt": 8, "transfer": 9, "moe_layer": 10,
                "cuda_exp": 11, "cuda_log": 12, "cuda_log1p": 13, "cuda_pow": 14}

    def eval(self, fn: str, records, out_stride: int = 1):
        """fs_eval: one pure cost-model / libm function per record on the device
        (include/frontier_b200.h, enum fs_eval_fn). Returns (out, status)."""
        rec = np.ascontiguousarray(np.atleast_2d(np.asarray(records, dtype=np.float64)))
        n, stride = rec.shape
        out = np.zeros((max(n, 1), out_stride), dtype=np.float64)
        st = np.zeros(max(n, 1), dtype=np.int32)
        self._check(self.lib.fs_eval(self.h, self.EVAL_FNS[fn], abi.ptr(rec), stride, n,
                                     abi.ptr(out), out_stride, abi.ptr(st)), "fs_eval")
        return out[:n], st[:n]


_default_engine: Engine | None = None


def default_engine() -> Engine:
    global _default_engine
    if _default_engine is None:
        import os as _os
        dev = int(_os.environ.get("LOCAL_RANK", "0"))
        _default_engine = Engine(dev)
    return _default_engine
