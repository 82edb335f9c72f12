"""numpy mirrors of the C ABI structs in include/frontier_b200.h.

Structured dtypes with align=True follow the C layout rules; `check_sizes`
compares them against the library's own sizeof values at load time.
"""

from __future__ import annotations

import ctypes

import numpy as np

MAX_PREFIX_BYTES = 192
MAX_EXPERTS = 1024
MAX_TOPK = 16
MAX_MICRO_BATCHES = 64
MAX_REPLICAS = 65536
MAX_FOREST_TREES = 256  # fs_forest.cuh kMaxForestTrees (per-warp leaf sort in shared memory)
DEFAULT_MAX_EVENTS = 50_000_000

MODE = {"colocated": 0, "pd": 1, "af": 2}
ROLE = {"colocated": 0, "prefill": 1, "decode": 2, "attention": 3, "ffn": 4}
ADMISSION = {"fcfs": 0, "fcfs_skip": 1, "priority": 2}
PRIORITY_KEY = {"prompt_tokens": 0, "arrival_time": 1}
ROUTING = {"uniform": 0, "dirichlet_skew": 1, "trace": 2}
PHASES = {0: "prefill", 1: "decode", 2: "af_decode"}
AF_RESOURCES = ("attn_exec", "a2f_link", "ffn_exec", "f2a_link")

COST_CTX = np.dtype([("peak_flops", "<f8"), ("mem_bw", "<f8"), ("kernel_overhead_us", "<f8"),
                     ("tp", "<i4"), ("ep", "<i4"), ("moe_tp", "<i4"), ("pp", "<i4")], align=True)

SEED_PREFIX = np.dtype([("bytes", "u1", (MAX_PREFIX_BYTES,)), ("len", "<i4"),
                        ("mid_blocks", "<i4"), ("mid", "<u4", (8,))], align=True)

REPLICA_DESC = np.dtype([("role", "<i4"), ("key_rank", "<i4"), ("kv_pool_tokens", "<i8"),
                         ("cost", COST_CTX), ("prefix", "<i4"), ("prefix_mb", "<i4")], align=True)

INSTANCE_DESC = np.dtype([
    ("mode", "<i4"), ("n_requests", "<i4"), ("req_offset", "<i8"),
    ("n_replicas", "<i4"), ("replica_offset", "<i4"),
    ("num_layers", "<i4"), ("d_model", "<i4"), ("d_ff", "<i4"), ("num_query_heads", "<i4"),
    ("num_kv_heads", "<i4"), ("head_dim", "<i4"), ("dtype_bytes", "<i4"),
    ("has_moe", "<i4"), ("num_experts", "<i4"), ("top_k", "<i4"), ("expert_d_ff", "<i4"),
    ("ffn_matrices", "<i4"),
    ("admission", "<i4"), ("priority_key", "<i4"), ("max_num_seqs", "<i4"),
    ("max_batch_tokens", "<i4"), ("paged", "<i4"), ("block_tokens", "<i4"),
    ("routing_policy", "<i4"), ("n_trace_counts", "<i4"), ("trace_offset", "<i8"),
    ("routing_alpha", "<f8"),
    ("af_micro_batches", "<i4"), ("af_attn_dp", "<i4"),
    ("af_attn", COST_CTX), ("af_ffn", COST_CTX),
    ("intra_latency_s", "<f8"), ("intra_bandwidth_bps", "<f8"),
    ("inter_latency_s", "<f8"), ("inter_bandwidth_bps", "<f8"),
    ("kv_bytes_per_token", "<i8"), ("max_events", "<i8"),
    ("total_gpus", "<i4"), ("attn_forest", "<i4"), ("gg_forest", "<i4"), ("pad0", "<i4"),
    ("est_cost", "<i8"),
], align=True)

METRIC_ROW = np.dtype([
    ("status", "<i4"), ("status_detail", "<i4"),
    ("iterations", "<i8"), ("events", "<i8"), ("total_tokens", "<i8"), ("makespan_ns", "<i8"),
    ("prefill_batches", "<i8"), ("decode_batches", "<i8"), ("af_steps", "<i8"),
    ("n_requests", "<i4"), ("n_tpot", "<i4"),
    ("makespan_s", "<f8"), ("throughput_tokens_per_s_per_gpu", "<f8"),
    ("ttft", "<f8", (4,)), ("tpot", "<f8", (4,)), ("e2e", "<f8", (4,)),
    ("bubble_fraction", "<f8"), ("avg_input_tokens", "<f8"), ("avg_output_tokens", "<f8"),
    ("af_busy_ns", "<i8", (4,)), ("af_busy_fraction", "<f8", (4,)),
    ("moe_layer_samples", "<i8"), ("routing_calls", "<i8"), ("routing_draws", "<i8"),
], align=True)

REPLICA_OUT = np.dtype([("busy_ns", "<i8"), ("busy_fraction", "<f8"),
                        ("steps_executed", "<i8")], align=True)

BATCH_REC = np.dtype([("replica", "<i4"), ("phase", "<i4"), ("t_complete", "<i8"),
                      ("duration_ns", "<i8"), ("n_members", "<i4"), ("member_offset", "<i4"),
                      ("moe_offset", "<i4"), ("n_moe", "<i4"), ("seq", "<i8"),
                      ("pool_used", "<i8"), ("af_step", "<i8")], align=True)

# fs_event_rec / enum fs_event_kind (core.py:38-51 EventKind order)
EVENT_REC = np.dtype([("t", "<i8"), ("seq", "<i8"), ("x", "<i8"), ("a", "<i4"), ("b", "<i4"),
                      ("c", "<i4"), ("replica", "<i2"), ("kind", "u1"), ("pad", "u1")],
                     align=True)
EVENT_KINDS = ("REQUEST_ARRIVAL", "BATCH_START", "BATCH_COMPLETE", "PREFILL_COMPLETE",
               "MEMORY_AVAILABLE", "KV_CACHE_TRANSFER_START", "KV_CACHE_TRANSFER_DONE",
               "ATTN_COMPUTE_DONE", "A_TO_F_TRANSFER_DONE", "FFN_COMPUTE_DONE",
               "F_TO_A_TRANSFER_DONE", "TOKEN_EMITTED", "REQUEST_COMPLETE")

ROUTE_REC = np.dtype([("replica", "<i4"), ("micro_batch", "<i4"), ("step", "<i8"),
                      ("layer", "<i4"), ("tokens", "<i4"), ("counts_offset", "<i4"),
                      ("n_experts", "<i4")], align=True)

ATTN_PARAMS = np.dtype([("num_query_heads", "<i4"), ("num_kv_heads", "<i4"), ("head_dim", "<i4"),
                        ("dtype_bytes", "<i4"), ("peak_flops", "<f8"), ("mem_bw", "<f8"),
                        ("kernel_overhead_us", "<f8")], align=True)

FOREST_DESC = np.dtype([("n_trees", "<i4"), ("n_features", "<i4"), ("tree_offset", "<i8")],
                       align=True)

LENGTH_DIST = np.dtype([("kind", "<i4"), ("pad", "<i4"), ("value", "<i8"), ("lo", "<i8"),
                        ("hi", "<i8"), ("mu", "<f8"), ("sigma", "<f8")], align=True)
WORKLOAD_DESC = np.dtype([("seed", "<u8"), ("n_requests", "<i4"), ("arrival_kind", "<i4"),
                          ("rate_rps", "<f8"), ("gap_ns", "<i8"), ("out_offset", "<i8"),
                          ("prompt", LENGTH_DIST), ("output", LENGTH_DIST)], align=True)
ARRIVAL_KINDS = {"poisson": 0, "fixed_interval": 1, "batch_at_zero": 2}
LENGTH_KINDS = {"fixed": 0, "uniform": 1, "lognormal": 2}

STRUCT_ORDER = (COST_CTX, SEED_PREFIX, REPLICA_DESC, INSTANCE_DESC, METRIC_ROW, REPLICA_OUT,
                BATCH_REC, ROUTE_REC, ATTN_PARAMS, FOREST_DESC, WORKLOAD_DESC, EVENT_REC)


class RequestSoA(ctypes.Structure):
    _fields_ = [("arrival_ns", ctypes.c_void_p), ("prompt_tokens", ctypes.c_void_p),
                ("output_tokens", ctypes.c_void_p), ("id_rank", ctypes.c_void_p)]


class ForestSetC(ctypes.Structure):
    _fields_ = [("forests", ctypes.c_void_p), ("n_forests", ctypes.c_int32),
                ("pad0", ctypes.c_int32), ("tree_root", ctypes.c_void_p),
                ("n_trees", ctypes.c_int64), ("feature", ctypes.c_void_p),
                ("threshold", ctypes.c_void_p), ("left", ctypes.c_void_p),
                ("right", ctypes.c_void_p), ("value", ctypes.c_void_p),
                ("n_nodes", ctypes.c_int64)]


class RequestOut(ctypes.Structure):
    _fields_ = [("first_token_ns", ctypes.c_void_p), ("done_ns", ctypes.c_void_p),
                ("completion_rank", ctypes.c_void_p)]


class LogC(ctypes.Structure):
    _fields_ = [
        ("batch_base", ctypes.c_void_p), ("batch_cap", ctypes.c_int32),
        ("member_base", ctypes.c_void_p), ("member_cap", ctypes.c_int32),
        ("moe_base", ctypes.c_void_p), ("moe_cap", ctypes.c_int32),
        ("route_base", ctypes.c_void_p), ("route_cap", ctypes.c_int32),
        ("counts_base", ctypes.c_void_p), ("counts_cap", ctypes.c_int32),
        ("batches", ctypes.c_void_p), ("members", ctypes.c_void_p), ("moe_ratio", ctypes.c_void_p),
        ("routes", ctypes.c_void_p), ("counts", ctypes.c_void_p),
        ("batch_count", ctypes.c_void_p), ("route_count", ctypes.c_void_p),
        ("truncated", ctypes.c_void_p),
        ("event_base", ctypes.c_void_p), ("event_cap", ctypes.c_int32), ("pad0", ctypes.c_int32),
        ("events", ctypes.c_void_p), ("event_count", ctypes.c_void_p),
    ]


def ptr(a: np.ndarray | None) -> int | None:
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def check_sizes(lib, fn_name: str) -> None:
    fn = getattr(lib, fn_name)
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
    out = np.zeros(16, dtype=np.int64)
    n = fn(ptr(out), 16)
    want = [dt.itemsize for dt in STRUCT_ORDER] + [ctypes.sizeof(LogC)]
    got = out[:n].tolist()
    if got[: len(want)] != want:
        raise RuntimeError(f"ABI struct size mismatch: library {got}, binding {want}")
