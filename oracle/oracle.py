"""ctypes wrapper of the C oracle (oracle/fs_oracle.c) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
legs may import this module. It consumes the same lowered arrays as the CUDA
engine (paper_2508_03148_b200.lower) and returns the same raw result layout,
so parity checks compare like with like.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from paper_2508_03148_b200 import abi
from paper_2508_03148_b200.costmodel import forest_set_struct
from paper_2508_03148_b200.engine import LogSpec, RawResults, alloc_results, make_log, soa
from paper_2508_03148_b200.lower import Lowered

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "build", "libfsoracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB):
        build()
    lib = ctypes.CDLL(LIB)
    vp = ctypes.c_void_p
    lib.fso_run_batch.restype = ctypes.c_int
    lib.fso_run_batch.argtypes = [vp, ctypes.c_int32, vp, vp, vp, abi.RequestSoA, vp, vp,
                                  abi.RequestOut, vp, ctypes.c_int, vp]
    lib.fso_router_seed.restype = ctypes.c_uint32
    lib.fso_router_seed.argtypes = [vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int32]
    lib.fso_routing_key.restype = None
    lib.fso_routing_key.argtypes = [ctypes.c_uint64, vp]
    lib.fso_route_uniform.restype = ctypes.c_int
    lib.fso_route_uniform.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                      ctypes.c_uint64, vp]
    lib.fso_route.restype = ctypes.c_int
    lib.fso_route.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                              ctypes.c_double, ctypes.c_uint64, vp]
    lib.fso_dirichlet_row.restype = None
    lib.fso_dirichlet_row.argtypes = [ctypes.c_int32, ctypes.c_double, ctypes.c_uint64, vp, vp]
    lib.fso_generate_workload.restype = ctypes.c_int
    lib.fso_generate_workload.argtypes = [vp, ctypes.c_int32, vp, vp, vp, vp, vp]
    lib.fso_collective.restype = ctypes.c_double
    lib.fso_collective.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_double,
                                   ctypes.c_double]
    lib.fso_gg_features.restype = ctypes.c_double
    lib.fso_gg_features.argtypes = [vp, ctypes.c_int, vp, ctypes.c_int, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_int, vp]
    lib.fso_attention_us.restype = ctypes.c_double
    lib.fso_attention_us.argtypes = [ctypes.c_int, vp, vp, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_int]
    lib.fso_linear_us.restype = ctypes.c_double
    lib.fso_linear_us.argtypes = [ctypes.c_int64] * 3 + [ctypes.c_double] * 3 + [ctypes.c_int]
    lib.fso_attention_forest.restype = ctypes.c_double
    lib.fso_attention_forest.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int, ctypes.c_int, vp]
    lib.fso_pysum.restype = ctypes.c_double
    lib.fso_pysum.argtypes = [vp, ctypes.c_int]
    lib.fso_libm.argtypes = [ctypes.c_int, vp, vp, vp, ctypes.c_int64]
    abi.check_sizes(lib, "fso_struct_sizes")
    _lib = lib
    return lib


def run(low: Lowered, log: LogSpec | None = None, threads: int = 1,
        log_sizes: dict | None = None) -> RawResults:
    lib = load()
    res = alloc_results(low)
    if log is not None:
        res.log = make_log(low.n_instances, log, log_sizes)
    pr = abi.RequestOut(abi.ptr(res.first_ns), abi.ptr(res.done_ns), abi.ptr(res.done_rank))
    fset = forest_set_struct(low.forests) if low.forests is not None else None
    lib.fso_run_batch(abi.ptr(low.descs), low.n_instances, abi.ptr(low.replicas),
                      abi.ptr(low.prefixes), abi.ptr(low.trace_counts), soa(low),
                      abi.ptr(res.rows), abi.ptr(res.replica_out), pr,
                      ctypes.byref(res.log.c_struct) if res.log is not None else None, threads,
                      ctypes.byref(fset) if fset is not None else None)
    return res


def router_seed(prefix: str, mb: int, step: int, layer: int) -> int:
    from paper_2508_03148_b200.lower import _prefix
    rec = np.array(_prefix(prefix), dtype=abi.SEED_PREFIX)
    return int(load().fso_router_seed(abi.ptr(rec), mb, step, layer))


def routing_key(seed: int) -> tuple[int, int]:
    k = np.zeros(2, dtype=np.uint64)
    load().fso_routing_key(seed, abi.ptr(k))
    return int(k[0]), int(k[1])


def route_uniform(T: int, E: int, k: int, seed: int) -> tuple[list[int], int]:
    c = np.zeros(E, dtype=np.int32)
    st = load().fso_route_uniform(T, E, k, seed, abi.ptr(c))
    return c.tolist(), st


def route(T: int, E: int, k: int, policy: str, seed: int, alpha: float = 0.3):
    """route_tokens(T, E, k, policy, seed, alpha).counts and a status (routing.py:65-113)."""
    c = np.zeros(E, dtype=np.int32)
    st = load().fso_route(T, E, k, abi.ROUTING[policy], alpha, seed, abi.ptr(c))
    return c.tolist(), st


def dirichlet_row(E: int, alpha: float, seed: int):
    """(popularity[E], first row of keys[E]) of route_tokens' dirichlet_skew stream."""
    pop = np.zeros(E)
    keys = np.zeros(E)
    load().fso_dirichlet_row(E, alpha, seed, abi.ptr(pop), abi.ptr(keys))
    return pop, keys


def attention_us(decode: bool, q, kv, hq, hkv, hd, peak, bw, ovh=5.0, dt=2) -> float:
    q = np.ascontiguousarray(q, dtype=np.int64)
    kv = np.ascontiguousarray(kv, dtype=np.int64)
    return load().fso_attention_us(int(decode), abi.ptr(q), abi.ptr(kv), len(q), hq, hkv, hd,
                                   peak, bw, ovh, dt)


def attention_forest(forests, forest: int, decode: bool, q, kv, hq: int, hkv: int, hd: int):
    """(prediction_us, features[17]) for one batch: AttentionFeatures.vector() and
    LearnedOperatorModel.predict_us (costmodel/features.py:101-115, model.py:126-136)."""
    q = np.ascontiguousarray(q, dtype=np.int64)
    kv = np.ascontiguousarray(kv, dtype=np.int64)
    x = np.zeros(17, dtype=np.float64)
    fset = forest_set_struct(forests)
    v = load().fso_attention_forest(ctypes.byref(fset), forest, int(decode), abi.ptr(q),
                                    abi.ptr(kv), len(q), hq, hkv, hd, abi.ptr(x))
    return v, x


def gg_features(counts, d_model: int, d_ff: int, top_k: int, forests=None, forest: int = 0):
    """(GroupedGemmFeatures(..., "local").vector(), learned prediction or 0.0)."""
    c = np.ascontiguousarray(counts, dtype=np.int64)
    x = np.zeros(12)
    fset = forest_set_struct(forests) if forests is not None else None
    v = load().fso_gg_features(ctypes.byref(fset) if fset is not None else None, forest,
                               abi.ptr(c), len(c), d_model, d_ff, top_k, abi.ptr(x))
    return x, v


def generate_workload(descs):
    """(arrival_ns, prompt, output, id_rank, status) for fs_workload_desc rows."""
    descs = np.ascontiguousarray(descs, dtype=abi.WORKLOAD_DESC)
    n_total = int((descs["out_offset"] + descs["n_requests"]).max()) if len(descs) else 0
    arr = np.zeros(max(n_total, 1), np.int64)
    pr = np.zeros(max(n_total, 1), np.int32)
    out = np.zeros(max(n_total, 1), np.int32)
    rk = np.zeros(max(n_total, 1), np.int32)
    st = np.zeros(max(len(descs), 1), np.int32)
    load().fso_generate_workload(abi.ptr(descs), len(descs), abi.ptr(arr), abi.ptr(pr),
                                 abi.ptr(out), abi.ptr(rk), abi.ptr(st))
    return arr[:n_total], pr[:n_total], out[:n_total], rk[:n_total], st[:len(descs)]


def libm(fn: str, x, y=None) -> np.ndarray:
    """The host C library's exp / log / log1p / pow elementwise (glibc, as numpy's
    distributions.c calls them)."""
    code = {"exp": 1, "log": 2, "log1p": 3, "pow": 4}[fn]
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(x if y is None else y, dtype=np.float64)
    out = np.zeros_like(x)
    load().fso_libm(code, x.ctypes.data, y.ctypes.data, out.ctypes.data, len(x))
    return out


def pysum(xs) -> float:
    a = np.ascontiguousarray(xs, dtype=np.float64)
    return load().fso_pysum(abi.ptr(a), len(a))


class OracleEngine:
    """The oracle behind the Engine interface (run(lowered, log=...)) -- lets tests
    drive the host API (simulate, make_simulation, refbind) on CPU."""

    def __init__(self, threads: int = 8) -> None:
        self.threads = threads
        self.last_launch_count = 0

    def run(self, low: Lowered, log: LogSpec | None = None, log_sizes: dict | None = None):
        return run(low, log=log, threads=self.threads, log_sizes=log_sizes)

    # the Engine's stage / launch / fetch / peer, as api.simulate's pipeline uses them
    def stage(self, low: Lowered) -> None:
        self._staged, self._result = low, None

    def launch(self, stream_ptr=None) -> None:
        self._result = run(self._staged, threads=self.threads)

    def fetch(self, low: Lowered | None = None, per_request: bool = True):
        return self._result

    def peer(self) -> "OracleEngine":
        p = getattr(self, "_peer", None)
        if p is None:
            p = self._peer = OracleEngine(self.threads)
        return p
