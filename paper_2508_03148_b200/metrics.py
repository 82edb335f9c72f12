"""Metric reports (reference: pkg/src/frontier_sim/metrics.py).

The reductions of `compute_metrics` (means, nearest-rank percentiles,
makespan, throughput, busy and bubble fractions) run on the device
(csrc/fs_metrics.cu); this module only re-shapes the device's metric row
into the reference's `MetricsBundle` and provides the report-format helpers
(`pareto_frontier`, `summary_csv_row`) used by the sweep driver.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import abi
from .errors import STATUS_EXCEPTIONS, SimulationError


class IncompleteTrace(Exception):
    """A run with requests that never completed was asked for metrics."""


@dataclass
class MetricsBundle:
    per_request: dict[str, dict[str, float | None]]
    ttft: dict[str, float] | None
    tpot: dict[str, float] | None
    e2e: dict[str, float] | None
    total_tokens: int
    makespan_s: float
    total_gpus: int
    throughput_tokens_per_s_per_gpu: float
    busy_fraction: dict[str, float]
    bubble_fraction: float | None
    expert_imbalance: list[float] | None
    workload_summary: dict[str, float]

    def to_dict(self) -> dict:
        return {
            "per_request": self.per_request,
            "aggregates": {"ttft_s": self.ttft, "tpot_s": self.tpot, "e2e_s": self.e2e},
            "total_tokens": self.total_tokens,
            "makespan_s": self.makespan_s,
            "total_gpus": self.total_gpus,
            "throughput_tokens_per_s_per_gpu": self.throughput_tokens_per_s_per_gpu,
            "busy_fraction": self.busy_fraction,
            "bubble_fraction": self.bubble_fraction,
            "expert_imbalance": self.expert_imbalance,
            "workload_summary": self.workload_summary,
        }


@dataclass
class InstanceResult:
    """Device outputs of one simulated instance (the analogue of the
    reference's EventTrace: what compute_metrics needs)."""

    index: int
    row: np.void
    replica_keys: list[str]
    replica_out: np.ndarray
    request_ids: list[str]
    arrival_ns: np.ndarray
    prompt: np.ndarray
    output: np.ndarray
    first_token_ns: np.ndarray
    done_ns: np.ndarray
    completion_rank: np.ndarray
    total_gpus: int
    mode: str
    batches: list[dict] | None = None
    routes: list[dict] | None = None
    log_truncated: bool = False
    pool_capacity: list[int] | None = None   # per replica (topology.py:289-302)
    has_moe: bool = False
    kv_bytes_per_token: int = 0
    af_micro_batches: int = 0
    event_log: np.ndarray | None = None      # fs_event_rec by seq (trace runs only)
    expert_imbalance: list[float] | None = None  # from a moe-ratio log (api.simulate)
    per_request_values: tuple | None = None  # (ttft, tpot, e2e) lists, split_results

    def trace(self):
        """The reference's EventTrace of this run (needs a run with an event log)."""
        from .trace import EventTrace
        if self.event_log is None:
            raise ValueError("this run did not record an event trace")
        return EventTrace(self, self.event_log)

    @property
    def status(self) -> int:
        return int(self.row["status"])

    @property
    def ok(self) -> bool:
        return self.status == 0

    @property
    def iterations(self) -> int:
        return int(self.row["iterations"])

    @property
    def events(self) -> int:
        return int(self.row["events"])

    def error(self) -> Exception | None:
        if self.ok:
            return None
        exc = STATUS_EXCEPTIONS.get(self.status, SimulationError)
        detail = int(self.row["status_detail"])
        if exc.__name__ == "RequestCannotFit" and 0 <= detail < len(self.request_ids):
            return exc(f"request {self.request_ids[detail]} cannot fit its replica's KV pool")
        return exc(f"instance {self.index}: {exc.__name__} (detail {detail})")

    def raise_for_status(self) -> None:
        err = self.error()
        if err is not None:
            raise err

    def completion_order(self) -> list[str]:
        order = np.argsort(self.completion_rank, kind="stable")
        return [self.request_ids[i] for i in order if self.completion_rank[i] >= 0]


def _per_request_columns(low, raw, o: int = 0, n: int | None = None) -> tuple[list, list, list]:
    """ttft / tpot / e2e of every request of the batch (or of requests [o, o+n)) as
    Python floats, in one vectorised pass with the reference's expressions
    (metrics.py:91-100): exact int64 ns differences, then the same IEEE divisions
    Python performs."""
    e = len(low.arrival) if n is None else o + n
    arr = low.arrival[o:e]
    with np.errstate(all="ignore"):
        ttft = (raw.first_ns[o:e] - arr) / 1e9
        e2e = (raw.done_ns[o:e] - arr) / 1e9
        n_out = low.output[o:e].astype(np.int64)
        tpot = (e2e - ttft) / (n_out - 1)
    tp = tpot.tolist()
    for j in np.flatnonzero(n_out <= 1).tolist():
        tp[j] = None
    return ttft.tolist(), tp, e2e.tolist()


def split_results(low, raw, modes: list[str], only: int | None = None):
    """One InstanceResult per instance (views into the batch arrays); `only`: just
    that instance's, returned alone."""
    out = []
    if only is None:
        cols = _per_request_columns(low, raw) if low.n_requests else ([], [], [])
    descs = low.descs
    f = {k: descs[k].tolist() for k in ("req_offset", "n_requests", "replica_offset",
                                        "n_replicas", "total_gpus", "has_moe",
                                        "kv_bytes_per_token", "af_micro_batches")}
    pool = low.replicas["kv_pool_tokens"].tolist()
    for i in (range(low.n_instances) if only is None else (only,)):
        o, n = f["req_offset"][i], f["n_requests"][i]
        ro, nr = f["replica_offset"][i], f["n_replicas"][i]
        if only is None:
            pv = (cols[0][o:o + n], cols[1][o:o + n], cols[2][o:o + n])
        else:
            pv = _per_request_columns(low, raw, o, n)
        res = InstanceResult(
            index=i, row=raw.rows[i], replica_keys=low.replica_keys[i],
            replica_out=raw.replica_out[ro:ro + nr], request_ids=low.request_ids[i],
            arrival_ns=low.arrival[o:o + n], prompt=low.prompt[o:o + n],
            output=low.output[o:o + n], first_token_ns=raw.first_ns[o:o + n],
            done_ns=raw.done_ns[o:o + n], completion_rank=raw.done_rank[o:o + n],
            total_gpus=f["total_gpus"][i], mode=modes[i],
            pool_capacity=pool[ro:ro + nr],
            has_moe=bool(f["has_moe"][i]), kv_bytes_per_token=f["kv_bytes_per_token"][i],
            af_micro_batches=f["af_micro_batches"][i],
            per_request_values=pv)
        if raw.log is not None:
            if raw.log.spec.batch_cap:
                res.batches = raw.log.instance_batches(i)
            if raw.log.spec.route_cap:
                res.routes = raw.log.instance_routes(i)
            res.log_truncated = bool(raw.log.truncated[i])
            if raw.log.spec.event_cap and res.ok and not res.log_truncated:
                res.event_log = raw.log.instance_events(i)
        out.append(res)
    return out[0] if only is not None else out


def _nan_to_none(x: float) -> float | None:
    return None if (x is None or (isinstance(x, float) and math.isnan(x))) else float(x)


def _agg(v) -> dict[str, float] | None:
    if math.isnan(float(v[1])):
        return None
    return {"mean": float(v[0]), "p50": float(v[1]), "p90": float(v[2]), "p99": float(v[3])}


def compute_metrics(result, deployment=None) -> MetricsBundle:
    """MetricsBundle of a device run (reference: metrics.py:81-178).

    `result` is an InstanceResult or the EventTrace `Simulation.run()` returns.
    All reductions were done on the device; per-request values are the
    reference's own expressions over the device's integer timestamps.
    """
    result = getattr(result, "result", result)  # EventTrace -> InstanceResult
    if len(result.request_ids) == 0:
        raise IncompleteTrace("trace contains no requests")  # metrics.py:88-89
    if not result.ok:
        raise IncompleteTrace(str(result.error()))
    row = result.row
    pv = getattr(result, "per_request_values", None)
    if pv is not None:
        per_request = {rid: {"ttft_s": a, "tpot_s": b, "e2e_s": c}
                       for rid, a, b, c in zip(result.request_ids, *pv)}
    else:
        per_request = {}
        for i, rid in enumerate(result.request_ids):
            arr = int(result.arrival_ns[i])
            ttft = (int(result.first_token_ns[i]) - arr) / 1e9
            e2e = (int(result.done_ns[i]) - arr) / 1e9
            n_out = int(result.output[i])
            per_request[rid] = {"ttft_s": ttft,
                                "tpot_s": (e2e - ttft) / (n_out - 1) if n_out > 1 else None,
                                "e2e_s": e2e}
    busy = {}
    for k, o in zip(result.replica_keys, result.replica_out):
        if int(o["steps_executed"]) > 0:
            busy[k] = float(o["busy_fraction"])
    if int(row["af_steps"]) > 0:
        for j, name in enumerate(abi.AF_RESOURCES):
            busy[name] = float(row["af_busy_fraction"][j])
    busy = dict(sorted(busy.items()))
    # expert_imbalance (metrics.py:105-109): [] without MoE; for MoE runs it needs a
    # batch log (run_one / make_simulation record one; simulate() re-runs the MoE
    # instances with one unless expert_imbalance=False, which leaves None here)
    imbalance: list[float] | None = []
    if result.expert_imbalance is not None:
        imbalance = result.expert_imbalance
    elif result.batches is not None:
        for b in result.batches:
            if b["moe_ratio"] is not None:
                imbalance.extend(round(x, 6) for x in b["moe_ratio"])
    elif result.has_moe:
        imbalance = None
    thr = float(row["throughput_tokens_per_s_per_gpu"])
    return MetricsBundle(
        per_request=per_request,
        ttft=_agg(row["ttft"]), tpot=_agg(row["tpot"]), e2e=_agg(row["e2e"]),
        total_tokens=int(row["total_tokens"]), makespan_s=float(row["makespan_s"]),
        total_gpus=result.total_gpus, throughput_tokens_per_s_per_gpu=thr,
        busy_fraction=busy, bubble_fraction=_nan_to_none(float(row["bubble_fraction"])),
        expert_imbalance=imbalance,
        workload_summary={"batch_size": len(result.request_ids),
                          "avg_input_tokens": float(row["avg_input_tokens"]),
                          "avg_output_tokens": float(row["avg_output_tokens"]),
                          "throughput_tokens_per_s_per_gpu": thr})


# -- report formats (metrics.py:181-222) ---------------------------------------------------

def _dominates(a: MetricsBundle, b: MetricsBundle) -> bool:
    """Higher-or-equal throughput and lower-or-equal p90 TPOT, one strictly."""
    ta = a.tpot["p90"] if a.tpot else math.inf
    tb = b.tpot["p90"] if b.tpot else math.inf
    xa, xb = a.throughput_tokens_per_s_per_gpu, b.throughput_tokens_per_s_per_gpu
    return xa >= xb and ta <= tb and (xa > xb or ta < tb)


def pareto_frontier(results: list[tuple[object, MetricsBundle]]) -> list[tuple[object, MetricsBundle]]:
    return [(tag, m) for i, (tag, m) in enumerate(results)
            if not any(_dominates(o, m) for j, (_, o) in enumerate(results) if j != i)]


SUMMARY_CSV_HEADER = [
    "config_hash", "throughput_tokens_per_s_per_gpu",
    "ttft_p50_s", "ttft_p90_s", "ttft_p99_s",
    "tpot_p50_s", "tpot_p90_s", "tpot_p99_s",
    "makespan_s",
]


def summary_csv_row(bundle: MetricsBundle, config_hash: str) -> list[str]:
    def pick(agg, key):
        return repr(agg[key]) if agg else ""
    return [config_hash, repr(bundle.throughput_tokens_per_s_per_gpu),
            pick(bundle.ttft, "p50"), pick(bundle.ttft, "p90"), pick(bundle.ttft, "p99"),
            pick(bundle.tpot, "p50"), pick(bundle.tpot, "p90"), pick(bundle.tpot, "p99"),
            repr(bundle.makespan_s)]
