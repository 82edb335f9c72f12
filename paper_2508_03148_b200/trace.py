"""Event trace of a device run (reference: core.py:85-129 EventTrace).

The engine records every scheduled event -- the no-op kinds included -- as a
fixed-size `fs_event_rec` at index `seq` of the instance's event array
(include/frontier_b200.h). Every scheduled event is dispatched, and the
reference dispatches in (timestamp, seq) order, so the trace is those
records sorted by (t, seq). This module renders them in the reference's
export format, `timestamp,seq,KIND,canonical_json(payload)` with a sha256
over the body, from the records plus what the host already holds (request
ids and lengths, replica keys, pool capacities, the batch log).

Payloads follow the handlers that schedule them:
  REQUEST_ARRIVAL          base.py:167-177
  BATCH_START              base.py:179-186
  BATCH_COMPLETE           base.py:233-255, af.py:494-505
  PREFILL_COMPLETE         colocated.py:75-83, pd.py:101-108, af.py:518-525
  TOKEN_EMITTED            base.py:188-194, colocated.py:93-97
  REQUEST_COMPLETE         base.py:196-206
  MEMORY_AVAILABLE         base.py:207-217, pd.py:194-205
  KV_CACHE_TRANSFER_START  pd.py:163-177
  KV_CACHE_TRANSFER_DONE   pd.py:181-190
  *_DONE (AF nodes)        af.py:177-194
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass
from enum import Enum
from typing import Any, Iterator

import numpy as np

from . import abi


class EventKind(str, Enum):
    """core.py:38-51 (same names, values and declaration order)."""

    REQUEST_ARRIVAL = "REQUEST_ARRIVAL"
    BATCH_START = "BATCH_START"
    BATCH_COMPLETE = "BATCH_COMPLETE"
    PREFILL_COMPLETE = "PREFILL_COMPLETE"
    MEMORY_AVAILABLE = "MEMORY_AVAILABLE"
    KV_CACHE_TRANSFER_START = "KV_CACHE_TRANSFER_START"
    KV_CACHE_TRANSFER_DONE = "KV_CACHE_TRANSFER_DONE"
    ATTN_COMPUTE_DONE = "ATTN_COMPUTE_DONE"
    A_TO_F_TRANSFER_DONE = "A_TO_F_TRANSFER_DONE"
    FFN_COMPUTE_DONE = "FFN_COMPUTE_DONE"
    F_TO_A_TRANSFER_DONE = "F_TO_A_TRANSFER_DONE"
    TOKEN_EMITTED = "TOKEN_EMITTED"
    REQUEST_COMPLETE = "REQUEST_COMPLETE"


_KINDS = list(EventKind)
assert [k.value for k in _KINDS] == list(abi.EVENT_KINDS)


@dataclass(frozen=True)
class SimEvent:
    """core.py:70-78."""

    timestamp: int
    seq: int
    kind: EventKind
    payload: dict[str, Any]

    def sort_key(self) -> tuple[int, int]:
        return (self.timestamp, self.seq)


def _canonical_payload(payload: dict[str, Any]) -> str:
    return json.dumps(payload, sort_keys=True, separators=(",", ":"))


def _micro_sizes(n: int, m: int) -> list[int]:
    """partition_micro_batches (af.py:244-258) sizes."""
    m_eff = min(m, n)
    if m_eff == 0:
        return []
    base, rem = divmod(n, m_eff)
    return [base + (1 if i < rem else 0) for i in range(m_eff)]


class EventTrace:
    """Append-only record of processed events, in pop order (core.py:85-129).

    Built from a device run: `records` / `lines()` are rendered on first use.
    `result` is the InstanceResult the metrics come from, so
    `compute_metrics(trace, deployment)` works as in the reference.
    """

    def __init__(self, result, events: np.ndarray) -> None:
        self.result = result
        order = np.argsort(events["t"], kind="stable")  # events are indexed by seq
        self._ev = events[order]
        if len(self._ev) and not np.array_equal(np.sort(self._ev["seq"]),
                                                np.arange(len(self._ev))):
            raise RuntimeError("event log is missing sequence numbers")
        self._records: list[SimEvent] | None = None
        self._lines: list[str] | None = None

    def remap_arrival_seq(self, order: list[int]) -> None:
        """Arrivals were simulated in time order; their seq is the caller's list
        index (base.py:167-177): order[j] is the list index of simulated request j."""
        arr = self._ev["kind"] == 0
        self._ev["seq"][arr] = np.asarray(order, dtype=np.int64)[self._ev["a"][arr]]
        self._records = self._lines = None

    # -- reference API -----------------------------------------------------------------
    def __len__(self) -> int:
        return len(self._ev)

    def __iter__(self) -> Iterator[SimEvent]:
        return iter(self.records)

    @property
    def records(self) -> list[SimEvent]:
        if self._records is None:
            self._records = self._render()
        return self._records

    def append(self, event: SimEvent) -> None:
        self.records.append(event)
        self._lines = None

    def lines(self) -> list[str]:
        if self._lines is None:
            self._lines = [f"{ev.timestamp},{ev.seq},{ev.kind.value},{_canonical_payload(ev.payload)}"
                           for ev in self.records]
        return list(self._lines)

    def body_bytes(self) -> bytes:
        body = "\n".join(self.lines())
        if body:
            body += "\n"
        return body.encode("utf-8")

    @property
    def hash(self) -> str:
        return hashlib.sha256(self.body_bytes()).hexdigest()

    def export(self, path: str) -> None:
        """Newline-delimited records plus a trailing `#hash=` footer (core.py:119-126)."""
        body = self.body_bytes()
        digest = hashlib.sha256(body).hexdigest()
        with open(path, "wb") as fh:
            fh.write(body)
            fh.write(f"#hash={digest}\n".encode("utf-8"))

    def events_of_kind(self, kind: EventKind) -> list[SimEvent]:
        return [ev for ev in self.records if ev.kind is kind]

    # -- rendering -------------------------------------------------------------------------
    def _render(self) -> list[SimEvent]:
        res = self.result
        ids = res.request_ids
        prompt = res.prompt.tolist()
        output = res.output.tolist()
        keys = res.replica_keys
        cap = res.pool_capacity
        batches = {b["index"]: b for b in (res.batches or [])}
        # TOKEN_EMITTED lists the batch completing on that replica at that instant
        by_completion = {(b["replica"], b["t_complete"]): b for b in batches.values()}
        moe = res.has_moe
        out: list[SimEvent] = []
        for e in self._ev.tolist():
            t, seq, x, a, b, c, rep, kind = e[0], e[1], e[2], e[3], e[4], e[5], e[6], e[7]
            k = _KINDS[kind]
            if kind == 0:
                p = {"request_id": ids[a], "prompt_tokens": prompt[a],
                     "output_tokens": output[a]}
            elif kind == 1:
                p = {"replica": keys[rep]}
            elif kind == 2:
                bt = batches[a]
                mids = [ids[m] for m in bt["members"]]
                ph = bt["phase"]
                if ph == "af_decode":
                    p = {"replica": keys[rep], "phase": ph, "request_ids": mids,
                         "query_tokens": len(mids), "duration_ns": bt["duration_ns"],
                         "step": bt["af_step"],
                         "micro_batch_sizes": _micro_sizes(len(mids), res.af_micro_batches),
                         "pool": {"used_tokens": bt["pool_used"], "capacity_tokens": cap[rep]}}
                else:
                    qt = sum(prompt[m] for m in bt["members"]) if ph == "prefill" else len(mids)
                    p = {"replica": keys[rep], "phase": ph, "request_ids": mids,
                         "query_tokens": qt, "duration_ns": bt["duration_ns"],
                         "pool": {"used_tokens": bt["pool_used"], "capacity_tokens": cap[rep]}}
                    if moe:
                        p["moe_imbalance"] = [round(v, 6) for v in bt["moe_ratio"]]
            elif kind == 3:
                p = {"request_id": ids[a], "replica": keys[rep]}
            elif kind == 4:
                p = {"replica": keys[rep], "request_id": ids[a], "freed_tokens": b,
                     "headroom_tokens": x}
            elif kind == 5:
                p = {"request_id": ids[a], "src": keys[c], "dst": keys[rep],
                     "bytes": res.kv_bytes_per_token * prompt[a],
                     "reservation": {"tokens": b, "used_after": x, "capacity": cap[rep]}}
            elif kind == 6:
                p = {"request_id": ids[a], "src": keys[c], "dst": keys[rep],
                     "bytes": res.kv_bytes_per_token * prompt[a]}
            elif 7 <= kind <= 10:
                p = {"step": c, "i": a, "k": b, "start_ns": x, "duration_ns": t - x,
                     "resource": abi.AF_RESOURCES[kind - 7]}
            elif kind == 11:
                bt = by_completion[(rep, t)]
                p = {"replica": keys[rep], "request_ids": [ids[m] for m in bt["members"]]}
            else:
                p = {"request_id": ids[a], "tokens_emitted": output[a],
                     "output_tokens": output[a], "prompt_tokens": prompt[a]}
            out.append(SimEvent(t, seq, k, p))
        return out
