"""Serving workflows (reference: pkg/src/frontier_sim/orchestrator/).

`make_simulation(mode, deployment, requests, policy, ...)` keeps the
reference's signature (orchestrator/__init__.py:43-50, base.py:71-81); the
returned object's `run()` executes the whole per-iteration event loop on the
GPU engine and returns the run's `EventTrace` (trace.py: the reference's
records, lines, sha256 hash and export, rendered from the device's event
log), which `compute_metrics` consumes. Requests passed in are updated in
place with their final lifecycle (tokens emitted, COMPLETE, state
timestamps), as the reference's handlers leave them.
"""

from __future__ import annotations

from .cluster import SchedulerPolicy
from .costmodel import as_learned_model, check_model_slots_engine
from .engine import Engine, LogSpec, default_engine
from .errors import RequestCannotFit, SimulationError  # noqa: F401  (re-exported)
from .lower import InstanceSpec, lower
from .metrics import InstanceResult, split_results
from .specs import AfPipelineConfig, RoutingPolicySpec
from .trace import EventTrace
from .topology import Deployment
from .workload import Request, RequestArrays, RequestState, arrays_from_requests

__all__ = ["AfPipelineConfig", "RoutingPolicySpec", "make_simulation", "Simulation",
           "ColocatedSimulation", "PdSimulation", "AfSimulation", "SimulationError",
           "RequestCannotFit", "detail_log_spec"]


def detail_log_spec(spec: InstanceSpec, routes: bool = False, events: bool = False) -> LogSpec:
    """Log capacities large enough for one instance's full batch log (and event trace).

    Every batch emits at least one token and every member emits exactly one,
    so both the batch count and the membership total are bounded by the
    output-token total. Events: N arrivals, PREFILL_COMPLETE, REQUEST_COMPLETE,
    two MEMORY_AVAILABLE and two KV-transfer events per request; per batch one
    BATCH_COMPLETE and one TOKEN_EMITTED; one BATCH_START per kick (<= one per
    arrival, batch completion and transfer completion); 4mL - m node events per
    AF step.
    """
    tokens = int(spec.requests.output.sum()) + 1
    model = spec.deployment.model
    L = model.num_layers
    moe = model.moe is not None
    log = LogSpec(batch_cap=tokens, member_cap=tokens, moe_cap=tokens * L if moe else 0)
    if events:
        n = len(spec.requests.output)
        per_step = 4 * spec.af.micro_batches * L if (spec.af and spec.deployment.mode == "af") else 0
        log.event_cap = 10 * n + tokens * (3 + per_step) + 16
    if routes and moe:
        m = spec.af.micro_batches if (spec.af and spec.deployment.mode == "af") else 1
        log.route_cap = tokens * L * max(1, m)
        log.counts_cap = log.route_cap * model.moe.num_experts
    return log


class Simulation:
    """One simulation instance executed on the device engine."""

    def __init__(self, mode: str, deployment: Deployment, requests: list[Request],
                 policy: SchedulerPolicy, af: AfPipelineConfig | None = None,
                 routing: RoutingPolicySpec | None = None, seed: int = 0,
                 attention_model=None, grouped_gemm_model=None, max_events: int | None = None,
                 engine: Engine | None = None, log_routes: bool = False) -> None:
        if mode not in ("colocated", "pd", "af"):
            raise ValueError(f"unknown mode {mode!r}")
        policy.validate()
        if mode == "af":
            (af or AfPipelineConfig()).validate()
        attention_model = as_learned_model(attention_model)
        grouped_gemm_model = as_learned_model(grouped_gemm_model)
        check_model_slots_engine(attention_model, grouped_gemm_model)
        self.mode = mode
        self.deployment = deployment
        self.requests = list(requests)
        # The engine consumes arrivals in time order; equal times keep list order,
        # which is the reference's dispatch order (seq = list index, base.py:167-177).
        self._order = sorted(range(len(self.requests)),
                             key=lambda i: self.requests[i].arrival_time)
        self.request_arrays: RequestArrays = arrays_from_requests(
            [self.requests[i] for i in self._order])
        self.spec = InstanceSpec(
            deployment=deployment, requests=self.request_arrays, policy=policy,
            af=af if mode == "af" else None, routing=routing or RoutingPolicySpec(), seed=seed,
            attention_model=attention_model, grouped_gemm_model=grouped_gemm_model,
            max_events=50_000_000 if max_events is None else max_events)
        self._engine = engine
        self.log_routes = log_routes
        self.result: InstanceResult | None = None

    def run(self) -> EventTrace:
        """Simulate on the device; returns the EventTrace (base.py:220-229)."""
        eng = self._engine or default_engine()
        low = lower([self.spec])
        raw = eng.run(low, log=detail_log_spec(self.spec, routes=self.log_routes, events=True))
        res = split_results(low, raw, [self.mode])[0]
        self.result = res
        self._update_requests(res)
        res.raise_for_status()
        trace = res.trace()
        if self._order != list(range(len(self._order))):
            trace.remap_arrival_seq(self._order)
        return trace

    def _update_requests(self, res: InstanceResult) -> None:
        for i, req in enumerate(self.requests[j] for j in self._order):
            done = int(res.done_ns[i])
            if done >= 0:
                req.tokens_emitted = req.output_tokens
                req.state = RequestState.COMPLETE
                req.state_times[RequestState.COMPLETE.value] = done
            first = int(res.first_token_ns[i])
            if first >= 0:
                req.state_times[RequestState.PREFILL_COMPLETE.value] = first


def make_simulation(mode, deployment, requests, policy, af=None, **kwargs) -> Simulation:
    return Simulation(mode, deployment, requests, policy, af=af, **kwargs)


def ColocatedSimulation(deployment, requests, policy, **kwargs) -> Simulation:  # noqa: N802
    return Simulation("colocated", deployment, requests, policy, **kwargs)


def PdSimulation(deployment, requests, policy, **kwargs) -> Simulation:  # noqa: N802
    return Simulation("pd", deployment, requests, policy, **kwargs)


def AfSimulation(deployment, requests, policy, af=None, **kwargs) -> Simulation:  # noqa: N802
    return Simulation("af", deployment, requests, policy, af=af, **kwargs)
