"""Batched entry points: `simulate(configs)` and `run_one(config)`.

`simulate` is the data-parallel hot path: N config documents (or parsed
DeploymentConfigs) are lowered once and stepped together on the GPU, one
warp per instance; the result is one MetricsBundle -- or the exception the
reference would have raised -- per instance, in input order. This replaces
the reference's per-point loop over `run_one` (cli.py:82-102, 197-237).
"""

from __future__ import annotations

import time

import numpy as np
from dataclasses import dataclass

from .config import DeploymentConfig, parse_config
from .costmodel import check_model_slots_engine
from .engine import Engine, LogSpec, default_engine
from .lower import InstanceSpec, Lowered, lower
from .metrics import InstanceResult, MetricsBundle, compute_metrics, split_results


@dataclass
class Failure:
    """A point that raised: mirrors the sweep's `failed: {Type}: {msg}` rows."""

    exception: Exception

    @property
    def status(self) -> str:
        return f"failed: {type(self.exception).__name__}: {self.exception}"


def instance_spec(config: DeploymentConfig, requests=None) -> InstanceSpec:
    """What `run_one` builds before `make_simulation` (cli.py:84-94). `requests`
    (RequestArrays) replaces the host generation when given (device_workload)."""
    attention_model, grouped_model = config.cost_model.load_models()
    check_model_slots_engine(attention_model, grouped_model)
    return InstanceSpec(
        deployment=config.deployment(),
        requests=requests if requests is not None else config.request_arrays(),
        policy=config.policy,
        af=config.af if config.mode == "af" else None, routing=config.routing, seed=config.seed,
        attention_model=attention_model, grouped_gemm_model=grouped_model)


@dataclass
class BatchRun:
    lowered: Lowered
    results: list[InstanceResult]
    seconds_lower: float
    seconds_device: float


def run_specs(specs: list[InstanceSpec], engine: Engine | None = None,
              log: LogSpec | None = None) -> BatchRun:
    eng = engine or default_engine()
    t0 = time.perf_counter()
    low = lower(specs)
    t1 = time.perf_counter()
    raw = eng.run(low, log=log)
    t2 = time.perf_counter()
    modes = [sp.deployment.mode for sp in specs]
    return BatchRun(low, split_results(low, raw, modes), t1 - t0, t2 - t1)


def device_request_arrays(configs: list[DeploymentConfig], engine: Engine | None = None):
    """Synthetic workloads of `configs` generated on the device in one call
    (fs_generate_workload); None for configs that read a trace file. Raises the
    reference's ValidationError for invalid distribution parameters, per config,
    through the returned list (an Exception entry)."""
    from .config import ValidationError
    from .workload import RequestArrays, WorkloadError, workload_descs
    eng = engine or default_engine()
    out: list = [None] * len(configs)
    idx, wl = [], []
    for i, cfg in enumerate(configs):
        if cfg.trace_path is not None:
            continue
        try:
            workload_descs([cfg.workload])
        except WorkloadError as exc:
            out[i] = ValidationError(str(exc))
            continue
        idx.append(i)
        wl.append(cfg.workload)
    if wl:
        descs = workload_descs(wl)
        arr, pr, ou, _, st = eng.generate_workload(descs)
        for j, i in enumerate(idx):
            if st[j] != 0:
                out[i] = ValidationError(f"workload generation failed (status {int(st[j])})")
                continue
            o, n = int(descs[j]["out_offset"]), int(descs[j]["n_requests"])
            out[i] = RequestArrays([f"r{k}" for k in range(n)], arr[o:o + n].copy(),
                                   pr[o:o + n].astype(np.int64), ou[o:o + n].astype(np.int64))
    return out


def simulate(configs: list, engine: Engine | None = None, base_dir: str = ".",
             device_workload: bool = False) -> list[MetricsBundle | Failure]:
    """Simulate every config on the GPU; per-instance errors become Failure entries.
    device_workload: draw the synthetic request streams on the device too."""
    out: list[MetricsBundle | Failure | None] = [None] * len(configs)
    specs, where = [], []
    parsed: list = [None] * len(configs)
    for i, c in enumerate(configs):
        try:
            parsed[i] = c if isinstance(c, DeploymentConfig) else parse_config(c, base_dir=base_dir)
        except Exception as exc:  # config-time failures (cli.py:229-233)
            out[i] = Failure(exc)
    pre: list = [None] * len(configs)
    if device_workload:
        ok = [i for i in range(len(configs)) if parsed[i] is not None]
        for i, r in zip(ok, device_request_arrays([parsed[i] for i in ok], engine)):
            pre[i] = r
    for i, cfg in enumerate(parsed):
        if cfg is None:
            continue
        try:
            if isinstance(pre[i], Exception):
                raise pre[i]
            specs.append(instance_spec(cfg, requests=pre[i]))
            where.append(i)
        except Exception as exc:  # config-time failures (cli.py:229-233)
            out[i] = Failure(exc)
    if specs:
        run = run_specs(specs, engine)
        for i, res in zip(where, run.results):
            out[i] = compute_metrics(res) if res.ok else Failure(res.error())
    return out


def run_one(config: DeploymentConfig, engine: Engine | None = None) -> dict:
    """Single-instance drop-in for the reference's run_one (cli.py:82-102)."""
    from .orchestrator import make_simulation
    spec = instance_spec(config)
    sim = make_simulation(config.mode, spec.deployment, spec.requests.to_requests(), spec.policy,
                          af=spec.af, routing=spec.routing, seed=spec.seed,
                          attention_model=spec.attention_model,
                          grouped_gemm_model=spec.grouped_gemm_model, engine=engine)
    trace = sim.run()
    return {"config": config, "trace": trace, "metrics": compute_metrics(trace, spec.deployment),
            "config_hash": config.config_hash()}
