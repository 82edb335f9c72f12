"""Binding for the reference package: run its own config objects on the B200 engine.

This is the module INTEGRATION.md has a maintainer add to `frontier_sim`
(as `frontier_sim/gpu.py`). Every function takes the reference's objects as
they come out of `frontier_sim.config.parse_config` (DeploymentConfig,
Deployment, Request, SchedulerPolicy, AfPipelineConfig, RoutingPolicySpec,
LearnedOperatorModel) -- or this package's mirrors of them, which have the
same fields -- and returns what the reference's functions return:

  make_simulation(...)  orchestrator/__init__.py:43-50 -> object whose run()
                        returns the EventTrace (base.py:220-229)
  run_one(config)       cli.py:82-102 -> {config, trace, metrics, config_hash}
  run_batch(configs)    [run_one(c)["metrics"] for c in configs], one device call;
                        a point that raises yields the exception (cli.py:229-233)

`engine` is an Engine (or anything with the same `run(lowered, log=...)`),
default: this process's engine on LOCAL_RANK's device.
"""

from __future__ import annotations

from .api import Failure, run_specs
from .costmodel import as_learned_model, check_model_slots_engine
from .lower import InstanceSpec
from .metrics import compute_metrics
from .orchestrator import Simulation
from .workload import arrays_from_requests


def make_simulation(mode, deployment, requests, policy, af=None, *, engine=None,
                    **kwargs) -> Simulation:
    """orchestrator.make_simulation with the same arguments (routing, seed,
    attention_model, grouped_gemm_model, max_events)."""
    return Simulation(mode, deployment, requests, policy, af=af, engine=engine, **kwargs)


def _models(config):
    att, gg = config.cost_model.load_models()       # config.py:110-119
    return as_learned_model(att), as_learned_model(gg)


def run_one(config, engine=None) -> dict:
    """cli.run_one (cli.py:82-102) on the device."""
    deployment = config.deployment()
    att, gg = _models(config)
    sim = make_simulation(config.mode, deployment, config.requests(), config.policy,
                          af=config.af, routing=config.routing, seed=config.seed,
                          attention_model=att, grouped_gemm_model=gg, engine=engine)
    trace = sim.run()
    return {"config": config, "trace": trace, "metrics": compute_metrics(trace, deployment),
            "config_hash": config.config_hash()}


def spec_of(config) -> InstanceSpec:
    """What run_one builds before make_simulation, as one InstanceSpec."""
    att, gg = _models(config)
    check_model_slots_engine(att, gg)
    reqs = sorted(config.requests(), key=lambda r: r.arrival_time)
    return InstanceSpec(deployment=config.deployment(), requests=arrays_from_requests(reqs),
                        policy=config.policy, af=config.af if config.mode == "af" else None,
                        routing=config.routing, seed=config.seed, attention_model=att,
                        grouped_gemm_model=gg)


def run_batch(configs, engine=None) -> list:
    """MetricsBundle (or the exception the reference raises) per config, in order;
    all points simulated in one batched device call."""
    out: list = [None] * len(configs)
    specs, where = [], []
    for i, c in enumerate(configs):
        try:
            specs.append(spec_of(c))
            where.append(i)
        except Exception as exc:  # config-time failures (cli.py:229-233)
            out[i] = exc
    if specs:
        from .api import _metrics_or_failure, attach_expert_imbalance
        run = run_specs(specs, engine)
        attach_expert_imbalance(specs, run.results, engine)
        for i, res in zip(where, run.results):
            m = _metrics_or_failure(res)
            out[i] = m.exception if isinstance(m, Failure) else m
    return out
