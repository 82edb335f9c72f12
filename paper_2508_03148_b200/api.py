"""Batched entry points: `simulate(configs)` and `run_one(config)`.

`simulate` is the data-parallel hot path: N config documents (or parsed
DeploymentConfigs) are lowered once and stepped together on the GPU, one
warp per instance; the result is one MetricsBundle -- or the exception the
reference would have raised -- per instance, in input order. This replaces
the reference's per-point loop over `run_one` (cli.py:82-102, 197-237).
"""

from __future__ import annotations

import gc
import math
import time
from contextlib import contextmanager

import numpy as np
from dataclasses import dataclass

from .config import DeploymentConfig, parse_config, parse_many
from .distributed import gather_rows, lpt_shards, merge_shards
from .costmodel import check_model_slots_engine
from . import abi
from .engine import Engine, LogSpec, default_engine
from .lower import InstanceSpec, Lowered, check_spec, lower
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
    spec = InstanceSpec(
        deployment=config.deployment(),
        requests=requests if requests is not None else config.request_arrays(),
        policy=config.policy,
        af=config.af if config.mode == "af" else None, routing=config.routing, seed=config.seed,
        attention_model=attention_model, grouped_gemm_model=grouped_model)
    check_spec(spec)
    return spec


class BatchRun:
    """A device run of lowered instances: `results` (one InstanceResult per
    instance) is built on first access -- metrics_many reads the lowered and raw
    columns directly and never needs it."""

    def __init__(self, lowered: Lowered, raw, modes: list[str], seconds_lower: float,
                 seconds_device: float):
        self.lowered, self.raw, self.modes = lowered, raw, modes
        self.seconds_lower, self.seconds_device = seconds_lower, seconds_device
        self._results: list[InstanceResult] | None = None

    @property
    def results(self) -> list[InstanceResult]:
        if self._results is None:
            self._results = split_results(self.lowered, self.raw, self.modes)
        return self._results


def run_specs(specs: list[InstanceSpec], engine: Engine | None = None,
              log: LogSpec | None = None) -> BatchRun:
    eng = engine or default_engine()
    t0 = time.perf_counter()
    low = lower(specs)
    t1 = time.perf_counter()
    raw = eng.run(low, log=log)
    t2 = time.perf_counter()
    modes = [sp.deployment.mode for sp in specs]
    return BatchRun(low, raw, modes, t1 - t0, t2 - t1)


def device_request_arrays(configs: list[DeploymentConfig], engine: Engine | None = None):
    """Synthetic workloads of `configs` generated on the device in one call
    (fs_generate_workload); None for configs that read a trace file. Raises the
    reference's ValidationError for invalid distribution parameters, per config,
    through the returned list (an Exception entry)."""
    from .config import ValidationError
    from .lower import shared_ids
    from .workload import RequestArrays, WorkloadError, workload_descs
    eng = engine or default_engine()
    out: list = [None] * len(configs)
    idx, wl = [], []
    bad: dict = {}  # distribution objects -> validation error (checked once per template)
    for i, cfg in enumerate(configs):
        if cfg.trace_path is not None:
            continue
        w = cfg.workload
        key = (id(w.arrival), id(w.prompt_len), id(w.output_len), w.num_requests)
        if key not in bad:
            try:
                w.validate()
                bad[key] = None
            except WorkloadError as exc:
                bad[key] = ValidationError(str(exc))
        if bad[key] is not None:
            out[i] = bad[key]
            continue
        idx.append(i)
        wl.append(w)
    if wl:
        descs = workload_descs(wl)
        arr, pr, ou, _, st = eng.generate_workload(descs)
        pr = pr.astype(np.int64)
        ou = ou.astype(np.int64)
        offs = descs["out_offset"].tolist()
        ns = descs["n_requests"].tolist()
        for j, i in enumerate(idx):
            if st[j] != 0:
                out[i] = ValidationError(f"workload generation failed (status {int(st[j])})")
                continue
            o, n = offs[j], ns[j]
            # ids r0..r{n-1}: synthetic arrivals are non-decreasing, so generation order
            # is request order (workload_descs); views into the generated arrays
            out[i] = RequestArrays(shared_ids(n), arr[o:o + n], pr[o:o + n], ou[o:o + n])
    return out


def _metrics_or_failure(res: InstanceResult) -> MetricsBundle | Failure:
    """compute_metrics, or the exception the reference would raise, as a Failure."""
    if not res.ok:
        return Failure(res.error())
    try:
        return compute_metrics(res)
    except Exception as exc:  # IncompleteTrace (e.g. no requests), metrics.py:115-121
        return Failure(exc)


_HOSTPY: list = []


def _hostpy():
    """csrc/fs_hostpy.c (per-request dictionaries in C), or None if not built."""
    if not _HOSTPY:
        from .native import load_hostpy
        _HOSTPY.append(load_hostpy())
    return _HOSTPY[0]


def metrics_many(run: BatchRun) -> list[MetricsBundle | Failure]:
    """[_metrics_or_failure(r) for r in run.results], built from the lowered and raw
    columns read once as Python values (numpy scalar access per field, and one
    InstanceResult per instance, are the cost of compute_metrics at sweep scale);
    identical bundles (tests/test_batch_host.py). InstanceResults are used only for
    failed instances and when a run carries logs or attached expert imbalance."""
    from .metrics import IncompleteTrace, _per_request_columns
    raw, low = run.raw, run.lowered
    if raw is None:
        return [_metrics_or_failure(r) for r in run.results]
    n_inst = low.n_instances
    if n_inst == 0:
        return []
    have = run._results  # InstanceResults, when something already built them
    if have is None and raw.log is not None:
        have = run.results  # batch logs: expert imbalance per instance
    rows, rep = raw.rows, raw.replica_out
    col = {f: rows[f].tolist() for f in ("status", "total_tokens", "makespan_s",
                                        "throughput_tokens_per_s_per_gpu", "bubble_fraction",
                                        "avg_input_tokens", "avg_output_tokens", "af_steps",
                                        "ttft", "tpot", "e2e", "af_busy_fraction")}
    rbusy, rsteps = rep["busy_fraction"].tolist(), rep["steps_executed"].tolist()
    descs = low.descs
    roff = descs["replica_offset"].tolist()
    qoff, qn = descs["req_offset"].tolist(), descs["n_requests"].tolist()
    gpus, moe = descs["total_gpus"].tolist(), descs["has_moe"].tolist()
    ttft_c, tpot_c, e2e_c = (_per_request_columns(low, raw) if low.n_requests
                             else ([], [], []))
    nan = math.isnan
    host = _hostpy()

    def agg(v):
        return None if nan(v[1]) else {"mean": v[0], "p50": v[1], "p90": v[2], "p99": v[3]}

    out = []
    for i in range(n_inst):
        if col["status"][i] != 0:
            r = have[i] if have is not None else split_results(low, raw, run.modes, only=i)
            out.append(Failure(r.error()))
            continue
        ids = low.request_ids[i]
        if len(ids) == 0:
            out.append(Failure(IncompleteTrace("trace contains no requests")))
            continue
        o, n = qoff[i], qn[i]
        if host is not None and type(ids) is list:
            per_request = host.per_request(ids, ttft_c, tpot_c, e2e_c, o)
        else:
            per_request = {rid: {"ttft_s": a, "tpot_s": b, "e2e_s": c}
                           for rid, a, b, c in zip(ids, ttft_c[o:o + n], tpot_c[o:o + n],
                                                   e2e_c[o:o + n])}
        busy = {}
        ro = roff[i]
        for j, k in enumerate(low.replica_keys[i]):
            if rsteps[ro + j] > 0:
                busy[k] = rbusy[ro + j]
        if col["af_steps"][i] > 0:
            for j, name in enumerate(abi.AF_RESOURCES):
                busy[name] = col["af_busy_fraction"][i][j]
        busy = dict(sorted(busy.items()))
        r = have[i] if have is not None else None
        if r is not None and r.expert_imbalance is not None:
            imbalance = r.expert_imbalance
        elif r is not None and r.batches is not None:
            imbalance = [round(x, 6) for b in r.batches if b["moe_ratio"] is not None
                         for x in b["moe_ratio"]]
        else:
            imbalance = None if moe[i] else []
        thr = col["throughput_tokens_per_s_per_gpu"][i]
        bub = col["bubble_fraction"][i]
        out.append(MetricsBundle(
            per_request=per_request, ttft=agg(col["ttft"][i]), tpot=agg(col["tpot"][i]),
            e2e=agg(col["e2e"][i]), total_tokens=col["total_tokens"][i],
            makespan_s=col["makespan_s"][i], total_gpus=gpus[i],
            throughput_tokens_per_s_per_gpu=thr, busy_fraction=busy,
            bubble_fraction=None if nan(bub) else bub, expert_imbalance=imbalance,
            workload_summary={"batch_size": len(ids),
                              "avg_input_tokens": col["avg_input_tokens"][i],
                              "avg_output_tokens": col["avg_output_tokens"][i],
                              "throughput_tokens_per_s_per_gpu": thr}))
    return out


def attach_expert_imbalance(specs: list[InstanceSpec], results: list[InstanceResult],
                            engine: Engine | None = None) -> None:
    """Fill InstanceResult.expert_imbalance for the successful MoE instances: they are
    simulated once more with a batch log sized exactly from the first run's counts
    (batches = iterations, members = total_tokens, moe values = L per prefill/decode
    batch); the values arrive from the device already as round(x, 6)."""
    idx = [i for i, (sp, r) in enumerate(zip(specs, results))
           if r.ok and sp.deployment.model.moe is not None]
    if not idx:
        return
    eng = engine or default_engine()
    sub = [specs[i] for i in idx]
    rows = [results[i].row for i in idx]
    nb = [int(r["iterations"]) for r in rows]
    nm = [int(r["total_tokens"]) for r in rows]
    ne = [(int(r["prefill_batches"]) + int(r["decode_batches"])) * sp.deployment.model.num_layers
          for r, sp in zip(rows, sub)]
    spec = LogSpec(batch_cap=max(nb), member_cap=max(nm), moe_cap=max(max(ne), 1))
    raw = eng.run(lower(sub), log=spec, log_sizes={"batch": nb, "member": nm, "moe": ne})
    for j, i in enumerate(idx):
        if raw.log.truncated[j]:
            raise RuntimeError(f"instance {i}: moe-ratio log truncated on the re-run")
        results[i].expert_imbalance = raw.log.moe_imbalance(j)


# ---- multi-GPU sharding ----------------------------------------------------

def process_group(distributed: bool | None):
    """torch.distributed when it should shard (initialised, world > 1), else None."""
    if distributed is False:
        return None
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover
        dist = None
    if dist is not None and dist.is_available() and dist.is_initialized() \
            and dist.get_world_size() > 1:
        return dist
    if distributed:
        raise RuntimeError("distributed=True needs an initialised torch.distributed group")
    return None


def config_cost(config: DeploymentConfig) -> int:
    """Host estimate of an instance's device time for LPT sharding: iterations are
    ~ output tokens, each costs ~ L layers, MoE layers route T x E keys
    (lower._estimate_cost's shape, from the config alone -- no workload drawn)."""
    m = config.model
    wl = config.workload
    if wl is None:
        out_tokens = 256 * 64
    else:
        o = wl.output_len
        mean = (o.value if o.kind == "fixed" else (o.lo + o.hi) / 2 if o.kind == "uniform"
                else min(max(math.exp(o.mu + o.sigma * o.sigma / 2), o.lo), o.hi))
        out_tokens = wl.num_requests * (mean + 1)
    work = out_tokens * m.num_layers
    if m.moe is not None:
        work *= 1 + m.moe.num_experts / 4
    return int(work)


def parse_all(configs: list, base_dir: str = ".") -> list:
    """Parsed DeploymentConfigs, or Failure entries for the points that fail to
    parse (cli.py:229-233); documents that differ only in their seeds share one
    parse and validation (config.parse_many)."""
    out = list(configs)
    idx = [i for i, c in enumerate(configs) if not isinstance(c, Failure)]
    for i, p in zip(idx, parse_many([configs[i] for i in idx], base_dir, on_error=Failure)):
        out[i] = p
    return out


def shard_plan(configs: list, world: int, base_dir: str = "."):
    """(parsed configs or Failures, LPT shards over ranks): same on every rank."""
    parsed = parse_all(configs, base_dir)
    costs = [config_cost(p) if isinstance(p, DeploymentConfig) else 0 for p in parsed]
    return parsed, lpt_shards(costs, world)


def _simulate_sharded(dist, configs, engine, base_dir, device_workload, expert_imbalance):
    rank, world = dist.get_rank(), dist.get_world_size()
    parsed, shards = shard_plan(configs, world, base_dir)
    mine = shards[rank]
    local = simulate([parsed[i] for i in mine], engine=engine, base_dir=base_dir,
                     device_workload=device_workload, expert_imbalance=expert_imbalance,
                     distributed=False)
    gathered: list = [None] * world
    dist.all_gather_object(gathered, local)  # bundles carry per-request dicts: pickled
    out: list = [None] * len(configs)
    for idx, res in zip(shards, gathered):
        for i, r in zip(idx, res):
            out[i] = r
    return out


@contextmanager
def _gc_paused():
    """A batch allocates a few objects per request and instance and frees none of
    them until it returns; the cyclic collector's passes over that growing heap
    are pure overhead here (reference counting still frees everything)."""
    was = gc.isenabled()
    gc.disable()
    try:
        yield
    finally:
        if was:
            gc.enable()


def simulate(configs: list, engine: Engine | None = None, base_dir: str = ".",
             device_workload: bool = False, expert_imbalance: bool = True,
             distributed: bool | None = None) -> list[MetricsBundle | Failure]:
    """Simulate every config on the GPU; per-instance errors become Failure entries.
    device_workload: draw the synthetic request streams on the device too.
    expert_imbalance: fill MetricsBundle.expert_imbalance for MoE configs (a second
    device pass over them, see attach_expert_imbalance); False leaves it None --
    the sweep's CSV and frontier do not use it.
    distributed: with torch.distributed initialised (world > 1; None = auto), every
    rank simulates its LPT shard on its own GPU and the results are all-gathered,
    so each rank returns the full list in input order."""
    dist = process_group(distributed)
    if dist is not None:
        return _simulate_sharded(dist, configs, engine, base_dir, device_workload,
                                 expert_imbalance)
    with _gc_paused():
        return _simulate_local(configs, engine, base_dir, device_workload, expert_imbalance)


PIPELINE_MIN = 256  # instances below which simulate() runs one batch


def _pipeline_groups(parsed: list, pre: list) -> list[list[int]]:
    """simulate()'s batches, in launch order: the MoE configs first (the longest device
    wave), then the rest, so building and lowering the second batch on the host runs
    while the first is on the GPU, and metrics of the first are built while the second
    runs. Small or single-family inputs stay one batch. Instances are independent, so
    the split changes no result (tests/test_gpu_parity.py)."""
    ok = [i for i, c in enumerate(parsed) if c is not None and not isinstance(pre[i], Exception)]
    if len(ok) < PIPELINE_MIN:
        return [ok]
    moe = [i for i in ok if parsed[i].model.moe is not None]
    rest = [i for i in ok if parsed[i].model.moe is None]
    return [g for g in (moe, rest) if g]


def _simulate_local(configs, engine, base_dir, device_workload, expert_imbalance):
    out: list[MetricsBundle | Failure | None] = [None] * len(configs)
    parsed: list = [None] * len(configs)
    for i, p in enumerate(parse_all(configs, base_dir)):
        if isinstance(p, Failure):
            out[i] = p
        else:
            parsed[i] = p
    pre: list = [None] * len(configs)
    if device_workload:
        ok = [i for i in range(len(configs)) if parsed[i] is not None]
        for i, r in zip(ok, device_request_arrays([parsed[i] for i in ok], engine)):
            pre[i] = r
    for i, r in enumerate(pre):
        if isinstance(r, Exception):
            out[i] = Failure(r)
    eng = engine or default_engine()
    launched = []  # (engine, lowered, specs, where), each batch on its own engine
    for g, idx in enumerate(_pipeline_groups(parsed, pre)):
        specs, where = [], []
        for i in idx:
            try:
                specs.append(instance_spec(parsed[i], requests=pre[i]))
                where.append(i)
            except Exception as exc:  # config-time failures (cli.py:229-233)
                out[i] = Failure(exc)
        if not specs:
            continue
        e = eng if g == 0 else eng.peer()
        t0 = time.perf_counter()
        low = lower(specs)
        e.stage(low)
        e.launch()
        launched.append((e, low, specs, where, time.perf_counter() - t0))
    for e, low, specs, where, t_low in launched:
        t1 = time.perf_counter()
        raw = e.fetch(low)
        run = BatchRun(low, raw, [sp.deployment.mode for sp in specs], t_low,
                       time.perf_counter() - t1)
        if expert_imbalance:
            attach_expert_imbalance(specs, run.results, e)
        for i, m in zip(where, metrics_many(run)):
            out[i] = m
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


# ---- rows-only path: the sweep driver's fixed-size metric rows --------------------------

@dataclass
class SweepRows:
    """Metric rows of a batch of configs, in input order: `rows` (fs_metric_row) for
    every instance that reached the device, `failed` = {index: "Type: msg"} for the
    others (their rows are zero), `config_hash` and `total_gpus` per instance (None
    if it never reached the device)."""

    rows: np.ndarray
    failed: dict[int, str]
    config_hash: list[str | None]
    total_gpus: list[int | None]

    def bundle(self, i: int) -> MetricsBundle | None:
        return None if i in self.failed else bundle_from_row(self.rows[i], self.total_gpus[i])


def simulate_rows(configs: list, engine: Engine | None = None, base_dir: str = ".",
                  device_workload: bool = False, distributed: bool | None = None) -> SweepRows:
    """simulate() reduced to the fixed-size metric rows, which is all a sweep's CSV and
    frontier read. Multi-GPU: LPT shards per rank, one all-gather of the rows over
    the process group (NCCL on the B200 box) plus the failure texts."""
    with _gc_paused():
        return _simulate_rows(configs, engine, base_dir, device_workload, distributed)


def _simulate_rows(configs, engine, base_dir, device_workload, distributed) -> SweepRows:
    dist = process_group(distributed)
    world, rank = (dist.get_world_size(), dist.get_rank()) if dist is not None else (1, 0)
    parsed, shards = shard_plan(configs, world, base_dir)
    mine = shards[rank]
    specs, where, failed, hashes = [], [], {}, {}
    pre: dict[int, object] = {}
    if device_workload:
        ok = [i for i in mine if isinstance(parsed[i], DeploymentConfig)]
        for i, r in zip(ok, device_request_arrays([parsed[i] for i in ok], engine)):
            pre[i] = r
    for i in mine:
        p = parsed[i]
        try:
            if isinstance(p, Failure):
                raise p.exception
            if isinstance(pre.get(i), Exception):
                raise pre[i]
            sp = instance_spec(p, requests=pre.get(i))
            specs.append(sp)
            where.append(i)
            hashes[i] = (p.config_hash(), sp.deployment.total_gpus)
        except Exception as exc:
            failed[i] = f"{type(exc).__name__}: {exc}"
    local = np.zeros(len(mine), dtype=abi.METRIC_ROW)
    if specs:
        run = run_specs(specs, engine)
        pos = {i: j for j, i in enumerate(mine)}
        for i, res in zip(where, run.results):
            local[pos[i]] = res.row
            if not res.ok:
                failed[i] = f"{type(res.error()).__name__}: {res.error()}"
            elif len(res.request_ids) == 0:
                failed[i] = "IncompleteTrace: trace contains no requests"
    if dist is None:
        rows = merge_shards(shards, [local], len(configs))
        meta = [(failed, hashes)]
    else:
        rows = merge_shards(shards, gather_rows(local, world, _row_device()), len(configs))
        meta: list = [None] * world
        dist.all_gather_object(meta, (failed, hashes))
    all_failed, all_hash = {}, {}
    for f, h in meta:
        all_failed.update(f)
        all_hash.update(h)
    n = len(configs)
    return SweepRows(rows, dict(sorted(all_failed.items())),
                     [all_hash[i][0] if i in all_hash else None for i in range(n)],
                     [all_hash[i][1] if i in all_hash else None for i in range(n)])


def _row_device():
    """Where gather_rows stages its buffers: this rank's GPU under NCCL, host for gloo."""
    import torch
    import torch.distributed as dist
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return None


def bundle_from_row(row: np.void, total_gpus: int) -> MetricsBundle:
    """The aggregate part of a MetricsBundle from its metric row (what summary_csv_row
    and pareto_frontier read); per_request / busy / expert_imbalance are not in a row."""
    from .metrics import _agg, _nan_to_none
    thr = float(row["throughput_tokens_per_s_per_gpu"])
    return MetricsBundle(
        per_request={}, ttft=_agg(row["ttft"]), tpot=_agg(row["tpot"]), e2e=_agg(row["e2e"]),
        total_tokens=int(row["total_tokens"]), makespan_s=float(row["makespan_s"]),
        total_gpus=total_gpus, throughput_tokens_per_s_per_gpu=thr, busy_fraction={},
        bubble_fraction=_nan_to_none(float(row["bubble_fraction"])), expert_imbalance=None,
        workload_summary={"batch_size": int(row["n_requests"]),
                          "avg_input_tokens": float(row["avg_input_tokens"]),
                          "avg_output_tokens": float(row["avg_output_tokens"]),
                          "throughput_tokens_per_s_per_gpu": thr})
