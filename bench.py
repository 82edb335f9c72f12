"""Benchmark: simulated iterations/s over the C5 config sweep (BASELINE.json metric).

A *step* is one pass of the hot path over one batch of synthetic input: the
whole 4,096-instance C5 design-space sweep (64 configs x 64 trace seeds, 64
requests each: SURVEY.md section 8(d)) simulated to completion on the GPU,
metric rows included. An *iteration* is one BATCH_COMPLETE event (prefill
batch, decode step or AF step), counted by the engine.

  value  device-resident inputs (fs_stage once, fs_launch_async per step),
         CUDA events on the launch stream, L2 flushed between steps (outside
         the events), max over ranks; whole-job iterations / time.
  e2e    the drop-in C-ABI call fs_run_batch with HOST buffers each step:
         H2D of descriptors + request SoA, both kernels, D2H of metric rows,
         replica rows and per-request times, wall clock.

Multi-GPU (torchrun): one process per GPU.
  --scaling weak (default): each rank simulates its own 4,096 instances
         (disjoint seeds), then one NCCL all-gather of the fixed-size metric rows.
  --scaling strong: ONE 4,096-instance sweep LPT-sharded over the ranks by
         api.config_cost (the product path's sharding, api.shard_plan); e2e
         includes the NCCL all-gather of the rows every step. `--impl reference` times the CPU port of the
reference path (oracle/fs_oracle.c, all host threads) on a bounded sample of
the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "simulated iterations/sec over config sweep"
UNIT = "iterations/s"
SEED_STRIDE = 1_000_000


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seeds", type=int, default=64, help="trace seeds per config (64 -> 4096)")
    ap.add_argument("--requests", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c2", action="store_true", help="skip the C2 attention-cost kernel leg")
    ap.add_argument("--no-api", action="store_true", help="skip the simulate() end-to-end leg")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the per-config (C1/C3/C4) batches")
    ap.add_argument("--cpu-sample-seeds", type=int, default=8,
                    help="seeds per config of the main arm's cpu_baseline sample")
    ap.add_argument("--reference-seeds", type=int, default=None,
                    help="seeds per config the reference arm times (default: --seeds, the "
                         "same workload as the GPU arm)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_docs(rank: int, n_seeds: int, n_requests: int):
    from paper_2508_03148_b200 import workloads as W
    return W.c5_sweep(n_seeds=n_seeds, n_requests=n_requests, seed_base=1000 + SEED_STRIDE * rank)


def lower_docs(docs):
    from paper_2508_03148_b200.api import instance_spec
    from paper_2508_03148_b200.config import parse_many
    from paper_2508_03148_b200.lower import lower
    return lower([instance_spec(c) for c in parse_many(docs)])


def routing_peak():
    """The routing core's measured peak on this GPU model (scripts/micro/philox_peak.cu:
    Philox4x64-10 blocks -> 32-bit keys -> top-3 of 8 -> tally, committed under
    profiles/): keys/s of the rolled-loop code sim_kernel runs, at 8 warps per SM
    (its occupancy) and the best over occupancies, and of the unrolled variant."""
    path = os.path.join(ROOT, "profiles", "philox_peak_r2.json")
    try:
        rows = [json.loads(l) for l in open(path) if l.startswith('{"kernel"')]
    except Exception:
        return None
    rolled8 = [r["G_keys_per_s"] for r in rows if r["kernel"] == "rolled" and r["warps_per_sm"] == 8]
    rolled = [r["G_keys_per_s"] for r in rows if r["kernel"] == "rolled"]
    unrolled = [r["G_keys_per_s"] for r in rows if r["kernel"].startswith("unrolled")]
    if not rolled8:
        return None
    return {"rolled_8_warps_per_sm": rolled8[0] * 1e9, "rolled_best": max(rolled) * 1e9,
            "unrolled_best": max(unrolled) * 1e9, "source": "profiles/philox_peak_r2.json"}


def imad_wide_rate():
    """Measured IMAD.WIDE.U32 lane-ops per clock per SM (scripts/micro/imad_rates.cu)."""
    try:
        for line in open(os.path.join(ROOT, "profiles", "imad_rates_r2.json")):
            r = json.loads(line)
            if r.get("op") == "imad_wide32":
                return float(r["ops_per_clk_per_sm"])
    except Exception:
        pass
    return None


def cpu_count() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_oracle_sample(n_requests: int, sample_seeds: int, threads: int, rank: int = 0):
    """CPU port of the reference path on all 64 configs x `sample_seeds` seeds."""
    from oracle import oracle
    docs = workload_docs(rank, sample_seeds, n_requests)
    low = lower_docs(docs)
    oracle.load()
    t0 = time.perf_counter()
    res = oracle.run(low, threads=threads)
    dt = time.perf_counter() - t0
    its = int(res.rows["iterations"].sum())
    return its, dt, len(docs)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        return False

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for name, v in zip(names, s[4:8]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_summary(kernel: str) -> dict:
    """`kernel`'s entry in the committed ncu --set full summary (profiles/)."""
    path = os.path.join(ROOT, "profiles", "ncu_full_summary.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        for name, v in d.items():  # kernel variants carry a suffix (e.g. _tpb)
            if name == kernel or name.startswith(kernel + "_"):
                return v
    except Exception:
        pass
    return {}


def ncu_kernels(kernel: str) -> list[dict]:
    """Every summary entry of `kernel` (variants: analytic::sim_kernel, dense::sim_kernel)."""
    path = os.path.join(ROOT, "profiles", "ncu_full_summary.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
    except Exception:
        return []
    return [v for name, v in d.items()
            if name == kernel or name.startswith(kernel + "_") or name.endswith("::" + kernel)]


def ncu_traffic(kernel: str, waves: bool = False):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary;
    waves=True sums its launches within one step (the sim kernel's two waves)."""
    ks = [k.get("dram_bytes_per_launch") for k in ncu_kernels(kernel)]
    if not ks or None in ks:
        return None
    return sum(ks) if waves else ks[0]


def algorithmic_bytes(low, rows) -> int:
    """SURVEY.md 8(d) DES-step bytes: 16 B per batch membership (a member's
    context and remaining-token counters read + written) plus one read of the
    instance inputs and one write of its outputs."""
    import numpy as np
    memberships = int(rows["total_tokens"].sum())  # each membership emits exactly one token
    n_req = low.n_requests
    inputs = (low.descs.nbytes + low.replicas.nbytes + low.prefixes.nbytes
              + n_req * (8 + 4 + 4 + 4))
    outputs = rows.nbytes + n_req * (8 + 8 + 4)
    return 16 * memberships + inputs + outputs + 0 * int(np.int64(0))


def bench_attention_cost(eng, device: int, steps: int, warmup: int, n_batches: int = 1 << 20):
    """C2: analytic refined-attention cost over 2^20 skewed 72-request batches.

    HBM-bound segmented reduction (csrc/fs_costs.cu). Inputs (~0.6 GB) exceed
    the 126 MB L2, so no flush is needed between steps. Returns a dict for
    the bench line.
    """
    import torch

    from paper_2508_03148_b200 import workloads as W
    from paper_2508_03148_b200.engine import attn_params
    q, kv, off, dec = W.attention_batches(n_batches)
    dev = f"cuda:{device}"
    tq = torch.from_numpy(q).to(dev)
    tkv = torch.from_numpy(kv).to(dev)
    toff = torch.from_numpy(off).to(dev)
    tdec = torch.from_numpy(dec).to(dev)
    out = torch.empty(n_batches, dtype=torch.float64, device=dev)
    st = torch.empty(n_batches, dtype=torch.int32, device=dev)
    prm = attn_params(32, 8, 128, 2, 2.25e15, 8e12, 5.0)
    stream = torch.cuda.Stream(device=device)

    def time_launches(launch):
        for _ in range(max(warmup, 1)):
            launch()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        for s, e in ev:
            s.record(stream)
            launch()
            e.record(stream)
        torch.cuda.synchronize()
        return sum(s.elapsed_time(e) for s, e in ev) / steps

    ms = time_launches(lambda: eng.attention_cost_dev(
        tq.data_ptr(), tkv.data_ptr(), toff.data_ptr(), tdec.data_ptr(), n_batches, prm,
        out.data_ptr(), st.data_ptr(), stream.cuda_stream))
    n_el = int(off[-1])
    alg = 8 * n_el + 8 * (n_batches + 1) + n_batches + 8 * n_batches + 4 * n_batches
    peak, kind = measured_peaks()
    gbs = alg / (ms / 1e3) / 1e9
    ok = bool((st == 0).all().item())
    res = {"workload": f"{n_batches} batches x 72 requests, lognormal(6.5,1.4) kv lengths, "
                       "alternating decode / prefill", "batches_per_s": n_batches / (ms / 1e3),
           "ms_per_launch": ms, "algorithmic_bytes_per_launch": alg,
           "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",
                        "frac": gbs / peak, "traffic": ncu_traffic("attention_cost_kernel"),
                        "peak_source": kind},
           "all_status_ok": ok}
    # learned mode: the C2 forest (make_attention_suite(5000, seed=11) -> fit_model(seed=7),
    # 100 trees, depth <= 12) over the same batches: 17 features + 100 tree walks + sort
    model_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tests", "golden",
                              "forest_c2.json.gz")
    if os.path.exists(model_path):
        from paper_2508_03148_b200.costmodel import ForestSet, load_model_file
        fs = ForestSet()
        fs.add(load_model_file(model_path))
        eng.set_forests(fs)
        out2 = torch.empty(n_batches, dtype=torch.float64, device=dev)
        ms2 = time_launches(lambda: eng.attention_forest_dev(
            0, tq.data_ptr(), tkv.data_ptr(), toff.data_ptr(), tdec.data_ptr(), n_batches, prm,
            out2.data_ptr(), stream.cuda_stream))
        alg2 = 8 * n_el + 8 * (n_batches + 1) + n_batches + 8 * n_batches
        gbs2 = alg2 / (ms2 / 1e3) / 1e9
        res["learned"] = {
            "model": "forest_c2 (100 trees)", "batches_per_s": n_batches / (ms2 / 1e3),
            "ms_per_launch": ms2, "algorithmic_bytes_per_launch": alg2,
            "tree_walks_per_s": 100 * n_batches / (ms2 / 1e3),
            "roofline": {"bound": "hbm", "achieved": gbs2, "peak": peak, "unit": "GB/s",
                         "frac": gbs2 / peak, "traffic": ncu_traffic("attention_forest_kernel"),
                         "peak_source": kind,
                         "note": "tree walks are L2-latency bound; HBM fraction is low by design"}}
    return res


def _dirichlet(doc: dict, alpha: float = 0.3) -> dict:
    doc["routing"] = {"policy": "dirichlet_skew", "alpha": alpha}
    return doc


def bench_configs(device: int, reps: int = 2):
    """The other BASELINE.json configs as batches of independent seeds on one GPU:
    C1 (Llama-2-7B co-located, 1,000 requests), C3 (PD 70B, tight 30 GB decode
    pool), C4 (DeepSeek-V3 AF m=2 and co-located EP=8, 64 requests). Each row:
    instances, iterations, device ms per batch (CUDA events, inputs resident)
    and the C port of the reference on one host core for one instance."""
    import torch

    from oracle import oracle
    from paper_2508_03148_b200 import workloads as W
    from paper_2508_03148_b200.engine import Engine
    cases = {
        "C1_colocated_llama7b_1000req": (lambda s: W.c1_colocated(1000, seed=s), 296),
        "C3_pd_70b_tight_300req": (lambda s: W.c3_pd(300, seed=s, tight=True), 296),
        "C4_af_dsv3_m2_64req": (lambda s: W.c4_af(64, seed=s), 148),
        "C4_colocated_dsv3_ep8_64req": (lambda s: W.c4_colocated_ep(64, seed=s), 148),
        "C4_colocated_dsv3_ep8_dirichlet0.3_64req": (lambda s: _dirichlet(W.c4_colocated_ep(64, seed=s)),
                                                     148),
    }
    out = {}
    stream = torch.cuda.Stream(device=device)
    for name, (make, n) in cases.items():
        low = lower_docs([make(1 + i) for i in range(n)])
        eng = Engine(device)
        eng.stage(low)
        eng.launch(stream.cuda_stream)
        torch.cuda.synchronize()
        rows = eng.fetch(low, per_request=False).rows
        ms = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            eng.launch(stream.cuda_stream)
            b.record(stream)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        its = int(rows["iterations"].sum())
        one = lower_docs([make(1)])
        t0 = time.perf_counter()
        ref = oracle.run(one, threads=1)
        cpu_s = time.perf_counter() - t0
        out[name] = {"instances": n, "iterations": its, "ms": min(ms),
                     "iterations_per_s": its / (min(ms) / 1e3),
                     "all_ok": bool((rows["status"] == 0).all()),
                     "routing_draws": int(rows["routing_draws"].sum()),
                     "cpu_port_1core_iterations_per_s": int(ref.rows["iterations"][0]) / cpu_s}
    return out


def routing_line(draws: int, step_ms: float, sm_mhz: float | None = None) -> dict:
    rate = draws / (step_ms / 1e3)
    pk = routing_peak()
    out = {"draws_per_step": draws, "draws_per_s": rate,
           "note": "uniform-router Philox4x64-10 keys (T x E per call) drawn inside sim_kernel; "
                   "frac = keys/s over the whole step against the routing core's measured peak "
                   "at sim_kernel's occupancy (8 warps/SM)"}
    if pk:
        out.update({"peak": pk["rolled_8_warps_per_sm"], "frac": rate / pk["rolled_8_warps_per_sm"],
                    "peak_best_occupancy": pk["rolled_best"], "peak_unrolled": pk["unrolled_best"],
                    "peak_source": pk["source"]})
    # the multiplier bound: 80 IMAD.WIDE.U32 per Philox4x64-10 block at
    # the measured 25.6 lane-ops per clock per SM (profiles/imad_rates_r2.json)
    wide = imad_wide_rate()
    if wide:
        blocks_peak = wide * 148 * (sm_mhz or 1965.0) * 1e6 / 80
        out["imad_wide_bound"] = {"unit": "Philox blocks/s", "achieved": rate / 4,
                                  "peak": blocks_peak, "frac": rate / 4 / blocks_peak,
                                  "imad_wide_per_block": 80,
                                  "lane_ops_per_clk_per_sm": wide,
                                  "source": "profiles/imad_rates_r2.json"}
    return out


def bench_learned_sweep(device: int, seeds: int = 8, reps: int = 2):
    """C5's 64 configs in learned mode (cost_model.mode learned with the C2 attention
    forest, model.py:294-327): every iteration's attention cost is a 100-tree forest
    prediction over the batch's attention_v1 features, inside sim_kernel's learned
    variant. Device ms per batch (inputs resident) and iterations/s."""
    import copy as _copy

    import torch

    from paper_2508_03148_b200.engine import Engine
    model = os.path.join(ROOT, "tests", "golden", "forest_c2.json.gz")
    if not os.path.exists(model):
        return None
    docs = workload_docs(0, seeds, 64)
    for d in docs:
        d["cost_model"] = {"mode": "learned", "attention_model": model}
    low = lower_docs([_copy.deepcopy(d) for d in docs])
    eng = Engine(device)
    stream = torch.cuda.Stream(device=device)
    eng.stage(low)
    eng.launch(stream.cuda_stream)
    torch.cuda.synchronize()
    rows = eng.fetch(low, per_request=False).rows
    ms = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        eng.launch(stream.cuda_stream)
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    its = int(rows["iterations"].sum())
    return {"workload": f"C5 64 configs x {seeds} seeds, learned attention (forest_c2, 100 trees)",
            "instances": low.n_instances, "iterations": its, "ms": min(ms),
            "iterations_per_s": its / (min(ms) / 1e3), "all_ok": bool((rows["status"] == 0).all())}


def main():
    args = parse_args()
    rank, world, local = dist_env()
    if world != args.gpus and args.gpus != 1:
        pass  # trust WORLD_SIZE when launched by torchrun
    if args.impl == "reference":
        return main_reference(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist

    # one rank per GPU; FS_BENCH_BACKEND=gloo runs several ranks on fewer GPUs
    # (a functional check of the multi-rank path on a 1-GPU box, not a measurement)
    backend = os.environ.get("FS_BENCH_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cdev = f"cuda:{local}" if backend == "nccl" else "cpu"  # device of the collectives' tensors
    from paper_2508_03148_b200 import abi
    from paper_2508_03148_b200.engine import Engine

    t_low0 = time.perf_counter()
    strong = args.scaling == "strong"
    if strong:  # one fixed sweep, LPT-sharded like api.simulate / simulate_rows
        from paper_2508_03148_b200.api import shard_plan
        all_docs = workload_docs(0, args.seeds, args.requests)
        _, shards = shard_plan(all_docs, world)
        docs = [all_docs[i] for i in shards[rank]]
    else:
        docs = workload_docs(rank, args.seeds, args.requests)
    low = lower_docs(docs)
    t_low = time.perf_counter() - t_low0
    eng = Engine(local)
    stream = torch.cuda.Stream(device=local)
    eng.stage(low)
    flush = torch.empty(int(256 * 2**20) // 4, dtype=torch.float32, device=f"cuda:{local}")

    # warm-up (also validates every instance ran)
    for _ in range(max(args.warmup, 1)):
        eng.launch(stream.cuda_stream)
    torch.cuda.synchronize()
    res = eng.fetch(low, per_request=False)
    if (res.rows["status"] != 0).any():
        bad = int((res.rows["status"] != 0).sum())
        raise SystemExit(f"{bad} instances failed: statuses {np.unique(res.rows['status'])}")
    iters_per_step = int(res.rows["iterations"].sum())
    draws_per_step = int(res.rows["routing_draws"].sum())
    launches_per_step = eng.last_launch_count

    # timed region: device-resident inputs
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                flush.zero_()  # > L2 (126 MB): evict the previous step's state
                starts[i].record(stream)
                eng.launch(stream.cuda_stream)
                ends[i].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device=cdev)
    its = torch.tensor([iters_per_step * args.steps], dtype=torch.float64, device=cdev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(its, op=dist.ReduceOp.SUM)
    max_ms = float(t.item())
    total_its = float(its.item())
    value = total_its / (max_ms / 1e3)

    # kernel share: time the simulation kernel alone vs the metrics kernel
    # (events around each phase of one extra launch are not possible inside the
    # library; the ncu launch list in profiles/ gives the split).

    # end-to-end through the C ABI with host buffers (H2D + kernels + D2H); in strong
    # scaling also the all-gather of every rank's metric rows (the sweep's result)
    from paper_2508_03148_b200.distributed import gather_rows
    e2e_times = []
    raw = None
    for i in range(args.warmup + args.steps):
        if world > 1 and i == args.warmup:
            dist.barrier()
        t0 = time.perf_counter()
        raw = eng.run(low)
        if strong and world > 1:
            gathered = gather_rows(raw.rows, world, cdev if backend == "nccl" else None)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            e2e_times.append(dt)
    if strong and world > 1:
        got = sum(int(g["iterations"].sum()) for g in gathered)
        if got * args.steps != int(total_its):
            raise SystemExit(f"gathered rows hold {got} iterations, expected {total_its / args.steps}")
    e2e_s = torch.tensor([sum(e2e_times)], dtype=torch.float64, device=cdev)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_value = total_its / float(e2e_s.item())
    h2d = (low.descs.nbytes + low.replicas.nbytes + low.prefixes.nbytes + low.trace_counts.nbytes
           + low.arrival.nbytes + low.prompt.nbytes + low.output.nbytes + low.id_rank.nbytes)
    d2h = (raw.rows.nbytes + raw.replica_out.nbytes + raw.first_ns.nbytes + raw.done_ns.nbytes
           + raw.done_rank.nbytes)
    assert (raw.rows["iterations"] == res.rows["iterations"]).all()

    # the user-facing call: simulate(config documents) -- parse, validate, draw the
    # workloads on the device, lower, run, compute_metrics -- timed once per rank
    api = None
    if not args.no_api:
        from paper_2508_03148_b200.api import simulate, simulate_rows
        import copy as _copy
        # warm-up call on the same documents (buffers sized, the pipeline's peer engine
        # created), as a caller that simulates more than once sees it
        simulate(_copy.deepcopy(docs), engine=eng, device_workload=True, expert_imbalance=False)
        if strong and world > 1:
            mine_docs = _copy.deepcopy(all_docs)  # the caller's documents, outside the clock
            dist.barrier()
            t0 = time.perf_counter()
            sr = simulate_rows(mine_docs, engine=eng, device_workload=True)
            api_s = time.perf_counter() - t0
            n_fail = len(sr.failed)
            note = ("simulate_rows(all docs, device_workload=True) under torchrun: every rank "
                    "parses, LPT-shards, simulates its shard; rows all-gathered over NCCL")
            api_its = int(sr.rows["iterations"].sum())
        else:
            call_docs = _copy.deepcopy(docs)  # the caller's documents, outside the clock
            t0 = time.perf_counter()
            bundles = simulate(call_docs, engine=eng, device_workload=True,
                               expert_imbalance=False)
            api_s = time.perf_counter() - t0
            n_fail = sum(1 for b in bundles if not hasattr(b, "to_dict"))
            note = ("simulate(docs, device_workload=True, expert_imbalance=False): config "
                    "parsing and validation, device workload generation, lowering, "
                    "fs_run_batch, compute_metrics (MetricsBundle per instance)")
            api_its = iters_per_step
        api = {"value": api_its / api_s, "unit": UNIT, "seconds": api_s, "failures": n_fail,
               "note": note}

    # the only collective: gather every rank's fixed-size metric rows (NCCL)
    gather_ms = None
    if world > 1 and not strong:
        rows_t = torch.from_numpy(raw.rows.view(np.uint8).copy()).to(cdev)
        out = [torch.empty_like(rows_t) for _ in range(world)]
        torch.cuda.synchronize()
        g0 = time.perf_counter()
        dist.all_gather(out, rows_t)
        torch.cuda.synchronize()
        gather_ms = (time.perf_counter() - g0) * 1e3
        # every rank's rows arrived intact: their iterations add up to the job total
        got = sum(int(np.frombuffer(o.cpu().numpy().tobytes(), dtype=abi.METRIC_ROW)
                      ["iterations"].sum()) for o in out)
        if got * args.steps != int(total_its):
            raise SystemExit(f"gathered rows hold {got} iterations, expected {total_its / args.steps}")

    # roofline of the dominant kernel (the DES step kernel)
    alg_bytes = algorithmic_bytes(low, res.rows)
    peak, peak_kind = measured_peaks()
    avg_ms = max_ms / args.steps
    achieved = alg_bytes / (avg_ms / 1e3) / 1e9
    traffic = ncu_traffic("sim_kernel", waves=True)

    # the DES step kernel is instruction-issue bound, not HBM bound: its
    # instruction roofline from the committed ncu capture (warp instructions per
    # launch, same workload) over this run's step time vs 148 SMs x 4 issue/clk
    issue = None
    sims = ncu_kernels("sim_kernel")  # the MoE wave and the dense wave of a step
    summ = {"warp_instructions": sum(k.get("warp_instructions", 0) for k in sims),
            "issue_active_pct": [k.get("issue_active_pct") for k in sims],
            "source": sorted({k.get("source") for k in sims})} if sims else {}
    if summ.get("warp_instructions"):
        sm_mhz = (clocks.summary() or {}).get("sm_max_mhz") or 1965.0
        peak_ips = 148 * 4 * sm_mhz * 1e6
        ips = summ["warp_instructions"] / (avg_ms / 1e3)
        issue = {"bound": "issue", "unit": "warp-instructions/s", "achieved": ips,
                 "peak": peak_ips, "frac": ips / peak_ips,
                 "warp_instructions_per_launch": summ["warp_instructions"],
                 "ncu_issue_active_pct": summ.get("issue_active_pct"),
                 "source": summ.get("source")}

    c2 = None
    if not args.no_c2:
        c2 = bench_attention_cost(eng, local, args.steps, args.warmup)

    configs = None
    learned = None
    if rank == 0 and world == 1 and not args.no_configs:
        configs = bench_configs(local)
        learned = bench_learned_sweep(local)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = cpu_count()
        c_its, c_dt, n_inst = run_oracle_sample(args.requests, args.cpu_sample_seeds, threads)
        s_its, s_dt, s_inst = run_oracle_sample(args.requests, 1, 1)  # one core, serial
        cpu = {"value": c_its / c_dt, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"C5 configs x {args.cpu_sample_seeds} seeds = {n_inst} instances "
                         f"({c_its} iterations) in {c_dt:.2f}s on {threads} threads "
                         f"({cpu_model()}); oracle/fs_oracle.c",
               "serial_1core": {"value": s_its / s_dt, "unit": UNIT,
                                "sample": f"C5 configs x 1 seed = {s_inst} instances "
                                          f"({s_its} iterations) in {s_dt:.2f}s"}}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64+int64", "data": "synthetic",
            "config": {"workload": "C5 design-space sweep: 64 configs x "
                                   f"{args.seeds} seeds x {args.requests} requests "
                                   + ("in total, LPT-sharded over the GPUs" if strong else "per GPU"),
                       "instances_per_gpu": low.n_instances, "iterations_per_step": int(total_its) // args.steps,
                       "parallelism": f"instances sharded over {world} GPU(s), NCCL gather of rows",
                       "l2": "flushed between steps (256 MB write, outside events)"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "host_lowering_s": t_low},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "sim_kernel: MoE wave (analytic) + dense wave (dense variant)",
                         "algorithmic_bytes_per_launch": alg_bytes, "peak_source": peak_kind},
            "issue": issue,
            "api_end_to_end": api,
            "routing": routing_line(draws_per_step * world, max_ms / args.steps,
                                    (clocks.summary() or {}).get("sm_max_mhz")),
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
            "gpu_launches": launches_per_step * args.steps,
            "gather_ms": gather_ms,
            "step_ms": step_ms,
            "c2_attention_cost": c2,
            "baseline_configs": configs,
            "c5_learned": learned,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def main_reference(args, rank, world):
    """CPU port of the reference path (oracle/fs_oracle.c) with every host thread."""
    if rank != 0:
        return
    threads = cpu_count()
    from oracle import oracle
    ref_seeds = args.reference_seeds or args.seeds
    docs = workload_docs(0, ref_seeds, args.requests)
    low = lower_docs(docs)
    oracle.load()
    times = []
    its = 0
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        res = oracle.run(low, threads=threads)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
            its = int(res.rows["iterations"].sum())
    value = its * len(times) / sum(times)
    sample = (f"C5 configs x {ref_seeds} seeds = {low.n_instances} instances "
              f"({its} iterations) per step on {threads} threads ({cpu_model()})")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sum(times) / len(times) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64+int64", "data": "synthetic",
            "config": {"workload": f"C5 design-space sweep: 64 configs x {args.seeds} seeds x "
                                   f"{args.requests} requests per GPU"
                                   + ("" if ref_seeds == args.seeds else
                                      f" (timed on a {ref_seeds}-seed sample of every config)"),
                       "instances_per_step": low.n_instances},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
