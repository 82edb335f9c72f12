"""Config documents for the BASELINE workloads.

Every builder returns a plain JSON-able document in the reference's config
schema (reference: pkg/src/frontier_sim/config.py:364-493), so the same
document feeds this engine's `parse_config` and, in the container that has
it, the reference's own `parse_config`.

Tags:
  C1  co-located Llama-2-7B shape, 1 replica, 1k-request Poisson trace
  C2  skewed varlen attention batches (see `attention_batches`)
  C3  PD 70B shape, tp=4, roomy / tight decode pool
  C4  DeepSeek-V3 shape MoE: AF (m=2) and co-located EP=8
  C5  64 configs x 64 seeds sweep (A: dense co-located, B: dense PD,
      C: Mixtral MoE co-located EP)
"""

from __future__ import annotations

import copy
import itertools

import numpy as np

B200_HW = {
    "peak_flops": 2.25e15,
    "mem_bw": 8e12,
    "hbm_capacity_bytes": 180e9,
    "kernel_overhead_us": 5.0,
}
NETWORK = {
    "intra_replica": {"latency_s": 5e-6, "bandwidth_bps": 900e9},
    "inter_cluster": {"latency_s": 20e-6, "bandwidth_bps": 50e9},
}
LLAMA2_7B = {"num_layers": 32, "d_model": 4096, "d_ff": 11008,
             "num_query_heads": 32, "num_kv_heads": 32, "head_dim": 128}
DENSE_70B = {"num_layers": 80, "d_model": 8192, "d_ff": 28672,
             "num_query_heads": 64, "num_kv_heads": 8, "head_dim": 128}
DEEPSEEK_V3 = {"num_layers": 61, "d_model": 7168, "d_ff": 18432,
               "num_query_heads": 128, "num_kv_heads": 128, "head_dim": 56,
               "moe": {"num_experts": 256, "top_k": 8, "expert_d_ff": 2048}}
MIXTRAL_8X7B = {"num_layers": 32, "d_model": 4096, "d_ff": 14336,
                "num_query_heads": 32, "num_kv_heads": 8, "head_dim": 128,
                "moe": {"num_experts": 8, "top_k": 2, "expert_d_ff": 14336}}


def poisson_workload(n: int, rate: float, prompt_mu: float = 6.0, output_mu: float = 5.0,
                     seed: int | None = None) -> dict:
    doc = {
        "num_requests": n,
        "arrival": {"kind": "poisson", "rate_rps": rate},
        "prompt_tokens": {"kind": "lognormal", "mu": prompt_mu, "sigma": 1.0, "lo": 8, "hi": 4096},
        "output_tokens": {"kind": "lognormal", "mu": output_mu, "sigma": 0.8, "lo": 1, "hi": 1024},
    }
    if seed is not None:
        doc["seed"] = seed
    return doc


def _hw(hbm: float | None = None) -> dict:
    hw = dict(B200_HW)
    if hbm is not None:
        hw["hbm_capacity_bytes"] = hbm
    return hw


def c1_colocated(n_requests: int = 1000, seed: int = 1) -> dict:
    return {
        "mode": "colocated", "seed": seed, "model": copy.deepcopy(LLAMA2_7B),
        "clusters": [{"id": "c0", "role": "colocated", "gpus_per_replica": 1, "hardware": _hw()}],
        "network": copy.deepcopy(NETWORK),
        "workload": poisson_workload(n_requests, 20.0),
    }


def c3_pd(n_requests: int = 300, seed: int = 1, tight: bool = True) -> dict:
    par = {"tp": 4}
    return {
        "mode": "pd", "seed": seed, "model": copy.deepcopy(DENSE_70B),
        "clusters": [
            {"id": "p0", "role": "prefill", "gpus_per_replica": 4, "hardware": _hw(),
             "parallelism": dict(par)},
            {"id": "d0", "role": "decode", "gpus_per_replica": 4,
             "hardware": _hw(30e9 if tight else None), "parallelism": dict(par)},
        ],
        "network": copy.deepcopy(NETWORK),
        "workload": poisson_workload(n_requests, 5.0),
    }


def c4_af(n_requests: int = 64, seed: int = 1, micro_batches: int = 2) -> dict:
    par = {"attn_tp": 8, "attn_dp": 1, "moe_tp": 1, "moe_ep": 8}
    return {
        "mode": "af", "seed": seed, "model": copy.deepcopy(DEEPSEEK_V3),
        "clusters": [
            {"id": "attn", "role": "attention", "gpus_per_replica": 8, "hardware": _hw(),
             "parallelism": dict(par)},
            {"id": "ffn", "role": "ffn", "gpus_per_replica": 8, "hardware": _hw(),
             "parallelism": dict(par)},
        ],
        "network": copy.deepcopy(NETWORK),
        "af": {"micro_batches": micro_batches},
        "routing": {"policy": "uniform"},
        "workload": poisson_workload(n_requests, 50.0, prompt_mu=5.0, output_mu=3.0),
    }


def c4_colocated_ep(n_requests: int = 64, seed: int = 1) -> dict:
    return {
        "mode": "colocated", "seed": seed, "model": copy.deepcopy(DEEPSEEK_V3),
        "clusters": [{"id": "c0", "role": "colocated", "gpus_per_replica": 8, "hardware": _hw(),
                      "parallelism": {"tp": 1, "ep": 8}}],
        "network": copy.deepcopy(NETWORK),
        "routing": {"policy": "uniform"},
        "workload": poisson_workload(n_requests, 50.0, prompt_mu=5.0, output_mu=3.0),
    }


def c5_sweep_configs(n_requests: int = 64) -> list[dict]:
    """The 64 C5 design points (seed filled in by `c5_sweep`)."""
    out: list[dict] = []
    for tp, mns in itertools.product((1, 2, 4, 8), (32, 64, 128, 256)):  # A: dense co-located
        out.append({
            "mode": "colocated", "model": copy.deepcopy(LLAMA2_7B),
            "clusters": [{"id": "c0", "role": "colocated", "gpus_per_replica": tp,
                          "hardware": _hw(), "parallelism": {"tp": tp}}],
            "network": copy.deepcopy(NETWORK), "policies": {"max_num_seqs": mns},
            "workload": poisson_workload(n_requests, 20.0),
        })
    pd_ratios = ((1, 1), (1, 2), (2, 1), (1, 3), (3, 1), (2, 3), (3, 2), (2, 2))
    for tp, mns, (p, d) in itertools.product((2, 4), (64, 256), pd_ratios):  # B: dense PD
        out.append({
            "mode": "pd", "model": copy.deepcopy(LLAMA2_7B),
            "clusters": [
                {"id": "p0", "role": "prefill", "num_replicas": p, "gpus_per_replica": tp,
                 "hardware": _hw(), "parallelism": {"tp": tp}},
                {"id": "d0", "role": "decode", "num_replicas": d, "gpus_per_replica": tp,
                 "hardware": _hw(), "parallelism": {"tp": tp}},
            ],
            "network": copy.deepcopy(NETWORK), "policies": {"max_num_seqs": mns},
            "workload": poisson_workload(n_requests, 20.0),
        })
    for ep, mns in itertools.product((1, 2, 4, 8), (32, 64, 128, 256)):  # C: MoE co-located EP
        out.append({
            "mode": "colocated", "model": copy.deepcopy(MIXTRAL_8X7B),
            "clusters": [{"id": "c0", "role": "colocated", "gpus_per_replica": ep,
                          "hardware": _hw(), "parallelism": {"ep": ep}}],
            "network": copy.deepcopy(NETWORK), "policies": {"max_num_seqs": mns},
            "routing": {"policy": "uniform"},
            "workload": poisson_workload(n_requests, 20.0),
        })
    return out


def c5_sweep(n_seeds: int = 64, n_requests: int = 64, seed_base: int = 1000,
             configs: list[int] | None = None) -> list[dict]:
    """C5: every design point x `n_seeds` trace seeds.

    Instance seed = seed_base + 64 * config + s; the
    workload seed defaults to the master seed, as in the reference config.
    """
    base = c5_sweep_configs(n_requests)
    docs = []
    for ci, doc in enumerate(base):
        if configs is not None and ci not in configs:
            continue
        for s in range(n_seeds):
            d = copy.deepcopy(doc)
            d["seed"] = seed_base + 64 * ci + s
            docs.append(d)
    return docs


def attention_batches(n_batches: int, batch_size: int = 72, seed: int = 72,
                      mu: float = 6.5, sigma: float = 1.4):
    """C2: skewed varlen attention batches in CSR form.

    kv_len = clip(rint(lognormal(mu, sigma)), 16, 32768); even batches are
    decode (q = 1), odd batches prefill (q = kv). Returns (q_lens, kv_lens,
    offsets, is_decode) as numpy arrays.
    """
    rng = np.random.default_rng(seed)
    kv = np.clip(np.rint(rng.lognormal(mu, sigma, size=n_batches * batch_size)),
                 16, 32768).astype(np.int32)
    is_decode = (np.arange(n_batches) % 2 == 0).astype(np.uint8)
    q = kv.copy()
    q.reshape(n_batches, batch_size)[is_decode.astype(bool)] = 1
    offsets = np.arange(n_batches + 1, dtype=np.int64) * batch_size
    return q, kv, offsets, is_decode
