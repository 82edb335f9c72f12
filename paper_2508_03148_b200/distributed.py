"""Multi-GPU sweep sharding.

Sweep instances are independent (each point owns a private simulation,
reference SPEC.md:678), so the data path has no collective: every rank
simulates its own shard of instances on its own GPU, and the only exchange
is one all-gather of the fixed-size metric rows at the end (NCCL over
NVLink/NVSwitch on the B200 box, gloo in the CPU tests).

Sharding is longest-processing-time (LPT) on the host's per-instance cost
estimate, so the slowest rank's share is balanced even when MoE instances
cost orders of magnitude more than dense ones.
"""

from __future__ import annotations

import heapq

import numpy as np


def lpt_shards(costs: list[int] | np.ndarray, world: int) -> list[list[int]]:
    """Greedy LPT: assign instances (largest cost first) to the least-loaded rank.

    Ties break by rank index; each rank's list keeps the original instance order.
    """
    costs = np.asarray(costs, dtype=np.int64)
    order = np.argsort(-costs, kind="stable")
    heap = [(0, r) for r in range(world)]
    shards: list[list[int]] = [[] for _ in range(world)]
    for i in order.tolist():
        load, r = heapq.heappop(heap)
        shards[r].append(i)
        heapq.heappush(heap, (load + int(costs[i]), r))
    return [sorted(s) for s in shards]


def gather_rows(rows: np.ndarray, world: int, device=None) -> list[np.ndarray]:
    """All-gather each rank's structured metric-row array (variable length).

    Uses the default torch.distributed process group (NCCL on GPUs, gloo on
    CPU). Returns the per-rank arrays in rank order.
    """
    import torch
    import torch.distributed as dist

    raw = np.ascontiguousarray(rows).view(np.uint8)
    n = torch.tensor([raw.size], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    cap = int(max(int(s.item()) for s in sizes))
    buf = torch.zeros(cap, dtype=torch.uint8, device=device)
    buf[: raw.size] = torch.from_numpy(raw.copy()).to(device=buf.device)
    outs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf)
    return [o[: int(s.item())].cpu().numpy().view(rows.dtype) for o, s in zip(outs, sizes)]


def merge_shards(shards: list[list[int]], per_rank_rows: list[np.ndarray], n: int) -> np.ndarray:
    """Reassemble per-rank rows into the global instance order."""
    out = np.zeros(n, dtype=per_rank_rows[0].dtype)
    for idx, rows in zip(shards, per_rank_rows):
        out[np.asarray(idx, dtype=np.int64)] = rows
    return out
