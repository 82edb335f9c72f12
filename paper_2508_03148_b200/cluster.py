"""Replica-level scheduling policy (reference: pkg/src/frontier_sim/cluster.py:96-118).

Only the policy *description* lives on the host; admission, KV-pool
accounting and batch costing (cluster.py:36-93, 145-346) run inside the
device engine (csrc/engine.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

ADMISSIONS = ("fcfs", "fcfs_skip", "priority")
PRIORITY_KEYS = ("prompt_tokens", "arrival_time")
MEMORY_MODES = ("exact", "paged")


@dataclass(frozen=True)
class SchedulerPolicy:
    admission: str = "fcfs"
    priority_key: str = "prompt_tokens"
    max_num_seqs: int = 256
    max_batch_tokens: int = 8192
    memory_mode: str = "exact"
    block_tokens: int = 16

    def validate(self) -> None:
        if self.admission not in ADMISSIONS:
            raise ValueError(f"unknown admission policy {self.admission!r}")
        if self.priority_key not in PRIORITY_KEYS:
            raise ValueError(f"unknown priority key {self.priority_key!r}")
        if self.max_num_seqs < 1 or self.max_batch_tokens < 1:
            raise ValueError("batch budgets must be positive")
        if self.memory_mode not in MEMORY_MODES:
            raise ValueError(f"unknown memory mode {self.memory_mode!r}")
        if self.block_tokens < 1:
            raise ValueError("block_tokens must be >= 1")

    def pool_block_tokens(self) -> int | None:
        return self.block_tokens if self.memory_mode == "paged" else None
