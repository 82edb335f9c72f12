"""Small configuration records shared by config parsing and the orchestrator.

reference: orchestrator/af.py:56-62 (AfPipelineConfig),
orchestrator/base.py:86-90 (RoutingPolicySpec).
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class AfPipelineConfig:
    micro_batches: int = 2

    def validate(self) -> None:
        if self.micro_batches < 1:
            raise ValueError("micro_batches must be >= 1")


@dataclass(frozen=True)
class RoutingPolicySpec:
    policy: str = "uniform"  # uniform | dirichlet_skew | trace
    alpha: float = 0.3
    trace_counts: tuple[int, ...] | None = None
