"""Exception types raised for per-instance device status codes.

Names match the exceptions the reference raises for the same condition so
callers that catch them keep working (reference files in brackets).
"""

from __future__ import annotations


class SimulationError(Exception):
    """[orchestrator/base.py:78] queue drained with unfinished requests."""


class RequestCannotFit(SimulationError):
    """[orchestrator/base.py:82] a request's KV footprint can never fit."""


class SimCoreError(Exception):
    """[core.py:54]"""


class SchedulingInPast(SimCoreError):
    """[core.py:58]"""


class EventBudgetExceeded(SimCoreError):
    """[core.py:66]"""


class RoutingError(Exception):
    """[costmodel/routing.py:25]"""


class InvalidTopK(Exception):
    """[costmodel/routing.py:21]"""


class TopologyMismatch(Exception):
    """[costmodel/moe.py:19]"""


class EmptyBatch(Exception):
    """[costmodel/features.py:17]"""


class RoutingTie(Exception):
    """Two uniform routing keys tied exactly at the top-k boundary. The
    reference's np.argpartition resolves such a tie in an implementation-
    defined way, so the engine reports it instead of guessing."""


class UnsupportedOnDevice(NotImplementedError):
    """The configuration needs a feature the device engine does not have yet."""


class EngineCapacityError(Exception):
    """A configuration exceeds a compiled engine limit (FS_MAX_*)."""


class EngineInternalError(RuntimeError):
    """An engine invariant was violated (a bug: please report)."""


# enum fs_status (include/frontier_b200.h) -> exception type
class ModelFileError(Exception):
    """[costmodel/model.py:49] malformed or tampered operator-model file."""


class SchemaMismatch(Exception):
    """[costmodel/model.py:33] a model's feature schema does not fit its use."""


STATUS_EXCEPTIONS = {
    1: RequestCannotFit,
    2: SimulationError,
    3: EventBudgetExceeded,
    4: SchedulingInPast,
    5: RoutingError,
    6: TopologyMismatch,
    7: EmptyBatch,
    8: InvalidTopK,
    9: RoutingTie,
    10: UnsupportedOnDevice,
    11: EngineCapacityError,
    12: EngineInternalError,
    13: ValueError,
    14: SchemaMismatch,
}
