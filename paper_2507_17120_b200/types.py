"""Data model shared by the window API and the drop-in classes.

Names and fields follow the reference (workload.py:25-51,
batch_controller.py:21-67, bucket_manager.py:56-69).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

from . import _native as N


class TaskClass(Enum):
    """workload.py:25-27 (class 0 = ONLINE dispatches first, pd_sim.py:449-450)."""
    ONLINE = "online"
    OFFLINE = "offline"


class DispatchPolicy(Enum):
    """batch_controller.py:21-25."""
    SJF = "sjf"
    LJF = "ljf"
    EARLIEST_ARRIVAL = "earliest_arrival"
    FCFS = "fcfs"


class MemoryAccounting(Enum):
    """batch_controller.py:28-30."""
    PADDED = "padded"
    EXACT = "exact"


def enum_value(x):
    """The reference compares its enums by identity (`is`); a caller that swaps these
    classes into bucketsim passes bucketsim's own enum members, so members of any enum
    are matched by their value ("online", "sjf", "padded", ...)."""
    return x.value if isinstance(x, Enum) else x


def is_online(task_class) -> bool:
    return enum_value(task_class) == TaskClass.ONLINE.value


def is_offline(task_class) -> bool:
    return enum_value(task_class) == TaskClass.OFFLINE.value


def policy_code(p) -> int:
    if isinstance(p, int) and not isinstance(p, Enum):
        if p not in (N.POLICY_FCFS, N.POLICY_SJF, N.POLICY_LJF):
            raise ValueError(f"unknown dispatch policy {p}")
        return p
    p = DispatchPolicy(enum_value(p))
    return {DispatchPolicy.SJF: N.POLICY_SJF, DispatchPolicy.LJF: N.POLICY_LJF,
            DispatchPolicy.FCFS: N.POLICY_FCFS,
            DispatchPolicy.EARLIEST_ARRIVAL: N.POLICY_FCFS}[p]


def accounting_code(a) -> int:
    if isinstance(a, int) and not isinstance(a, Enum):
        if a not in (N.ACCOUNTING_PADDED, N.ACCOUNTING_EXACT):
            raise ValueError(f"unknown memory accounting {a}")
        return a
    a = MemoryAccounting(enum_value(a))
    return N.ACCOUNTING_PADDED if a is MemoryAccounting.PADDED else N.ACCOUNTING_EXACT


@dataclass
class Request:
    """workload.py:30-51 (only the fields the scheduling path reads are required)."""
    id: int
    arrival_time: float
    input_len: int
    output_len: int | None
    task_class: object
    slo_ttft: float | None = None
    slo_e2e: float | None = None
    enqueue_time: float | None = None
    prefill_start: float | None = None
    first_token_time: float | None = None
    completion_time: float | None = None


@dataclass(frozen=True)
class StructuralChange:
    """bucket_manager.py:56-63."""
    kind: str  # "split" | "merge" | "skip"
    parent_low: int
    parent_up: int
    midpoint: int | None = None


@dataclass(frozen=True)
class PartitionViolation:
    """bucket_manager.py:66-69."""
    kind: str
    detail: str


@dataclass(frozen=True)
class BatchPlan:
    """batch_controller.py:44-56."""
    request_ids: tuple
    requests: tuple
    max_input_len: int
    token_sum: int
    footprint: int
    created_at: float
    source_bucket: tuple

    def __len__(self) -> int:
        return len(self.requests)


@dataclass(frozen=True)
class OversizeRejection:
    """batch_controller.py:59-67."""
    request: Request
    footprint: int
    safe_mem: int


CHANGE_KIND = {N.CHANGE_SPLIT: "split", N.CHANGE_MERGE: "merge", N.CHANGE_SKIP: "skip"}
