"""Reference-shaped (bucketsim) surface over the B200 window path.

Drop-in classes for the scheduling path with the reference's names, argument
meaning and error behaviour (bucket_manager.py, batch_controller.py):

* `BucketSet` / `Bucket` — the stateful bucket structure the simulator drives
  (`assign`, `adjust_buckets`, `check_partition`, counters, `dirty`).  The set keeps
  an incremental per-length histogram of its queued requests (+1 on assign, -1 when
  form_batch removes a batch; revalidated against the queued total, recounted if the
  deques were changed behind its back), and the split / merge decisions of
  `adjust_buckets` run on the GPU as one Alg. 1 pass from the current edges over that
  histogram (K2, `max_passes=1`); the host then moves the Python `Request` objects
  between the deques exactly as bucket_manager.py:148-188 does.
* `BatchController` — `form_batch` runs K4+K5 on the GPU over the bucket's
  class-filtered candidates and returns the first batch of the drain (one
  form_batch call, batch_controller.py:141-191), with the same side effects
  (admitted and rejected requests leave the deque, `rejections` grows).
* `schedule_requests` — the whole window from reference `Request`
  objects to reference `BatchPlan` / `OversizeRejection` / `StructuralChange`
  records, via one `WindowScheduler.schedule` call.

Host-side work here is only what the reference API forces: Python objects in and
out (the deques are part of the public surface).  Counts, decisions, ordering and
sizing are computed by the CUDA kernels; there is no CPU fallback.
"""

from __future__ import annotations

import bisect
from collections import deque
from dataclasses import dataclass, field
from operator import attrgetter
from typing import Deque, Iterator, Sequence

import numpy as np

from . import _native as N
from .memory_model import GpuConfig, ModelConfig, safe_memory
from .types import (BatchPlan, DispatchPolicy, MemoryAccounting, OversizeRejection,
                    PartitionViolation, Request, StructuralChange, TaskClass, policy_code)

_ARRIVAL_ORDER = attrgetter("arrival_time", "id")


def order_requests(requests: Sequence[Request], policy: DispatchPolicy) -> list[Request]:
    """batch_controller.py:33-41 (object-level helper; the window path orders on the GPU)."""
    if policy is DispatchPolicy.SJF:
        key = lambda r: (r.input_len, r.arrival_time, r.id)  # noqa: E731
    elif policy is DispatchPolicy.LJF:
        key = lambda r: (-r.input_len, r.arrival_time, r.id)  # noqa: E731
    else:
        key = lambda r: (r.arrival_time, r.id)  # noqa: E731
    return sorted(requests, key=key)


# ---- scheduler pool: one WindowScheduler per (device, L, classes, ...) shape --------
_POOL: dict = {}


def _scheduler(n: int, **kw):
    from .window import WindowScheduler
    key = tuple(sorted((k, v if not isinstance(v, (list, tuple)) else tuple(v))
                       for k, v in kw.items()))
    s = _POOL.get(key)
    if s is None or s.max_requests < n:
        cap = max(1024, 1 << max(0, int(n - 1).bit_length()))
        s = WindowScheduler(max_requests=cap, **kw)
        _POOL[key] = s
    return s


def _class_index(task_class, classes: list) -> int:
    for i, c in enumerate(classes):
        if task_class is c:
            return i
    raise ValueError(f"unknown task class {task_class!r}")


# ---- bucket_manager.py ---------------------------------------------------------------
@dataclass
class Bucket:
    """bucket_manager.py:22-53."""
    low: int
    up: int
    requests: Deque[Request] = field(default_factory=deque)
    # per-length counts of the owning BucketSet (kept current on add / remove_ids)
    _counts: np.ndarray | None = field(default=None, repr=False, compare=False)

    def __post_init__(self) -> None:
        self.mid = (self.low + self.up) // 2
        self.short_count = sum(1 for r in self.requests if r.input_len < self.mid)

    def __len__(self) -> int:
        return len(self.requests)

    def add(self, request: Request) -> None:
        self.requests.append(request)
        if request.input_len < self.mid:
            self.short_count += 1
        if self._counts is not None:
            self._counts[request.input_len] += 1

    def remove_ids(self, ids: set) -> None:
        kept: Deque[Request] = deque()
        for r in self.requests:
            if r.id in ids:
                if r.input_len < self.mid:
                    self.short_count -= 1
                if self._counts is not None:
                    self._counts[r.input_len] -= 1
            else:
                kept.append(r)
        self.requests = kept

    def token_mass(self) -> int:
        return sum(r.input_len for r in self.requests)


class BucketSet:
    """Ordered contiguous buckets + split/merge policy (bucket_manager.py:72-216).
    Split/merge decisions run on the GPU (one K2 pass over the incremental histogram)."""

    def __init__(self, max_seq_len: int, split_threshold: float = 0.5,
                 buckets: list[Bucket] | None = None):
        if max_seq_len < 1:
            raise ValueError("max_seq_len must be >= 1")
        if not 0.0 < split_threshold <= 1.0:
            raise ValueError("split_threshold must be in (0, 1]")
        self.max_seq_len = max_seq_len
        self.split_threshold = split_threshold
        self.buckets: list[Bucket] = buckets if buckets is not None else [Bucket(0, max_seq_len)]
        # incremental per-length histogram of the queued requests: +1 on
        # assign / Bucket.add, -1 on Bucket.remove_ids; adjust_buckets uploads it
        self._counts = np.zeros(max_seq_len, np.int64)
        self._rebuild_counts()
        self.dirty = True
        self.assign_calls = 0
        self.assign_comparisons = 0
        self.last_assign_comparisons = 0
        self.adjust_calls = 0
        self.adjust_bucket_scans = 0
        self.requests_moved = 0

    def __len__(self) -> int:
        return len(self.buckets)

    @property
    def total_requests(self) -> int:
        return sum(len(b) for b in self.buckets)

    def iter_requests(self) -> Iterator[Request]:
        for b in self.buckets:
            yield from b.requests

    def edges(self) -> list[int]:
        return [b.low for b in self.buckets] + [self.buckets[-1].up]

    def _rebuild_counts(self) -> bool:
        """Recount from the deques (construction, or after the deques were changed
        behind the set's back); False if some queued length is outside [0, L)."""
        self._counts[:] = 0
        lens = np.fromiter((r.input_len for r in self.iter_requests()), np.int64)
        ok = bool(lens.size == 0 or (lens.min() >= 0 and lens.max() < self.max_seq_len))
        if ok:
            np.add.at(self._counts, lens, 1)
        for b in self.buckets:
            b._counts = self._counts if ok else None
        return ok

    def _current_counts(self) -> np.ndarray | None:
        """The incremental histogram, revalidated in O(L + K): every bucket must be
        attached and the counts must add up to the queued total; otherwise recount."""
        if (all(b._counts is self._counts for b in self.buckets)
                and int(self._counts.sum()) == self.total_requests):
            return self._counts
        return self._counts if self._rebuild_counts() else None

    def assign(self, request: Request) -> int:
        """bucket_manager.py:110-131 (bisect over the uppers; same result and counters)."""
        if not 0 <= request.input_len < self.max_seq_len:
            raise ValueError(
                f"input_len {request.input_len} outside [0, {self.max_seq_len}); "
                "truncation should have been applied")
        self.assign_calls += 1
        self.dirty = True
        ups = [b.up for b in self.buckets]
        idx = bisect.bisect_right(ups, request.input_len)
        b = self.buckets[idx]
        b.requests.append(request)
        if request.input_len < b.mid:
            b.short_count += 1
        if b._counts is not None:
            b._counts[request.input_len] += 1
        self.assign_comparisons += idx + 1
        self.last_assign_comparisons = idx + 1
        return idx

    def adjust_buckets(self, n_max: int) -> list[StructuralChange]:
        """One Alg. 1 pass (bucket_manager.py:133-191); decisions from the GPU."""
        self.adjust_calls += 1
        self.adjust_bucket_scans += len(self.buckets)
        edges = self.edges()
        counts = self._current_counts()
        if counts is not None:  # K2 on the incremental histogram (C*L words uploaded)
            sched = _scheduler(1, max_seq_len=self.max_seq_len, n_classes=1,
                               policies=(DispatchPolicy.FCFS,),
                               split_threshold=self.split_threshold, kv_bytes_per_token=1,
                               current_safe=0, truncate=False)
            new_edges, changes, _ = sched.boundaries_from_hist(
                counts, init_edges=edges, n_max=int(n_max), max_passes=1)
        else:  # a queued length outside [0, L): K1 latches it and the reference error is raised
            reqs = list(self.iter_requests())
            lens = np.fromiter((r.input_len for r in reqs), np.int32, len(reqs))
            sched = _scheduler(len(reqs), max_seq_len=self.max_seq_len, n_classes=1,
                               policies=(DispatchPolicy.FCFS,),
                               split_threshold=self.split_threshold, kv_bytes_per_token=1,
                               current_safe=0, truncate=False)
            new_edges, changes, _ = sched.boundaries(lens, init_edges=edges, n_max=int(n_max),
                                                     max_passes=1)
        new_edges = [int(e) for e in new_edges]
        if not changes:
            self.dirty = False
            return []
        if changes[0].kind == "merge":  # bucket_manager.py:148-156
            merged = sorted(self.iter_requests(), key=_ARRIVAL_ORDER)
            self.requests_moved += len(merged)
            self.buckets = [Bucket(0, self.max_seq_len, deque(merged), self._counts)]
            return changes
        split_mid = {c.parent_low: c.midpoint for c in changes if c.kind == "split"}
        new_buckets: list[Bucket] = []
        for b in self.buckets:  # stable partition, bucket_manager.py:171-188
            mid = split_mid.get(b.low)
            if mid is None:
                new_buckets.append(b)
                continue
            left = Bucket(b.low, mid, deque(r for r in b.requests if r.input_len < mid),
                          b._counts)
            right = Bucket(mid, b.up, deque(r for r in b.requests if r.input_len >= mid),
                           b._counts)
            self.requests_moved += len(b.requests)
            new_buckets.extend((left, right))
        self.buckets = new_buckets
        assert self.edges() == new_edges
        if all(c.kind == "skip" for c in changes):
            self.dirty = False
        return changes

    def check_partition(self) -> PartitionViolation | None:
        """bucket_manager.py:193-216."""
        if not self.buckets:
            return PartitionViolation("gap", f"no buckets cover [0, {self.max_seq_len})")
        if self.buckets[0].low != 0:
            return PartitionViolation("gap", f"no bucket covers [0, {self.buckets[0].low})")
        if self.buckets[-1].up != self.max_seq_len:
            return PartitionViolation(
                "gap", f"no bucket covers [{self.buckets[-1].up}, {self.max_seq_len})")
        for b in self.buckets:
            if not 0 <= b.low < b.up <= self.max_seq_len:
                return PartitionViolation("bounds", f"bucket [{b.low}, {b.up}) is malformed")
        for a, b in zip(self.buckets, self.buckets[1:]):
            if a.up < b.low:
                return PartitionViolation("gap", f"gap at [{a.up}, {b.low})")
            if a.up > b.low:
                return PartitionViolation("overlap", f"overlap at [{b.low}, {a.up})")
        for b in self.buckets:
            for r in b.requests:
                if not b.low <= r.input_len < b.up:
                    return PartitionViolation(
                        "misfiled", f"request {r.id} with length {r.input_len} sits in [{b.low}, {b.up})")
        return None


# ---- batch_controller.py --------------------------------------------------------------
class BatchController:
    """batch_controller.py:70-191; form_batch sizing runs on the GPU (K4 + K5)."""

    def __init__(self, model: ModelConfig, gpu: GpuConfig,
                 accounting: MemoryAccounting = MemoryAccounting.PADDED):
        self.model = model
        self.gpu = gpu
        self.accounting = accounting
        self.base_safe = safe_memory(gpu)
        self.current_safe = self.base_safe
        self.kv_per_token = model.kv_bytes_per_token
        self.rejections: list[OversizeRejection] = []

    def on_memory_change(self, new_safe: int) -> int:
        if new_safe < 0:
            raise ValueError("safe memory must be >= 0")
        self.current_safe = new_safe
        return self.token_budget()

    def token_budget(self) -> int:
        return self.current_safe // self.kv_per_token

    def current_n_max(self, bucket_set: BucketSet) -> int:
        total = bucket_set.total_requests
        if total == 0:
            return 1
        mean_len = sum(r.input_len for r in bucket_set.iter_requests()) / total
        return max(1, int(self.token_budget() // mean_len))

    def select_bucket(self, bucket_set: BucketSet, task_class) -> int | None:
        if task_class is TaskClass.ONLINE:
            best_idx, best_key = None, None
            for idx, bucket in enumerate(bucket_set.buckets):
                for r in bucket.requests:
                    if r.task_class is not TaskClass.ONLINE:
                        continue
                    key = (r.arrival_time, r.id)
                    if best_key is None or key < best_key:
                        best_key, best_idx = key, idx
            return best_idx
        best_idx, best_mass = None, 0
        for idx, bucket in enumerate(bucket_set.buckets):
            mass = sum(r.input_len for r in bucket.requests if r.task_class is TaskClass.OFFLINE)
            if mass > best_mass:
                best_mass, best_idx = mass, idx
        return best_idx

    def _footprint(self, max_len: int, count: int, token_sum: int) -> int:
        if self.accounting is MemoryAccounting.PADDED:
            return self.kv_per_token * max_len * count
        return self.kv_per_token * token_sum

    def form_batch(self, bucket: Bucket, policy: DispatchPolicy, *, pledged: int = 0,
                   task_class=None, now: float = 0.0) -> BatchPlan | None:
        """batch_controller.py:141-191: the first batch of the bucket's drain."""
        headroom = self.current_safe - pledged
        if headroom <= 0:
            return None
        cands = [r for r in bucket.requests if task_class is None or r.task_class is task_class]
        if not cands:
            return None
        # arrival rank = (arrival_time, id) order (order_requests' tie-break)
        cands.sort(key=_ARRIVAL_ORDER)
        lens = np.fromiter((r.input_len for r in cands), np.int64, len(cands))
        L = int(max(self.model.max_seq_len, int(lens.max()) + 1))
        sched = _scheduler(len(cands), max_seq_len=L, n_classes=1, policies=(policy,),
                           adjust=False, kv_bytes_per_token=self.kv_per_token,
                           current_safe=self.current_safe, pledged=pledged,
                           accounting=self.accounting, truncate=False)
        res = sched.schedule(lens.astype(np.int32), np.zeros(len(cands), np.uint8))
        rb = res.req_batch.cpu().numpy()
        rr = res.req_row.cpu().numpy()
        b = res.batches()
        # the first form_batch call consumes positions [start_0, end_0) (or, when it
        # admits nothing, the rejected prefix before the blocking request)
        perm = res.perm.cpu().numpy()
        if len(b):
            end = int(b[0]["end"])
        else:
            end = len(perm)
            for j, i in enumerate(perm):
                if rb[i] == N.REQ_PENDING:
                    end = j
                    break
        admitted: list[Request] = [None] * (int(b[0]["n"]) if len(b) else 0)
        removed: set = set()
        for j in range(end):
            i = int(perm[j])
            r = cands[i]
            if rb[i] == N.REQ_REJECTED:
                self.rejections.append(OversizeRejection(r, self.kv_per_token * r.input_len,
                                                         self.current_safe))
                removed.add(r.id)
            elif rb[i] == 0:
                admitted[int(rr[i])] = r
                removed.add(r.id)
        if removed:
            bucket.remove_ids(removed)
        if not admitted:
            return None
        m = int(b[0]["max_input_len"])
        s = int(b[0]["token_sum"])
        return BatchPlan(request_ids=tuple(r.id for r in admitted), requests=tuple(admitted),
                         max_input_len=m, token_sum=s, footprint=int(b[0]["footprint"]),
                         created_at=now, source_bucket=(bucket.low, bucket.up))


# ---- whole window from reference objects ------------------------------------------------
@dataclass
class WindowSchedule:
    """Reference-shaped result of one window."""
    bucket_set: BucketSet
    changes: list
    n_max: int
    plans: list
    rejections: list
    pending: list


def schedule_requests(requests: Sequence[Request], model: ModelConfig, gpu: GpuConfig, *,
                      accounting: MemoryAccounting = MemoryAccounting.PADDED,
                      offline_policy: DispatchPolicy = DispatchPolicy.SJF,
                      split_threshold: float = 0.5, buckets: Sequence[int] | None = None,
                      adjust: bool = True, pledged: int = 0, truncate: bool = True,
                      now: float = 0.0, tok_off=None, tokens=None,
                      dispatch: bool = False) -> WindowSchedule:
    """The reference window composition on the GPU: assign every request,
    adjust_buckets(current_n_max) to the fixpoint, then for every bucket and class
    (ONLINE first) drain form_batch.  Requests may come in any order; the arrival
    rank is (arrival_time, id) as in order_requests.  Over-long inputs are scheduled
    at max_seq_len - 1 (pd_sim.py:382-383) without mutating the caller's objects.

    dispatch=True returns the plans in the order the simulator would start them
    instead — Simulator._next_plan repeated while it makes progress (pd_sim.py:448-462,
    select_bucket batch_controller.py:106-134) — computed by the K7 kernels; requests
    the loop never reaches stay pending."""
    L = model.max_seq_len
    reqs = sorted(requests, key=_ARRIVAL_ORDER)
    classes = [TaskClass.ONLINE, TaskClass.OFFLINE]
    lens = np.fromiter((r.input_len for r in reqs), np.int32, len(reqs))
    cls = np.fromiter((_class_index(r.task_class, classes) for r in reqs), np.uint8, len(reqs))
    sched = _scheduler(len(reqs), max_seq_len=L, n_classes=2,
                       policies=(DispatchPolicy.EARLIEST_ARRIVAL, offline_policy),
                       split_threshold=split_threshold, adjust=adjust,
                       buckets=None if buckets is None else tuple(buckets),
                       kv_bytes_per_token=model.kv_bytes_per_token,
                       current_safe=safe_memory(gpu), pledged=pledged,
                       accounting=accounting, truncate=truncate, dispatch=dispatch)
    res = sched.schedule(lens, cls, tok_off, tokens)
    h = res.to_host()
    edges = [int(e) for e in h["edges"]]
    b = h["batches"]
    rb, rr, perm = h["req_batch"], h["req_row"], h["perm"]
    plans, rejections = [], []
    members: list[list] = [[None] * int(x["n"]) for x in b]
    safe = safe_memory(gpu)
    for j in range(len(perm)):
        i = int(perm[j])
        if rb[i] >= 0:
            members[int(rb[i])][int(rr[i])] = reqs[i]
        elif rb[i] == N.REQ_REJECTED:
            rejections.append(OversizeRejection(reqs[i], model.kv_bytes_per_token * reqs[i].input_len,
                                                safe))
    C = 2
    order = h["emit_order"] if dispatch else range(len(b))
    for k in order:
        x = b[int(k)]
        bk = int(x["segment"]) // C
        plans.append(BatchPlan(request_ids=tuple(r.id for r in members[int(k)]),
                               requests=tuple(members[int(k)]), max_input_len=int(x["max_input_len"]),
                               token_sum=int(x["token_sum"]), footprint=int(x["footprint"]),
                               created_at=now, source_bucket=(edges[bk], edges[bk + 1])))
    bs = BucketSet(L, split_threshold,
                   buckets=[Bucket(lo, up) for lo, up in zip(edges[:-1], edges[1:])])
    pending = []
    for i in range(len(reqs)):
        if rb[i] == N.REQ_PENDING:
            pending.append(reqs[i])
            bs.buckets[int(h["bucket"][i])].add(reqs[i])
    return WindowSchedule(bucket_set=bs, changes=res.changes(), n_max=int(h["summary"]["n_max"]),
                          plans=plans, rejections=rejections, pending=pending)
