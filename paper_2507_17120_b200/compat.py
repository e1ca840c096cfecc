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
import copy
import heapq
from collections import deque
from dataclasses import dataclass
from operator import attrgetter
from typing import Iterator, Sequence

import numpy as np

from . import _native as N
from .memory_model import GpuConfig, LengthHistogram, ModelConfig, safe_memory
from .types import (BatchPlan, DispatchPolicy, MemoryAccounting, OversizeRejection,
                    PartitionViolation, Request, StructuralChange, TaskClass, enum_value,
                    is_online, is_offline)

_ARRIVAL_ORDER = attrgetter("arrival_time", "id")


def order_requests(requests: Sequence[Request], policy: DispatchPolicy) -> list[Request]:
    """batch_controller.py:33-41 (object-level helper; the window path orders on the GPU)."""
    v = enum_value(policy)
    if v == DispatchPolicy.SJF.value:
        key = lambda r: (r.input_len, r.arrival_time, r.id)  # noqa: E731
    elif v == DispatchPolicy.LJF.value:
        key = lambda r: (-r.input_len, r.arrival_time, r.id)  # noqa: E731
    else:
        key = lambda r: (r.arrival_time, r.id)  # noqa: E731
    return sorted(requests, key=key)


# ---- scheduler pool: one WindowScheduler per buffer shape ---------------------------
# Keyed only by what sizes the buffers (device, L, classes, dispatch); the memory state,
# policies, threshold and edges of a call are applied with WindowScheduler.configure,
# so varying current_safe / pledged does not allocate new contexts.
_POOL: dict = {}
_WINDOW_DEFAULTS = dict(split_threshold=0.5, adjust=True, max_passes=0, n_max=None, pledged=0,
                        accounting=MemoryAccounting.PADDED, truncate=True, pad_id=0)


def _scheduler(n: int, *, max_seq_len: int, n_classes: int, dispatch: bool = False,
               buckets=None, **params):
    import torch

    from .window import WindowScheduler
    params = {**_WINDOW_DEFAULTS, **params}
    key = (torch.cuda.current_device(), int(max_seq_len), int(n_classes), bool(dispatch))
    s = _POOL.get(key)
    if s is not None and s.max_requests < n:
        s.close()
        s = None
    if s is None:
        cap = max(1024, 1 << max(0, int(n - 1).bit_length()))
        s = WindowScheduler(max_requests=cap, max_seq_len=max_seq_len, n_classes=n_classes,
                            dispatch=dispatch, buckets=buckets, **params)
        _POOL[key] = s
    else:
        s.configure(buckets=buckets, **params)
    return s


def release_pool() -> None:
    """Free every pooled GPU context (tests / long-lived callers)."""
    for s in _POOL.values():
        s.close()
    _POOL.clear()


def _class_index(task_class, classes: list) -> int:
    v = enum_value(task_class)
    for i, c in enumerate(classes):
        if v == enum_value(c):
            return i
    raise ValueError(f"unknown task class {task_class!r}")


def _class_matches(r, task_class) -> bool:
    """form_batch's filter (`r.task_class is task_class`, batch_controller.py:155) with
    enum members compared by value (see types.enum_value)."""
    return task_class is None or enum_value(r.task_class) == enum_value(task_class)


# ---- bucket_manager.py ---------------------------------------------------------------
class Bucket:
    """bucket_manager.py:22-53 — `low`, `up`, `mid`, `short_count`, the FIFO deque
    `requests`, `add`, `remove_ids`, `token_mass`.

    Beyond the reference it keeps what the stateful path reads per call current in O(1):
    per-class aggregates for select_bucket (queued OFFLINE token mass; a heap of ONLINE
    (arrival_time, id) keys with lazy deletion), the owning set's per-length histogram,
    and form_batch's cached drains.  Requests form_batch removes are tombstoned and the
    deque is compacted the next time `requests` is read, so a drain costs O(batch) per
    call instead of the reference's O(bucket) rebuild (bucket_manager.py:42-50).
    Changes made to the deque behind the bucket's back are detected by its length and
    the aggregates recomputed."""

    __slots__ = ("low", "up", "mid", "short_count", "_dq", "_dead", "_counts", "_n",
                 "_offline_mass", "_online", "_gone", "_version", "_drains")

    def __init__(self, low: int, up: int, requests=None, _counts: np.ndarray | None = None):
        self.low = low
        self.up = up
        self._counts = _counts
        self._dq: deque = requests if requests is not None else deque()
        self._dead: set = set()
        self._version = 0
        self._drains: dict = {}
        self.mid = (self.low + self.up) // 2
        self.short_count = sum(1 for r in self._dq if r.input_len < self.mid)
        self._reset_aggregates()

    # -- reference surface --
    @property
    def requests(self) -> deque:
        if self._dead:
            self._compact()
        return self._dq

    @requests.setter
    def requests(self, value) -> None:
        self._dq = value
        self._dead = set()
        self._touch()
        self._reset_aggregates()

    def __len__(self) -> int:
        return len(self._dq) - len(self._dead)

    def __repr__(self) -> str:
        return f"Bucket(low={self.low}, up={self.up}, requests={self.requests!r})"

    def __eq__(self, other) -> bool:
        if not isinstance(other, Bucket):
            return NotImplemented
        return (self.low, self.up, list(self.requests)) == (other.low, other.up,
                                                            list(other.requests))

    __hash__ = None

    def add(self, request: Request) -> None:
        if self._dead and id(request) in self._dead:
            self._compact()  # re-added before its tombstone was compacted away
        self._dq.append(request)
        if request.input_len < self.mid:
            self.short_count += 1
        if self._counts is not None:
            self._counts[request.input_len] += 1
        self._agg_add(request)
        self._touch()

    def remove_ids(self, ids: set) -> None:
        kept: deque = deque()
        for r in self.requests:
            if r.id in ids:
                if r.input_len < self.mid:
                    self.short_count -= 1
                if self._counts is not None:
                    self._counts[r.input_len] -= 1
                self._agg_remove(r)
            else:
                kept.append(r)
        self._dq = kept
        self._touch()

    def token_mass(self) -> int:
        return sum(r.input_len for r in self.requests)

    # -- bookkeeping --
    def _touch(self) -> None:
        self._version += 1
        self._drains.clear()

    def _compact(self) -> None:
        dead = self._dead
        self._dq = deque(r for r in self._dq if id(r) not in dead)
        self._dead = set()

    @classmethod
    def _split_of(cls, b: "Bucket", mid: int) -> tuple["Bucket", "Bucket"]:
        """The stable partition of `b` at `mid` (bucket_manager.py:171-188) with both
        children's aggregates (short counts, OFFLINE mass, ONLINE heap) gathered in the
        same single pass over the parent's requests."""
        kind: dict = {}  # task-class object -> 1 online, 2 offline, 0 other
        parts = []
        for lo, up in ((b.low, mid), (mid, b.up)):
            c = cls.__new__(cls)
            c.low, c.up, c._counts = lo, up, b._counts
            c._dq, c._dead, c._version, c._drains, c._gone = deque(), set(), 0, {}, {}
            c.mid = (lo + up) // 2
            parts.append(c)
        left, right = parts
        lq, rq = left._dq.append, right._dq.append
        lmid, rmid = left.mid, right.mid
        l_short = r_short = l_off = r_off = 0
        l_on, r_on = [], []
        for r in b.requests:
            x = r.input_len
            tc = r.task_class
            k = kind.get(tc)
            if k is None:
                k = kind[tc] = 1 if is_online(tc) else (2 if is_offline(tc) else 0)
            if x < mid:
                lq(r)
                if x < lmid:
                    l_short += 1
                if k == 2:
                    l_off += x
                elif k == 1:
                    l_on.append((r.arrival_time, r.id))
            else:
                rq(r)
                if x < rmid:
                    r_short += 1
                if k == 2:
                    r_off += x
                elif k == 1:
                    r_on.append((r.arrival_time, r.id))
        for c, sc, off, on in ((left, l_short, l_off, l_on), (right, r_short, r_off, r_on)):
            heapq.heapify(on)
            c.short_count, c._offline_mass, c._online, c._n = sc, off, on, len(c._dq)
        return left, right

    def _reset_aggregates(self) -> None:
        live = [r for r in self._dq if id(r) not in self._dead] if self._dead else self._dq
        self._n = len(live)
        self._offline_mass = sum(r.input_len for r in live if is_offline(r.task_class))
        self._online = [(r.arrival_time, r.id) for r in live if is_online(r.task_class)]
        heapq.heapify(self._online)
        self._gone: dict = {}

    def _agg_add(self, r) -> None:
        self._n += 1
        if is_offline(r.task_class):
            self._offline_mass += r.input_len
        elif is_online(r.task_class):
            heapq.heappush(self._online, (r.arrival_time, r.id))

    def _agg_remove(self, r) -> None:
        self._n -= 1
        if is_offline(r.task_class):
            self._offline_mass -= r.input_len
        elif is_online(r.task_class):
            k = (r.arrival_time, r.id)
            self._gone[k] = self._gone.get(k, 0) + 1

    def _aggregates_current(self) -> None:
        if self._n != len(self):  # the deque was changed behind the bucket's back
            self._reset_aggregates()
            self._touch()

    def _oldest_online(self):
        self._aggregates_current()
        h, gone = self._online, self._gone
        while h and gone.get(h[0]):
            gone[h[0]] -= 1
            heapq.heappop(h)
        return h[0] if h else None

    def _queued_offline_mass(self) -> int:
        self._aggregates_current()
        return self._offline_mass

    def _consume(self, reqs) -> None:
        """Remove the given request objects (those a cached drain call consumed) in
        O(len(reqs)): tombstones + the same counter updates as remove_ids."""
        dead = self._dead
        for r in reqs:
            dead.add(id(r))
            if r.input_len < self.mid:
                self.short_count -= 1
            if self._counts is not None:
                self._counts[r.input_len] -= 1
            self._agg_remove(r)
        self._version += 1
        if len(dead) > 64 and 2 * len(dead) > len(self._dq):
            self._compact()


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
        self._lengths = np.arange(max_seq_len, dtype=np.int64)
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
                and all(b._n == len(b) for b in self.buckets)
                and int(self._counts.sum()) == self.total_requests):
            return self._counts
        return self._counts if self._rebuild_counts() else None

    def queued_length_sum(self) -> int:
        """Σ input_len over the queued requests from the histogram (O(L))."""
        counts = self._current_counts()
        if counts is None:
            return sum(r.input_len for r in self.iter_requests())
        return int(counts @ self._lengths)

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
        self.buckets[idx].add(request)
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
            left, right = Bucket._split_of(b, mid)
            self.requests_moved += len(left) + len(right)
            new_buckets.extend((left, right))
        self.buckets = new_buckets
        assert self.edges() == new_edges
        if all(c.kind == "skip" for c in changes):
            self.dirty = False
        return changes

    def length_histogram(self, bins: int = 64) -> LengthHistogram:
        """The simulator's monitor histogram of the queued lengths
        (LengthHistogram.from_samples(lengths, bins, (0, max_seq_len)), pd_sim.py:829-831),
        binned on the GPU from the incremental per-length counts (f2)."""
        return _monitor(self, bins)[0]

    def expected_waste(self, bins: int = 64) -> float:
        """expected_waste(length_histogram(bins), [(b.low, b.up) ...]) — the per-tick
        monitor statistic (pd_sim.py:828-833, memory_model.py:160-191), on the GPU."""
        return _monitor(self, bins)[1]

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


@dataclass(frozen=True)
class BoundaryFit:
    """bucket_manager.py:219-223."""
    boundary: float
    iterations: int
    converged: bool


def optimal_boundary_oracle(hist: LengthHistogram, low: float, up: float, tol: float,
                            max_iters: int = 100) -> BoundaryFit:
    """bucket_manager.py:226-249: the reference's test-only conditional-mean boundary
    (U <- mean(S | low <= S < U) from U = up until it moves by < tol * (up - low)); kept
    for API completeness — the scheduling path uses the midpoint split (K2)."""
    if tol <= 0:
        raise ValueError("tol must be > 0")
    if hist.mass_in(low, up) == 0:
        raise ValueError(f"histogram has no mass in [{low}, {up})")
    u, eps = float(up), tol * (up - low)
    for it in range(1, max_iters + 1):
        m = hist.conditional_mean(low, u)
        if m is None:
            return BoundaryFit(u, it, True)
        if abs(u - m) < eps:
            return BoundaryFit(m, it, True)
        u = m
    return BoundaryFit(u, max_iters, False)


def _monitor(bs: BucketSet, bins: int):
    """(LengthHistogram, expected_waste) of the set's queued requests (f2, K8 on the
    GPU over the incremental histogram; the reference errors for an empty queue)."""
    counts = bs._current_counts()
    if counts is None:
        raise ValueError("a queued length lies outside [0, max_seq_len)")
    sched = _scheduler(1, max_seq_len=bs.max_seq_len, n_classes=1,
                       policies=(DispatchPolicy.FCFS,), kv_bytes_per_token=1, current_safe=0,
                       truncate=False)
    return sched.monitor_from_hist(counts, bs.edges(), bins=bins)


# ---- batch_controller.py --------------------------------------------------------------
class _Drain:
    """form_batch's calls on one bucket for one (class, policy, pledged, memory) key,
    computed once on the GPU (K4 + K5 over the class-filtered bucket) and handed out
    one call at a time while the bucket is unchanged."""

    __slots__ = ("cands", "calls", "pos", "version")

    def __init__(self, cands, calls, version):
        self.cands = cands
        self.calls = calls      # [(rejected idx array, admitted idx array, meta | None)]
        self.pos = 0
        self.version = version


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
        """batch_controller.py:93-104; Σ input_len from the set's incremental histogram
        (O(L)) instead of a pass over every queued request."""
        total = bucket_set.total_requests
        if total == 0:
            return 1
        mean_len = bucket_set.queued_length_sum() / total
        return max(1, int(self.token_budget() // mean_len))

    def select_bucket(self, bucket_set: BucketSet, task_class) -> int | None:
        """batch_controller.py:106-134 over per-bucket aggregates kept by the buckets
        (O(K) per call instead of O(queued requests))."""
        if is_online(task_class):
            best_idx, best_key = None, None
            for idx, bucket in enumerate(bucket_set.buckets):
                key = bucket._oldest_online()
                if key is not None and (best_key is None or key < best_key):
                    best_key, best_idx = key, idx
            return best_idx
        best_idx, best_mass = None, 0
        for idx, bucket in enumerate(bucket_set.buckets):
            mass = bucket._queued_offline_mass()
            if mass > best_mass:
                best_mass, best_idx = mass, idx
        return best_idx

    def _footprint(self, max_len: int, count: int, token_sum: int) -> int:
        if enum_value(self.accounting) == MemoryAccounting.PADDED.value:
            return self.kv_per_token * max_len * count
        return self.kv_per_token * token_sum

    def _plan_drain(self, bucket: Bucket, policy, pledged: int, task_class) -> _Drain:
        """The whole drain of the bucket's class-filtered candidates (form_batch
        repeated until it returns None), from one K4 + K5 launch sequence."""
        cands = [r for r in bucket.requests if _class_matches(r, task_class)]
        calls = []
        if cands:
            # arrival rank = (arrival_time, id) order (order_requests' tie-break)
            cands.sort(key=_ARRIVAL_ORDER)
            lens = np.fromiter((r.input_len for r in cands), np.int64, len(cands))
            L = int(max(self.model.max_seq_len, int(lens.max()) + 1))
            sched = _scheduler(len(cands), max_seq_len=L, n_classes=1, policies=(policy,),
                               adjust=False, kv_bytes_per_token=self.kv_per_token,
                               current_safe=self.current_safe, pledged=pledged,
                               accounting=self.accounting, truncate=False)
            res = sched.schedule(lens.astype(np.int32), np.zeros(len(cands), np.uint8))
            perm = res.perm.cpu().numpy()
            rb = res.req_batch.cpu().numpy()[perm]       # outcome in drain order
            b = res.batches()
            lo = 0
            for k in range(len(b)):
                hi = int(b[k]["end"])
                seg_pos = np.arange(lo, hi)
                calls.append((perm[seg_pos[rb[lo:hi] == N.REQ_REJECTED]],
                              perm[seg_pos[rb[lo:hi] == k]],
                              (int(b[k]["max_input_len"]), int(b[k]["token_sum"]),
                               int(b[k]["footprint"]))))
                lo = hi
            # the call after the last batch removes the rejected requests before the
            # blocking one (or the rest) and admits nothing
            pend = np.nonzero(rb[lo:] == N.REQ_PENDING)[0]
            hi = lo + (int(pend[0]) if len(pend) else len(perm) - lo)
            if hi > lo:
                calls.append((perm[lo:hi], perm[:0], None))
        return _Drain(cands, calls, bucket._version)

    def form_batch(self, bucket: Bucket, policy: DispatchPolicy, *, pledged: int = 0,
                   task_class=None, now: float = 0.0) -> BatchPlan | None:
        """batch_controller.py:141-191: the next batch of the bucket's drain.  The drain
        is computed on the GPU once per (bucket state, class, policy, pledged, memory)
        and its calls are handed out while the bucket is unchanged."""
        headroom = self.current_safe - pledged
        if headroom <= 0:
            return None
        key = (enum_value(task_class) if task_class is not None else None, enum_value(policy),
               pledged, self.current_safe, enum_value(self.accounting), self.kv_per_token)
        bucket._aggregates_current()
        d = bucket._drains.get(key)
        if d is None or d.version != bucket._version:
            d = self._plan_drain(bucket, policy, pledged, task_class)
            bucket._drains[key] = d
        if d.pos >= len(d.calls):
            return None
        rej_idx, adm_idx, meta = d.calls[d.pos]
        d.pos += 1
        cands = d.cands
        for i in rej_idx:
            r = cands[i]
            self.rejections.append(OversizeRejection(r, self.kv_per_token * r.input_len,
                                                     self.current_safe))
        admitted = tuple(cands[i] for i in adm_idx)
        consumed = [cands[i] for i in rej_idx]
        consumed.extend(admitted)
        if consumed:
            # drains of other classes on this bucket stay valid: their candidates are
            # untouched; any drain over this class (or over all classes) is dropped
            before = bucket._version
            bucket._consume(consumed)
            for k2, d2 in list(bucket._drains.items()):
                if d2 is d or (k2[0] is not None and key[0] is not None and k2[0] != key[0]
                               and d2.version == before):
                    d2.version = bucket._version
                else:
                    del bucket._drains[k2]
        if meta is None:
            return None
        m, s, fp = meta
        return BatchPlan(request_ids=tuple(r.id for r in admitted), requests=admitted,
                         max_input_len=m, token_sum=s, footprint=fp,
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
            r = reqs[i]
            pending.append(r)
            if r.input_len >= L and truncate:
                # filed under L - 1 like the simulator's truncated copy (pd_sim.py:382-383);
                # the caller's object is left as it was
                r = copy.copy(r)
                r.input_len = L - 1
            bs.buckets[int(h["bucket"][i])].add(r)
    return WindowSchedule(bucket_set=bs, changes=res.changes(), n_max=int(h["summary"]["n_max"]),
                          plans=plans, rejections=rejections, pending=pending)
