"""The GPU-backed BucketSet's incremental per-length histogram — host
bookkeeping only, no GPU: +1 on assign / Bucket.add, -1 on remove_ids, carried through
splits and merges, revalidated against the queued total and recounted when the deques
are changed behind the set's back."""
from collections import deque

import numpy as np

from paper_2507_17120_b200.compat import Bucket, BucketSet
from paper_2507_17120_b200.types import Request, TaskClass


def _req(rid, length):
    return Request(rid, float(rid), length, 10, TaskClass.OFFLINE)


def _expected(bs):
    h = np.zeros(bs.max_seq_len, np.int64)
    for r in bs.iter_requests():
        h[r.input_len] += 1
    return h


def test_counts_track_assign_add_remove():
    bs = BucketSet(64, buckets=[Bucket(0, 16), Bucket(16, 64, deque([_req(100, 20), _req(101, 63)]))])
    assert np.array_equal(bs._counts, _expected(bs))
    rng = np.random.default_rng(5)
    for i in range(200):
        bs.assign(_req(i, int(rng.integers(0, 64))))
    assert np.array_equal(bs._counts, _expected(bs))
    bs.buckets[1].add(_req(500, 30))
    ids = {r.id for r in list(bs.buckets[1].requests)[::3]}
    bs.buckets[1].remove_ids(ids)
    assert np.array_equal(bs._counts, _expected(bs))
    assert bs._current_counts() is bs._counts


def test_counts_recount_after_outside_mutation():
    bs = BucketSet(64)
    for i in range(10):
        bs.assign(_req(i, i))
    bs.buckets[0].requests.append(_req(99, 40))       # bypasses assign / add
    assert not np.array_equal(bs._counts, _expected(bs))
    assert np.array_equal(bs._current_counts(), _expected(bs))
    bs.buckets = [Bucket(0, 64, deque([_req(1, 5), _req(2, 6)]))]  # replaced wholesale
    assert np.array_equal(bs._current_counts(), _expected(bs))
    assert all(b._counts is bs._counts for b in bs.buckets)


def test_counts_unavailable_for_out_of_range_lengths():
    bs = BucketSet(64, buckets=[Bucket(0, 64, deque([_req(1, 70)]))])
    assert bs._current_counts() is None  # adjust_buckets then takes the K1 path, which raises


def test_select_bucket_host_aggregates_and_foreign_enums():
    """select_bucket runs on per-bucket aggregates (no GPU); bucketsim-style enum
    members from another Enum class are matched by value; deque edits behind the
    bucket's back are picked up."""
    from enum import Enum

    from paper_2507_17120_b200 import GpuConfig, ModelConfig
    from paper_2507_17120_b200.compat import BatchController

    class TC(Enum):
        ONLINE = "online"
        OFFLINE = "offline"

    def r(i, n, a, c):
        return Request(i, a, n, 1, c)

    b0 = Bucket(0, 100, deque([r(0, 50, 5.0, TC.ONLINE), r(1, 90, 1.0, TC.OFFLINE)]))
    b1 = Bucket(100, 200, deque([r(2, 150, 2.0, TC.ONLINE), r(3, 120, 3.0, TaskClass.OFFLINE)]))
    bs = BucketSet(200, buckets=[b0, b1])
    ctl = BatchController(ModelConfig(1, 1, 1, 2, 200), GpuConfig(10**6, 0, 0.0))
    assert ctl.select_bucket(bs, TC.ONLINE) == 1
    assert ctl.select_bucket(bs, TaskClass.ONLINE) == 1
    assert ctl.select_bucket(bs, TC.OFFLINE) == 1          # 120 > 90
    b1.remove_ids({2, 3})
    assert ctl.select_bucket(bs, TC.ONLINE) == 0
    assert ctl.select_bucket(bs, TC.OFFLINE) == 0
    b1.requests.append(r(9, 199, 0.5, TC.ONLINE))         # behind the bucket's back
    assert ctl.select_bucket(bs, TC.ONLINE) == 1
    b0.requests.clear()
    b1.requests.clear()
    assert ctl.select_bucket(bs, TC.ONLINE) is None and ctl.select_bucket(bs, TC.OFFLINE) is None
    assert ctl.current_n_max(bs) == 1


def test_select_bucket_and_n_max_match_reference_scan_randomised():
    """Aggregates vs the reference's O(N) scans (batch_controller.py:93-134) under
    random add / remove_ids / consume sequences."""
    from paper_2507_17120_b200 import GpuConfig, ModelConfig
    from paper_2507_17120_b200.compat import BatchController
    rng = np.random.default_rng(9)
    bs = BucketSet(256, buckets=[Bucket(0, 64), Bucket(64, 128), Bucket(128, 256)])
    ctl = BatchController(ModelConfig(1, 1, 1, 2, 256), GpuConfig(10**7, 0, 0.0))
    live = []
    for step in range(3000):
        if rng.random() < 0.6 or not live:
            req = Request(step, float(rng.integers(0, 500)), int(rng.integers(0, 256)), 1,
                          [TaskClass.ONLINE, TaskClass.OFFLINE][int(rng.integers(0, 2))])
            bs.assign(req)
            live.append(req)
        else:
            b = bs.buckets[int(rng.integers(0, 3))]
            qs = list(b.requests)
            if qs:
                pick = [qs[int(i)] for i in rng.integers(0, len(qs), int(rng.integers(1, 4)))]
                if rng.random() < 0.5:
                    b.remove_ids({x.id for x in pick})
                else:
                    b._consume(list({id(x): x for x in pick}.values()))
        for cls in (TaskClass.ONLINE, TaskClass.OFFLINE):
            want = _ref_select(bs, cls)
            assert ctl.select_bucket(bs, cls) == want, step
        total = bs.total_requests
        want_n = 1 if total == 0 else max(1, int(ctl.token_budget() // (
            sum(x.input_len for x in bs.iter_requests()) / total)))
        assert ctl.current_n_max(bs) == want_n


def _ref_select(bs, cls):
    if cls is TaskClass.ONLINE:
        best_idx, best_key = None, None
        for idx, b in enumerate(bs.buckets):
            for r in b.requests:
                if r.task_class is not TaskClass.ONLINE:
                    continue
                key = (r.arrival_time, r.id)
                if best_key is None or key < best_key:
                    best_key, best_idx = key, idx
        return best_idx
    best_idx, best_mass = None, 0
    for idx, b in enumerate(bs.buckets):
        mass = sum(r.input_len for r in b.requests if r.task_class is TaskClass.OFFLINE)
        if mass > best_mass:
            best_mass, best_idx = mass, idx
    return best_idx
