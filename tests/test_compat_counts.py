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
