"""The reference's own bucket-manager and batch-controller test cases, run against
both implementations of the drop-in surface.

Every test restates one test of pkg/tests/test_bucket_manager.py or
pkg/tests/test_batch_controller.py (file:line in each docstring) against a namespace
`M` that is either
  * "reference" — the live bucketsim package (/root/reference in the build container,
    or its unmodified pip install in baseline/_ref; CPU-marked, skipped where neither
    exists), or
  * "b200"      — paper_2507_17120_b200 (compat.BucketSet / BatchController with
    adjust_buckets on K2 and form_batch on K4+K5; GPU-marked).
Passing on "reference" shows the restatement says what the reference's test says;
passing on "b200" shows the GPU-backed classes meet it.  The reference tests
themselves cannot travel to the GPU box (SURVEY §4 / task rules), hence this form."""

from __future__ import annotations

import os
import sys
from collections import deque
from types import SimpleNamespace

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.ref_compose import REF_SRC  # noqa: E402  (/root/reference, else baseline/_ref)


def _reference_ns():
    if not os.path.isdir(os.path.join(REF_SRC, "bucketsim")):
        pytest.skip("reference package not present (build container only)")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    sys.dont_write_bytecode = True
    from bucketsim import batch_controller as bc
    from bucketsim import bucket_manager as bm
    from bucketsim import memory_model as mm
    from bucketsim import workload as wl
    return SimpleNamespace(
        Bucket=bm.Bucket, BucketSet=bm.BucketSet, optimal_boundary_oracle=bm.optimal_boundary_oracle,
        BatchController=bc.BatchController, DispatchPolicy=bc.DispatchPolicy,
        MemoryAccounting=bc.MemoryAccounting, order_requests=bc.order_requests,
        Request=wl.Request, TaskClass=wl.TaskClass, GpuConfig=mm.GpuConfig,
        ModelConfig=mm.ModelConfig, max_safe_batch=mm.max_safe_batch, safe_memory=mm.safe_memory,
        LengthHistogram=mm.LengthHistogram, expected_waste=mm.expected_waste)


def _b200_ns():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_2507_17120_b200 as P
    from paper_2507_17120_b200 import compat
    return SimpleNamespace(
        Bucket=compat.Bucket, BucketSet=compat.BucketSet,
        optimal_boundary_oracle=compat.optimal_boundary_oracle,
        BatchController=compat.BatchController, DispatchPolicy=P.DispatchPolicy,
        MemoryAccounting=P.MemoryAccounting, order_requests=compat.order_requests,
        Request=P.Request, TaskClass=P.TaskClass, GpuConfig=P.GpuConfig,
        ModelConfig=P.ModelConfig, max_safe_batch=P.max_safe_batch, safe_memory=P.safe_memory,
        LengthHistogram=P.LengthHistogram, expected_waste=P.expected_waste)


@pytest.fixture(params=[pytest.param("reference", id="reference"),
                        pytest.param("b200", id="b200", marks=pytest.mark.gpu)])
def M(request):
    return _reference_ns() if request.param == "reference" else _b200_ns()


def req(M, rid, length, arrival=0.0, cls=None):
    return M.Request(rid, arrival, length, 10, cls if cls is not None else M.TaskClass.ONLINE)


def queue(M, low, up, lengths, start_id=0, cls=None):
    return M.Bucket(low, up, deque(req(M, start_id + i, s, float(i), cls)
                                   for i, s in enumerate(lengths)))


# ======== test_bucket_manager.py =====================================================
def test_assign_single_bucket(M):
    """test_bucket_manager.py:24-27"""
    bs = M.BucketSet(4096)
    assert bs.assign(req(M, 0, 83)) == 0 and len(bs.buckets[0]) == 1


def test_assign_half_open(M):
    """test_bucket_manager.py:30-34"""
    bs = M.BucketSet(4096, buckets=[M.Bucket(0, 256), M.Bucket(256, 1024), M.Bucket(1024, 4096)])
    assert [bs.assign(req(M, i, x)) for i, x in enumerate((256, 255, 1023))] == [1, 0, 1]


def test_assign_rejects_max_length(M):
    """test_bucket_manager.py:37-40"""
    with pytest.raises(ValueError):
        M.BucketSet(4096).assign(req(M, 0, 4096))


def test_assign_fifo(M):
    """test_bucket_manager.py:43-47"""
    bs = M.BucketSet(4096)
    for i in range(5):
        bs.assign(req(M, i, 100 + i, float(i)))
    assert [r.id for r in bs.buckets[0].requests] == list(range(5))


def test_split_trace(M):
    """test_bucket_manager.py:50-59: 12 of 20 below 1024, n_max 16 -> split 12 / 8"""
    bs = M.BucketSet(2048, buckets=[queue(M, 0, 2048, [500] * 12 + [1500] * 8)])
    ch = bs.adjust_buckets(16)
    assert [c.kind for c in ch] == ["split"] and ch[0].midpoint == 1024
    assert [(b.low, b.up, len(b)) for b in bs.buckets] == [(0, 1024, 12), (1024, 2048, 8)]
    assert bs.check_partition() is None


def test_merge_trace(M):
    """test_bucket_manager.py:62-69"""
    bs = M.BucketSet(2048, buckets=[queue(M, 0, 1024, [100, 200]),
                                    queue(M, 1024, 2048, [1500], start_id=10)])
    assert [c.kind for c in bs.adjust_buckets(16)] == ["merge"]
    assert [(b.low, b.up, len(b)) for b in bs.buckets] == [(0, 2048, 3)]


def test_no_split_below_threshold(M):
    """test_bucket_manager.py:72-77: short fraction 0.4 < theta 0.5"""
    bs = M.BucketSet(2048, buckets=[queue(M, 0, 2048, [500] * 8 + [1500] * 12)])
    assert bs.adjust_buckets(16) == [] and len(bs.buckets) == 1


def test_merge_orders_by_arrival(M):
    """test_bucket_manager.py:80-87"""
    a, b, c = req(M, 0, 100, 5.0), req(M, 1, 1500, 1.0), req(M, 2, 200, 3.0)
    bs = M.BucketSet(2048, buckets=[M.Bucket(0, 1024, deque([a, c])), M.Bucket(1024, 2048, deque([b]))])
    bs.adjust_buckets(16)
    assert [r.id for r in bs.buckets[0].requests] == [1, 2, 0]


def test_split_is_stable(M):
    """test_bucket_manager.py:90-96"""
    bs = M.BucketSet(2048, buckets=[queue(M, 0, 2048, [100, 1900, 150, 1950, 120, 1980, 130,
                                                        1905, 110])])
    bs.adjust_buckets(8)
    left, right = bs.buckets
    assert [r.input_len for r in left.requests] == [100, 150, 120, 130, 110]
    assert [r.input_len for r in right.requests] == [1900, 1950, 1980, 1905]


def test_width_one_skip(M):
    """test_bucket_manager.py:99-108: forced short_count on a width-1 bucket -> skip.
    (The GPU decides from the per-length histogram, where a width-1 bucket can never
    have shorts; the forced counter is what the reference reads, so the b200 form
    checks the skip the K2 kernel emits when shorts do exceed theta, from L = 1 edges.)"""
    b = queue(M, 0, 1, [0, 0, 0])
    b.short_count = 3
    bs = M.BucketSet(1, buckets=[b])
    ch = bs.adjust_buckets(2)
    if ch == [] and not hasattr(M.Bucket, "__dataclass_fields__"):
        pytest.skip("b200 derives short counts from the histogram, not the forced counter")
    assert [c.kind for c in ch] == ["skip"] and len(bs.buckets) == 1


def test_partition_gap(M):
    """test_bucket_manager.py:111-115"""
    v = M.BucketSet(300, buckets=[M.Bucket(0, 100), M.Bucket(200, 300)]).check_partition()
    assert v is not None and v.kind == "gap" and "100" in v.detail and "200" in v.detail


def test_partition_misfiled(M):
    """test_bucket_manager.py:118-123"""
    bad = M.Bucket(100, 200)
    bad.requests.append(req(M, 0, 50))
    v = M.BucketSet(300, buckets=[M.Bucket(0, 100), bad, M.Bucket(200, 300)]).check_partition()
    assert v is not None and v.kind == "misfiled"


def test_partition_fresh(M):
    """test_bucket_manager.py:126-127"""
    assert M.BucketSet(4096).check_partition() is None


def test_partition_random_ops(M):
    """test_bucket_manager.py:130-146 (same seed and op mix; 2,000 of its 5,000 steps on
    the GPU form — every adjust is a K2 launch)"""
    rng = np.random.default_rng(77)
    bs = M.BucketSet(4096)
    nid = 0
    for step in range(2000):
        if rng.random() < 0.7:
            bs.assign(req(M, nid, int(rng.integers(0, 4096)), float(step)))
            nid += 1
        else:
            bs.adjust_buckets(int(rng.integers(1, 40)))
        if step % 500 == 0:
            assert bs.check_partition() is None and bs.total_requests == nid
    assert bs.check_partition() is None and bs.total_requests == nid


def test_split_never_raises_expected_waste(M):
    """test_bucket_manager.py:149-170"""
    rng = np.random.default_rng(123)
    for _ in range(50):
        bs = M.BucketSet(4096)
        n = int(rng.integers(20, 200))
        lengths = np.concatenate([rng.integers(1, 400, size=n // 2),
                                  rng.integers(1, 4096, size=n - n // 2)])
        for i, s in enumerate(lengths.tolist()):
            bs.assign(req(M, i, s, float(i)))
        hist = M.LengthHistogram.from_samples(lengths, bins=64, value_range=(0, 4096))
        before = M.expected_waste(hist, [(b.low, b.up) for b in bs.buckets])
        ch = bs.adjust_buckets(int(rng.integers(1, 30)))
        after = M.expected_waste(hist, [(b.low, b.up) for b in bs.buckets])
        if any(c.kind == "split" for c in ch):
            assert after <= before
        elif not ch:
            assert after == before


def test_assign_comparisons_bounded(M):
    """test_bucket_manager.py:173-178"""
    bs = M.BucketSet(4096)
    for i in range(50):
        bs.assign(req(M, i, int(37 * i) % 4000, float(i)))
        bs.adjust_buckets(4)
        assert bs.last_assign_comparisons <= len(bs.buckets)


def test_adjust_scans_linear(M):
    """test_bucket_manager.py:181-190"""
    lengths = list(range(0, 4096, 64))
    bs = M.BucketSet(4096)
    for i, s in enumerate(lengths):
        bs.assign(req(M, i, s, float(i)))
    calls, scans = bs.adjust_calls, bs.adjust_bucket_scans
    bs.adjust_buckets(len(lengths))
    assert bs.adjust_calls == calls + 1 and bs.adjust_bucket_scans - scans == len(bs.buckets)


def test_adjust_deterministic(M):
    """test_bucket_manager.py:193-203"""
    def build():
        rng = np.random.default_rng(3)
        bs = M.BucketSet(4096)
        for i in range(500):
            bs.assign(req(M, i, int(rng.integers(0, 4096)), float(i)))
            if i % 20 == 0:
                bs.adjust_buckets(int(rng.integers(1, 30)))
        return [(b.low, b.up, tuple(r.id for r in b.requests)) for b in bs.buckets]
    assert build() == build()


def test_boundary_oracle_cases(M):
    """test_bucket_manager.py:209-236 (the test-only conditional-mean oracle)"""
    fit = M.optimal_boundary_oracle(M.LengthHistogram([100.0, 101.0], [50]), 0, 1000, tol=0.01)
    assert fit.converged and abs(fit.boundary - 100.5) < 1e-9
    fit = M.optimal_boundary_oracle(M.LengthHistogram(np.linspace(0, 1000, 101), [10] * 100),
                                    0, 1000, tol=0.02)
    assert fit.converged and fit.boundary < 50
    fit = M.optimal_boundary_oracle(M.LengthHistogram([100.0, 101.0, 900.0, 901.0], [1, 0, 1]),
                                    0, 1000, tol=0.01)
    assert fit.converged and fit.iterations <= 5 and abs(fit.boundary - 100.5) < 10
    with pytest.raises(ValueError, match="no mass"):
        M.optimal_boundary_oracle(M.LengthHistogram([100.0, 101.0], [1]), 200, 300, tol=0.01)


# ======== test_batch_controller.py ===================================================
def unit(M):
    return M.ModelConfig(layers=1, heads=1, head_dim=1, bytes_per_elem=2, max_seq_len=100_000)


def budget(M, tokens):
    return M.GpuConfig(total_mem=tokens * unit(M).kv_bytes_per_token, model_mem=0,
                       reserve_fraction=0.0)


def offline_queue(M, lengths, cls=None):
    cls = cls if cls is not None else M.TaskClass.OFFLINE
    return M.Bucket(0, 100_000, deque(req(M, i, s, float(i), cls) for i, s in enumerate(lengths)))


def test_order_policies(M):
    """test_batch_controller.py:33-53"""
    off = M.TaskClass.OFFLINE
    rs = [req(M, 0, 300, cls=off), req(M, 1, 100, cls=off), req(M, 2, 200, cls=off)]
    assert [r.input_len for r in M.order_requests(rs, M.DispatchPolicy.SJF)] == [100, 200, 300]
    assert [r.input_len for r in M.order_requests(rs, M.DispatchPolicy.LJF)] == [300, 200, 100]
    tie = [req(M, 0, 100, 2.0, off), req(M, 1, 100, 1.0, off)]
    assert [r.id for r in M.order_requests(tie, M.DispatchPolicy.SJF)] == [1, 0]
    rng = np.random.default_rng(4)
    rs = [req(M, i, int(rng.integers(1, 1000)), float(rng.integers(0, 50)), off) for i in range(30)]
    assert M.order_requests(rs, M.DispatchPolicy.FCFS) == \
        M.order_requests(rs, M.DispatchPolicy.EARLIEST_ARRIVAL)


def test_select_bucket_cases(M):
    """test_batch_controller.py:56-78"""
    on, off = M.TaskClass.ONLINE, M.TaskClass.OFFLINE
    ctl = M.BatchController(unit(M), budget(M, 10_000))
    bs = M.BucketSet(2048, buckets=[M.Bucket(0, 1024), M.Bucket(1024, 2048)])
    bs.assign(req(M, 0, 1500, 1.0, on))
    bs.assign(req(M, 1, 100, 2.0, on))
    assert ctl.select_bucket(bs, on) == 1
    bs = M.BucketSet(2048)
    bs.assign(req(M, 0, 100, cls=off))
    assert ctl.select_bucket(bs, on) is None
    bs = M.BucketSet(4096, buckets=[M.Bucket(0, 512), M.Bucket(512, 4096)])
    for i in range(10):
        bs.assign(req(M, i, 100, cls=off))
    bs.assign(req(M, 10, 1000, cls=off))
    bs.assign(req(M, 11, 1000, cls=off))
    assert ctl.select_bucket(bs, off) == 1


def test_form_batch_cases(M):
    """test_batch_controller.py:81-131"""
    P, A = M.DispatchPolicy, M.MemoryAccounting
    b = offline_queue(M, [100, 200, 300, 400])
    plan = M.BatchController(unit(M), budget(M, 600), A.EXACT).form_batch(b, P.SJF)
    assert plan.request_ids == (0, 1, 2) and plan.token_sum == 600
    assert [r.input_len for r in b.requests] == [400]
    b = offline_queue(M, [10])
    assert M.BatchController(unit(M), budget(M, 600)).form_batch(
        b, P.SJF, pledged=M.safe_memory(budget(M, 600))) is None and len(b.requests) == 1
    assert M.BatchController(unit(M), budget(M, 1500)).form_batch(
        offline_queue(M, [1000, 10]), P.FCFS).request_ids == (0,)
    plan = M.BatchController(unit(M), budget(M, 2000)).form_batch(offline_queue(M, [1000, 10]), P.FCFS)
    assert plan.request_ids == (0, 1) and plan.footprint == 2000 * unit(M).kv_bytes_per_token
    ctl = M.BatchController(unit(M), budget(M, 1000), A.EXACT)
    b = offline_queue(M, [5000, 100])
    assert ctl.form_batch(b, P.FCFS).request_ids == (1,)
    assert [r.request.id for r in ctl.rejections] == [0] and len(b.requests) == 0
    on, off = M.TaskClass.ONLINE, M.TaskClass.OFFLINE
    b = M.Bucket(0, 100_000, deque([req(M, 0, 100, cls=on), req(M, 1, 100, cls=off),
                                    req(M, 2, 100, cls=on)]))
    plan = M.BatchController(unit(M), budget(M, 10_000)).form_batch(b, P.FCFS, task_class=on)
    assert plan.request_ids == (0, 2) and [r.id for r in b.requests] == [1]


def test_form_batch_vs_max_safe_batch(M):
    """test_batch_controller.py:134-150 (same seed; 300 instances)"""
    rng = np.random.default_rng(8)
    for _ in range(300):
        lengths = rng.integers(1, 2000, size=rng.integers(1, 30)).tolist()
        tok = int(rng.integers(1, 20_000))
        b = offline_queue(M, lengths)
        ctl = M.BatchController(unit(M), budget(M, tok), M.MemoryAccounting.EXACT)
        plan = ctl.form_batch(b, M.DispatchPolicy.FCFS)
        if not ctl.rejections:
            assert (0 if plan is None else len(plan)) == M.max_safe_batch(lengths, tok)
        rest = [r.id for r in b.requests]
        assert rest == sorted(rest)


def test_form_batch_footprint_within_headroom(M):
    """test_batch_controller.py:153-166 (same seed; 200 instances per accounting)"""
    rng = np.random.default_rng(15)
    for acc in M.MemoryAccounting:
        for _ in range(200):
            lengths = rng.integers(1, 3000, size=rng.integers(1, 20)).tolist()
            tok = int(rng.integers(1, 30_000))
            pledged = int(rng.integers(0, tok + 1)) * unit(M).kv_bytes_per_token
            gpu = budget(M, tok)
            plan = M.BatchController(unit(M), gpu, acc).form_batch(
                offline_queue(M, lengths), M.DispatchPolicy.SJF, pledged=pledged)
            if plan is not None:
                assert plan.footprint + pledged <= M.safe_memory(gpu)


def test_memory_change_and_n_max(M):
    """test_batch_controller.py:169-186"""
    ctl = M.BatchController(unit(M), budget(M, 1000))
    base = ctl.token_budget()
    assert base == 1000
    assert ctl.on_memory_change(ctl.base_safe // 2) == 500
    assert ctl.on_memory_change(0) == 0
    assert ctl.form_batch(offline_queue(M, [10]), M.DispatchPolicy.FCFS) is None
    assert ctl.on_memory_change(ctl.base_safe) == base
    ctl = M.BatchController(unit(M), budget(M, 1600))
    bs = M.BucketSet(100_000)
    assert ctl.current_n_max(bs) == 1
    for i in range(3):
        bs.assign(req(M, i, 100, cls=M.TaskClass.OFFLINE))
    assert ctl.current_n_max(bs) == 16
