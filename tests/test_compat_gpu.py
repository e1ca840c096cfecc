"""The reference-shaped drop-in surface (compat.py) on the GPU.

Scenarios restated from the reference's own bucket-manager / batch-controller
tests (pkg/tests/test_bucket_manager.py, test_batch_controller.py),
run against the GPU-backed BucketSet / BatchController, plus whole-window
equivalence with the live-reference golden fixtures via schedule_requests."""

from collections import deque

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from golden_util import fixture_names, load  # noqa: E402
from paper_2507_17120_b200 import GpuConfig, ModelConfig, safe_memory  # noqa: E402
from paper_2507_17120_b200.compat import (BatchController, Bucket, BucketSet,  # noqa: E402
                                          schedule_requests)
from paper_2507_17120_b200.types import (DispatchPolicy, MemoryAccounting, Request,  # noqa: E402
                                         TaskClass)

UNIT = ModelConfig(1, 1, 1, 2, 100_000)  # 4 bytes of KV per token


def _req(rid, length, arrival=0.0, cls=TaskClass.OFFLINE):
    return Request(rid, arrival, length, 10, cls)


def _gpu_budget(tokens):
    return GpuConfig(total_mem=tokens * UNIT.kv_bytes_per_token, model_mem=0, reserve_fraction=0.0)


def _bucket(low, up, lengths, cls=TaskClass.OFFLINE):
    return Bucket(low, up, deque(_req(i, s, float(i), cls) for i, s in enumerate(lengths)))


# ---- BucketSet (bucket_manager.py) -------------------------------------------------
def test_assign_half_open_and_counters():
    bs = BucketSet(4096, buckets=[Bucket(0, 256), Bucket(256, 1024), Bucket(1024, 4096)])
    assert bs.assign(_req(0, 256)) == 1
    assert bs.assign(_req(1, 255)) == 0
    assert bs.assign(_req(2, 1023)) == 1
    assert bs.last_assign_comparisons == 2
    with pytest.raises(ValueError):
        bs.assign(_req(3, 4096))


def test_adjust_split_trace_12_8():
    bs = BucketSet(2048, buckets=[_bucket(0, 2048, [500] * 12 + [1500] * 8)])
    ch = bs.adjust_buckets(16)
    assert [c.kind for c in ch] == ["split"] and ch[0].midpoint == 1024
    assert [(b.low, b.up, len(b)) for b in bs.buckets] == [(0, 1024, 12), (1024, 2048, 8)]
    assert bs.check_partition() is None


def test_adjust_merge_orders_by_arrival():
    a, b, c = _req(0, 100, 5.0), _req(1, 1500, 1.0), _req(2, 200, 3.0)
    bs = BucketSet(2048, buckets=[Bucket(0, 1024, deque([a, c])), Bucket(1024, 2048, deque([b]))])
    ch = bs.adjust_buckets(16)
    assert [x.kind for x in ch] == ["merge"]
    assert [r.id for r in bs.buckets[0].requests] == [1, 2, 0]


def test_adjust_no_split_below_threshold_and_stable_partition():
    bs = BucketSet(2048, buckets=[_bucket(0, 2048, [500] * 8 + [1500] * 12)])
    assert bs.adjust_buckets(16) == [] and not bs.dirty
    bs = BucketSet(2048, buckets=[_bucket(0, 2048, [100, 1900, 150, 1950, 120, 1980, 130, 1905, 110])])
    bs.adjust_buckets(8)
    left, right = bs.buckets
    assert [r.input_len for r in left.requests] == [100, 150, 120, 130, 110]
    assert [r.input_len for r in right.requests] == [1900, 1950, 1980, 1905]


def test_partition_invariant_random_ops():
    rng = np.random.default_rng(77)
    bs = BucketSet(4096)
    nid = 0
    for step in range(600):
        if rng.random() < 0.7:
            bs.assign(_req(nid, int(rng.integers(0, 4096)), float(step)))
            nid += 1
        else:
            bs.adjust_buckets(int(rng.integers(1, 40)))
    assert bs.check_partition() is None and bs.total_requests == nid


# ---- BatchController (batch_controller.py) ------------------------------------------
def test_form_batch_exact_prefix_and_remaining_queue():
    bucket = _bucket(0, 100_000, [100, 200, 300, 400])
    ctl = BatchController(UNIT, _gpu_budget(600), MemoryAccounting.EXACT)
    plan = ctl.form_batch(bucket, DispatchPolicy.SJF)
    assert plan.request_ids == (0, 1, 2) and plan.token_sum == 600
    assert [r.input_len for r in bucket.requests] == [400]


def test_form_batch_padded_charges_batch_max():
    ctl = BatchController(UNIT, _gpu_budget(1500))
    assert ctl.form_batch(_bucket(0, 100_000, [1000, 10]), DispatchPolicy.FCFS).request_ids == (0,)
    ctl2 = BatchController(UNIT, _gpu_budget(2000))
    plan = ctl2.form_batch(_bucket(0, 100_000, [1000, 10]), DispatchPolicy.FCFS)
    assert plan.request_ids == (0, 1) and plan.footprint == 2000 * UNIT.kv_bytes_per_token


def test_form_batch_oversize_rejected_and_zero_headroom():
    bucket = _bucket(0, 100_000, [5000, 100])
    ctl = BatchController(UNIT, _gpu_budget(1000), MemoryAccounting.EXACT)
    plan = ctl.form_batch(bucket, DispatchPolicy.FCFS)
    assert plan.request_ids == (1,) and [r.request.id for r in ctl.rejections] == [0]
    assert len(bucket.requests) == 0
    b2 = _bucket(0, 100_000, [10])
    ctl2 = BatchController(UNIT, _gpu_budget(600))
    assert ctl2.form_batch(b2, DispatchPolicy.SJF, pledged=safe_memory(_gpu_budget(600))) is None
    assert len(b2.requests) == 1


def test_form_batch_class_filter_keeps_other_class_in_place():
    reqs = deque([_req(0, 100, cls=TaskClass.ONLINE), _req(1, 100, cls=TaskClass.OFFLINE),
                  _req(2, 100, cls=TaskClass.ONLINE)])
    bucket = Bucket(0, 100_000, reqs)
    ctl = BatchController(UNIT, _gpu_budget(10_000))
    plan = ctl.form_batch(bucket, DispatchPolicy.FCFS, task_class=TaskClass.ONLINE)
    assert plan.request_ids == (0, 2) and [r.id for r in bucket.requests] == [1]


def test_form_batch_tie_break_by_arrival_not_queue_order():
    reqs = deque([_req(0, 100, arrival=2.0), _req(1, 100, arrival=1.0)])
    ctl = BatchController(UNIT, _gpu_budget(150))
    plan = ctl.form_batch(Bucket(0, 100_000, reqs), DispatchPolicy.SJF)
    assert plan.request_ids == (1,)


def test_form_batch_matches_max_safe_batch_oracle():
    from paper_2507_17120_b200 import max_safe_batch
    rng = np.random.default_rng(8)
    for _ in range(40):
        lengths = rng.integers(1, 2000, size=int(rng.integers(1, 30))).tolist()
        budget = int(rng.integers(1, 20_000))
        bucket = _bucket(0, 100_000, lengths)
        ctl = BatchController(UNIT, _gpu_budget(budget), MemoryAccounting.EXACT)
        plan = ctl.form_batch(bucket, DispatchPolicy.FCFS)
        got = 0 if plan is None else len(plan)
        if not ctl.rejections:
            assert got == max_safe_batch(lengths, budget)


# ---- whole window from reference objects --------------------------------------------
@pytest.mark.parametrize("name", [n for n in fixture_names()
                                  if not n.startswith(("four_class", "one_pass"))])
@pytest.mark.parametrize("dispatch", [False, True])
def test_schedule_requests_matches_reference_fixture(name, dispatch):
    spec, lens, cls, ref = load(name)
    if dispatch and "disp_ids" not in ref:
        pytest.skip("no reference dispatch sequence for this fixture")
    if spec["n_classes"] != 2 or spec["policies"][0] != 0:
        pytest.skip("schedule_requests drives ONLINE=EARLIEST_ARRIVAL / OFFLINE=policy")
    if spec["kvpt"] % 2:
        pytest.skip("needs an even kv_bytes_per_token")
    model = ModelConfig(spec["kvpt"] // 2, 1, 1, 1, spec["l_max"])
    gpu = GpuConfig(spec["current_safe"], 0, 0.0)
    if safe_memory(gpu) != spec["current_safe"]:
        pytest.skip("safe memory not representable exactly")
    classes = [TaskClass.ONLINE, TaskClass.OFFLINE]
    reqs = [Request(i, float(i), int(x), 1, classes[int(c)]) for i, (x, c) in enumerate(zip(lens, cls))]
    pol = {0: DispatchPolicy.FCFS, 1: DispatchPolicy.SJF, 2: DispatchPolicy.LJF}[spec["policies"][1]]
    out = schedule_requests(reqs, model, gpu, accounting=[MemoryAccounting.PADDED,
                                                          MemoryAccounting.EXACT][spec["accounting"]],
                            offline_policy=pol, split_threshold=spec["theta"],
                            buckets=spec["init_edges"], adjust=spec["adjust"] and spec["max_passes"] == 0,
                            pledged=spec["pledged"], dispatch=dispatch)
    if spec["max_passes"]:
        pytest.skip("one-pass fixtures covered by BucketSet.adjust_buckets")
    ids = [i for p in out.plans for i in p.request_ids]
    if dispatch:  # Simulator._next_plan order (pd_sim.py:448-462)
        assert ids == ref["disp_ids"].tolist()
        assert np.diff(ref["disp_off"]).tolist() == [len(p) for p in out.plans]
        assert sorted(r.id for r in out.pending) == ref["disp_pending"].tolist()
        assert sorted(r.request.id for r in out.rejections) == ref["disp_rejected"].tolist()
        return
    assert ids == ref["batch_ids"].tolist()
    assert [(p.max_input_len, p.token_sum, p.footprint) for p in out.plans] == \
        [tuple(m[2:5]) for m in ref["batch_meta"].tolist()]
    assert [r.request.id for r in out.rejections] == ref["rejected"].tolist()
    assert sorted(r.id for r in out.pending) == ref["pending"].tolist()
    assert out.n_max == int(ref["n_max"])
    assert out.bucket_set.edges() == ref["edges"].tolist()


def test_trace_file_to_gpu_window(tmp_path):
    """f4 -> hot path: a reference-format CSV trace parsed by the native loader feeds the
    window scheduler; the result equals scheduling the same requests as objects."""
    from paper_2507_17120_b200 import trace as T
    rng = np.random.default_rng(3)
    n = 5000
    rows = ["arrival_s,input_tokens,output_tokens,class"]
    arr = np.cumsum(rng.exponential(0.01, n))
    lens = np.clip(np.rint(rng.lognormal(5.5, 1.1, n)), 1, 5000).astype(int)
    cl = rng.random(n) < 0.4
    for a, x, c in zip(arr, lens, cl):
        rows.append(f"{float(a)!r},{int(x)},16,{'online' if c else 'offline'}")
    p = tmp_path / "t.csv"
    p.write_text("\n".join(rows) + "\n")
    tr = T.load_trace_path(p)
    model = ModelConfig(16, 8, 64, 2, 4096)
    gpu = GpuConfig(8 << 30, 2 << 30, 0.1)
    out = schedule_requests(tr.requests(), model, gpu)
    from paper_2507_17120_b200.window import WindowScheduler
    s = WindowScheduler(model, gpu, max_requests=n)
    wl, wc = tr.window(model.max_seq_len)
    res = s.schedule(wl, wc)
    assert [len(p_) for p_ in out.plans] == res.batches()["n"].tolist()
    assert out.bucket_set.edges() == res.edges().tolist()
    s.close()


def test_boundaries_from_hist_equals_k1_path():
    """K2 on a caller-maintained histogram (the BucketSet's incremental counts) gives
    the same edges / change log / n_max as K1 + K2 on the lengths themselves."""
    import torch

    from paper_2507_17120_b200.window import WindowScheduler
    rng = np.random.default_rng(11)
    s = WindowScheduler(max_requests=50_000, max_seq_len=4096, n_classes=1,
                        policies=(DispatchPolicy.FCFS,), kv_bytes_per_token=2,
                        current_safe=10**9, truncate=False, device=torch.device("cuda", 0))
    for trial in range(12):
        n = int(rng.integers(0, 50_000))
        lens = np.clip(np.rint(rng.lognormal(5.5, 1.2, n)), 0, 4095).astype(np.int32)
        edges = [0, 4096] if trial % 3 == 0 else sorted({0, 4096, *map(int, rng.integers(1, 4095, 5))})
        n_max = int(rng.integers(1, 3000))
        passes = [1, 0][trial % 2]
        a = s.boundaries(lens, init_edges=edges, n_max=n_max, max_passes=passes)
        b = s.boundaries_from_hist(np.bincount(lens, minlength=4096), init_edges=edges,
                                   n_max=n_max, max_passes=passes)
        assert list(a[0]) == list(b[0])
        assert [(c.kind, c.parent_low, c.parent_up, c.midpoint) for c in a[1]] == \
               [(c.kind, c.parent_low, c.parent_up, c.midpoint) for c in b[1]]
        assert a[2]["n_max"] == b[2]["n_max"] and a[2]["total_global"] == b[2]["total_global"]


def test_adjust_after_outside_deque_mutation_recounts():
    """Requests appended to a deque without assign() are still counted by the next
    adjust_buckets (the incremental histogram is revalidated and rebuilt)."""
    bs = BucketSet(2048, buckets=[_bucket(0, 2048, [500] * 8)])
    for i in range(8):
        bs.buckets[0].requests.append(_req(100 + i, 1500))  # 8 + 8: no split at n_max 16
    assert bs.adjust_buckets(16) == []
    for i in range(8):
        bs.buckets[0].requests.append(_req(200 + i, 300))   # 16 short of 24 > n_max: split
    ch = bs.adjust_buckets(16)
    assert [c.kind for c in ch] == ["split"]
    assert [(b.low, b.up, len(b)) for b in bs.buckets] == [(0, 1024, 16), (1024, 2048, 8)]


# ---- round-2 drop-in fixes -------------------------------------------------
from enum import Enum  # noqa: E402


class _RefTaskClass(Enum):  # stands in for bucketsim.workload.TaskClass (identity differs)
    ONLINE = "online"
    OFFLINE = "offline"


class _RefPolicy(Enum):
    SJF = "sjf"
    LJF = "ljf"
    EARLIEST_ARRIVAL = "earliest_arrival"
    FCFS = "fcfs"


class _RefAccounting(Enum):
    PADDED = "padded"
    EXACT = "exact"


def _ref_form_batch(reqs, policy, kvpt, safe, pledged, cls, padded):
    """batch_controller.py:141-191 restated in plain Python (the test's checker):
    returns (plan tuple | None, rejected ids, remaining requests)."""
    from paper_2507_17120_b200.compat import order_requests
    headroom = safe - pledged
    if headroom <= 0:
        return None, [], list(reqs)
    cands = [r for r in reqs if cls is None or r.task_class.value == cls.value]
    if not cands:
        return None, [], list(reqs)
    adm, rej, removed = [], [], set()
    cur_max = cur_sum = 0
    for r in order_requests(cands, policy):
        if kvpt * r.input_len > safe:
            rej.append(r.id)
            removed.add(r.id)
            continue
        nm, ns = max(cur_max, r.input_len), cur_sum + r.input_len
        fp = kvpt * nm * (len(adm) + 1) if padded else kvpt * ns
        if fp > headroom:
            break
        adm.append(r)
        removed.add(r.id)
        cur_max, cur_sum = nm, ns
    rest = [r for r in reqs if r.id not in removed]
    if not adm:
        return None, rej, rest
    fp = kvpt * cur_max * len(adm) if padded else kvpt * cur_sum
    return (tuple(r.id for r in adm), cur_max, cur_sum, fp), rej, rest


@pytest.mark.parametrize("padded", [True, False])
def test_foreign_enums_select_form_footprint(padded):
    """pd_sim passes bucketsim's own enum members: they are matched by value."""
    acc = _RefAccounting.PADDED if padded else _RefAccounting.EXACT
    ctl = BatchController(UNIT, _gpu_budget(10_000), acc)
    assert ctl._footprint(40, 3, 48) == (120 if padded else 48) * UNIT.kv_bytes_per_token
    reqs = deque([_req(0, 300, 2.0, _RefTaskClass.OFFLINE), _req(1, 100, 1.0, _RefTaskClass.ONLINE),
                  _req(2, 200, 0.5, _RefTaskClass.OFFLINE), _req(3, 50, 3.0, _RefTaskClass.ONLINE)])
    bs = BucketSet(100_000, buckets=[Bucket(0, 100_000, reqs)])
    assert ctl.select_bucket(bs, _RefTaskClass.ONLINE) == 0
    assert ctl.select_bucket(bs, _RefTaskClass.OFFLINE) == 0
    plan = ctl.form_batch(bs.buckets[0], _RefPolicy.EARLIEST_ARRIVAL, task_class=_RefTaskClass.ONLINE)
    assert plan.request_ids == (1, 3)
    plan = ctl.form_batch(bs.buckets[0], _RefPolicy.SJF, task_class=_RefTaskClass.OFFLINE)
    assert plan.request_ids == (2, 0)
    assert ctl.select_bucket(bs, _RefTaskClass.ONLINE) is None
    out = schedule_requests([_req(i, 100 + i, float(i), [_RefTaskClass.ONLINE, _RefTaskClass.OFFLINE][i % 2])
                             for i in range(50)], UNIT, _gpu_budget(100_000),
                            accounting=acc, offline_policy=_RefPolicy.LJF)
    assert sum(len(p) for p in out.plans) == 50


def test_schedule_requests_truncated_pending_is_filed_at_l_minus_1():
    """truncate=True + pledged memory leaves pending requests; an over-long one is
    filed in the returned BucketSet under L-1 (no IndexError, partition valid) and the
    caller's object keeps its length."""
    model = ModelConfig(1, 1, 1, 2, 4096)
    gpu = GpuConfig(4 * 5000, 0, 0.0)  # 5000 tokens of KV
    reqs = [_req(i, x, float(i)) for i, x in enumerate([100, 9000, 3000, 4000, 50])]
    out = schedule_requests(reqs, model, gpu, pledged=4 * 2000, truncate=True)
    assert out.bucket_set.check_partition() is None
    assert reqs[1].input_len == 9000
    pend = {r.id for r in out.pending}
    assert 1 in pend or any(1 in p.request_ids for p in out.plans)
    lens = {r.id: r.input_len for r in out.bucket_set.iter_requests()}
    if 1 in lens:
        assert lens[1] == 4095
    assert out.bucket_set.total_requests == len(out.pending)


def test_pool_does_not_grow_with_memory_state():
    from paper_2507_17120_b200 import compat
    ctl = BatchController(UNIT, _gpu_budget(50_000))
    before = None
    for k in range(20):
        ctl.on_memory_change(UNIT.kv_bytes_per_token * (10_000 + 37 * k))
        ctl.form_batch(_bucket(0, 100_000, [100, 200, 300]), DispatchPolicy.SJF, pledged=4 * k)
        if before is None:
            before = len(compat._POOL)
    assert len(compat._POOL) == before


def test_cached_drains_equal_fresh_form_batch_calls():
    """form_batch hands out a drain computed once per bucket state; interleaved classes,
    policies, pledged memory, memory changes and arrivals between calls must give
    exactly the reference's call-by-call results."""
    rng = np.random.default_rng(31)
    kvpt = UNIT.kv_bytes_per_token
    for trial in range(6):
        safe_tokens = int(rng.integers(2_000, 20_000))
        padded = bool(trial % 2)
        acc = MemoryAccounting.PADDED if padded else MemoryAccounting.EXACT
        ctl = BatchController(UNIT, _gpu_budget(safe_tokens), acc)
        reqs = [_req(i, int(rng.integers(1, safe_tokens + 3000)), float(rng.integers(0, 50)),
                     [TaskClass.ONLINE, TaskClass.OFFLINE][int(rng.integers(0, 2))])
                for i in range(int(rng.integers(50, 400)))]
        bucket = Bucket(0, 100_000, deque(reqs))
        shadow = list(reqs)
        nid = len(reqs)
        for step in range(120):
            op = rng.random()
            if op < 0.1:
                r = _req(nid, int(rng.integers(1, 3000)), float(rng.integers(0, 60)),
                         [TaskClass.ONLINE, TaskClass.OFFLINE][int(rng.integers(0, 2))])
                nid += 1
                bucket.add(r)
                shadow.append(r)
                continue
            if op < 0.13:
                ctl.on_memory_change(kvpt * int(rng.integers(1_000, 20_000)))
                continue
            cls = [None, TaskClass.ONLINE, TaskClass.OFFLINE][int(rng.integers(0, 3))]
            pol = [DispatchPolicy.SJF, DispatchPolicy.LJF, DispatchPolicy.FCFS][int(rng.integers(0, 3)) if step % 5 == 0 else 0]
            pledged = int(rng.choice([0, 0, 0, kvpt * 500]))
            want, want_rej, shadow = _ref_form_batch(shadow, pol, kvpt, ctl.current_safe, pledged,
                                                     cls, padded)
            plan = ctl.form_batch(bucket, pol, pledged=pledged, task_class=cls)
            got = None if plan is None else (plan.request_ids, plan.max_input_len,
                                             plan.token_sum, plan.footprint)
            assert got == want, (trial, step)
            assert [x.request.id for x in ctl.rejections] == want_rej, (trial, step)
            ctl.rejections.clear()
            assert [r.id for r in bucket.requests] == [r.id for r in shadow], (trial, step)
            assert len(bucket) == len(shadow)
