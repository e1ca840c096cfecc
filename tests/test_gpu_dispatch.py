"""K7 dispatch order on the GPU vs the live reference and the oracle.

The reference fixtures hold the plan sequence of Simulator._next_plan repeated
(pd_sim.py:448-462) with the reference's own select_bucket / form_batch
(oracle/ref_compose._dispatch_loop).  The GPU sequence, rejections and still-queued
requests must be identical; four-class windows (no reference rule for classes >= 2)
are checked against the C restatement (oracle/bso.c: bso_dispatch)."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import cpu  # noqa: E402
from golden_util import fixture_names, load  # noqa: E402
from test_oracle_golden import dispatch_sequence  # noqa: E402
from paper_2507_17120_b200 import workloads as W  # noqa: E402
from paper_2507_17120_b200.window import WindowScheduler  # noqa: E402


def _sched(spec, n, **kw):
    return WindowScheduler(max_requests=max(n, 1), max_seq_len=spec["l_max"],
                           n_classes=spec["n_classes"], policies=spec["policies"],
                           split_threshold=spec["theta"], adjust=spec["adjust"],
                           max_passes=spec["max_passes"], buckets=spec["init_edges"],
                           kv_bytes_per_token=spec["kvpt"], current_safe=spec["current_safe"],
                           pledged=spec["pledged"], accounting=spec["accounting"],
                           truncate=spec["truncate"], dispatch=True, **kw)


def _ws(spec):
    return cpu.WindowSpec(l_max=spec["l_max"], n_classes=spec["n_classes"],
                          policies=spec["policies"], theta=spec["theta"], adjust=spec["adjust"],
                          max_passes=spec["max_passes"], kvpt=spec["kvpt"],
                          current_safe=spec["current_safe"], pledged=spec["pledged"],
                          accounting=spec["accounting"], truncate=spec["truncate"],
                          init_edges=spec["init_edges"])


def _check_vs_oracle(spec, lens, cls, h):
    o = cpu.window(_ws(spec), lens, cls)
    d = cpu.dispatch(_ws(spec), lens, o)
    assert np.array_equal(h["emit_order"], d.emit_order)
    assert np.array_equal(h["batch_emit"], d.batch_emit)
    assert np.array_equal(h["req_batch"], d.req_batch)
    assert np.array_equal(h["req_row"], d.req_row)
    s = h["summary"]
    assert s["n_dispatched"] == d.n_emitted
    assert s["n_rejected"] == d.n_rejected and s["n_pending"] == d.n_pending


DISPATCH_FIXTURES = [n for n in fixture_names() if "disp_ids" in load(n)[3]]


@pytest.mark.parametrize("name", DISPATCH_FIXTURES)
def test_gpu_dispatch_matches_reference(name):
    spec, lens, cls, ref = load(name)
    sched = _sched(spec, len(lens))
    h = sched.schedule(lens, cls).to_host()
    seq, off = dispatch_sequence(h["req_batch"], h["req_row"], h["emit_order"])
    assert np.array_equal(seq, ref["disp_ids"]), name
    assert np.array_equal(off, ref["disp_off"]), name
    assert np.array_equal(np.nonzero(h["req_batch"] == -2)[0], ref["disp_rejected"])
    assert np.array_equal(np.nonzero(h["req_batch"] == -1)[0], ref["disp_pending"])
    _check_vs_oracle(spec, lens, cls, h)
    sched.close()


def test_gpu_dispatch_four_classes_vs_oracle():
    spec, lens, cls, _ = load("four_class_exact")
    sched = _sched(spec, len(lens))
    _check_vs_oracle(spec, lens, cls, sched.schedule(lens, cls).to_host())
    sched.close()


@pytest.mark.parametrize("seed", range(int(os.environ.get("BS_RANDOM_CONFIGS", "10"))))
def test_gpu_dispatch_random_vs_oracle(seed):
    rng = np.random.default_rng(700 + seed)
    C = int(rng.integers(1, 5))
    L = int(rng.choice([16, 100, 1000, 4096]))
    n = int(rng.integers(1, 30000))
    lens = np.minimum(rng.geometric(4.0 / L, size=n) - (seed % 3 == 0), L - 1).astype(np.int32)
    cls = rng.integers(0, C, size=n).astype(np.uint8)
    kvpt = int(rng.choice([2, 6]))
    safe = kvpt * int(rng.integers(L // 2 + 1, 6 * L))
    pledged = int(rng.choice([0, 0, kvpt * int(rng.integers(1, L // 2 + 2))]))
    spec = dict(l_max=L, n_classes=C, policies=tuple(int(x) for x in rng.integers(0, 3, size=C)),
                theta=float(rng.choice([0.3, 0.5, 1.0])), adjust=bool(rng.integers(0, 2)),
                max_passes=0, init_edges=None, kvpt=kvpt, current_safe=safe, pledged=pledged,
                accounting=int(rng.integers(0, 2)), truncate=True)
    sched = _sched(spec, n)
    _check_vs_oracle(spec, lens, cls, sched.schedule(lens, cls).to_host())
    sched.close()


def test_gpu_dispatch_c2_full_size():
    """C2 at its full 1M size: the dispatch order equals the oracle's, and every batch
    is dispatched exactly once."""
    cfg, lens, cls = W.make_window("c2")
    spec = dict(l_max=cfg.l_max, n_classes=cfg.n_classes, policies=cfg.policies,
                theta=cfg.theta, adjust=cfg.adjust, max_passes=0, init_edges=cfg.init_edges,
                kvpt=cfg.kvpt, current_safe=cfg.current_safe, pledged=0,
                accounting=cfg.accounting, truncate=True)
    sched = _sched(spec, len(lens))
    h = sched.schedule(lens, cls).to_host()
    nb = len(h["batches"])
    assert np.array_equal(np.sort(h["emit_order"]), np.arange(nb))
    _check_vs_oracle(spec, lens, cls, h)
    # online plans come first (ONLINE is tried first in every _next_plan call)
    seg = h["batches"]["segment"][h["emit_order"]]
    first_offline = np.argmax(seg % 2 == 1)
    assert (seg[:first_offline] % 2 == 0).all() and (seg[first_offline:] % 2 == 1).all()
    sched.close()


def test_gpu_dispatch_graph_replay_and_reuse():
    """The dispatch stage replays inside the window's CUDA graph; windows of different
    shapes through one scheduler give the same answers as fresh ones."""
    dev = torch.device("cuda", 0)
    spec, lens, cls, _ = load("c2_n30000")
    sched = _sched(spec, 40000)
    L = torch.as_tensor(lens).to(dev)
    Cl = torch.as_tensor(cls).to(dev)
    want = sched.schedule(L, Cl).to_host()
    for _ in range(3):
        got = sched.schedule(L, Cl, graph=True).to_host()
        assert np.array_equal(got["emit_order"], want["emit_order"])
    spec2, lens2, cls2, ref2 = load("dispatch_online_rejects")
    sched2 = _sched(spec2, 40000)
    h2 = sched2.schedule(lens2, cls2).to_host()
    seq, off = dispatch_sequence(h2["req_batch"], h2["req_row"], h2["emit_order"])
    assert np.array_equal(seq, ref2["disp_ids"])
    sched.close()
    sched2.close()


@pytest.mark.parametrize("classes,pledged", [(2, 0), (3, 0), (2, 1)])
def test_gpu_dispatch_multi_cta_path(classes, pledged):
    """More than 8,192 form_batch calls: the cooperative multi-CTA path (chunked key
    scan, onesweep radix passes, grid barriers) against the oracle."""
    rng = np.random.default_rng(40 + classes + pledged)
    n = 120_000
    lens = np.clip(np.rint(rng.lognormal(4.0, 1.0, n)), 1, 1023).astype(np.int32)
    cls = rng.integers(0, classes, size=n).astype(np.uint8)
    kvpt = 2
    spec = dict(l_max=1024, n_classes=classes, policies=(0,) + (1,) * (classes - 1),
                theta=0.5, adjust=True, max_passes=0, init_edges=None, kvpt=kvpt,
                current_safe=kvpt * 1200, pledged=kvpt * 200 * pledged, accounting=0,
                truncate=True)
    sched = _sched(spec, n)
    h = sched.schedule(lens, cls).to_host()
    assert len(h["batches"]) > 8192
    _check_vs_oracle(spec, lens, cls, h)
    sched.close()


def test_gpu_dispatch_long_context_c4():
    """C4 shape (l_max 131,072: bucket ids need the full 17 key bits) vs the oracle."""
    cfg, lens, cls = W.make_window("c4", n=20_000, seed=3)
    spec = dict(l_max=cfg.l_max, n_classes=cfg.n_classes, policies=cfg.policies,
                theta=cfg.theta, adjust=cfg.adjust, max_passes=0, init_edges=cfg.init_edges,
                kvpt=cfg.kvpt, current_safe=cfg.current_safe, pledged=0,
                accounting=cfg.accounting, truncate=True)
    sched = _sched(spec, len(lens))
    _check_vs_oracle(spec, lens, cls, sched.schedule(lens, cls).to_host())
    sched.close()


@pytest.mark.parametrize("seed", [275, 1614])
def test_gpu_dispatch_blocked_bucket_reenters(seed):
    """Regression (found by a 2,000-configuration soak): a blocked null call first
    rejects the oversize requests before the blocking one, so its bucket re-enters
    select_bucket with a smaller key and the class may go on with other buckets —
    3-4 classes, pledged memory blocking several buckets."""
    test_gpu_dispatch_random_vs_oracle(seed)


def test_gpu_dispatch_large_blocked_buckets():
    """Pledged memory blocks two buckets of 20k requests each (length 3000 > headroom
    of 2500 tokens, admissible against current_safe): the key each re-enters
    select_bucket with is reduced over its 20k remaining requests by one warp per null
    call (it was a single-thread loop on the walk's critical path) — the
    dispatch order equals the oracle's."""
    rng = np.random.default_rng(77)
    n = 400_000
    lens = rng.choice(np.array([100, 200, 3000], np.int32), size=n, p=[0.45, 0.45, 0.10])
    cls = rng.integers(0, 2, size=n).astype(np.uint8)
    kvpt = 2
    spec = dict(l_max=4096, n_classes=2, policies=(0, 1), theta=0.5, adjust=True,
                max_passes=0, init_edges=None, kvpt=kvpt, current_safe=kvpt * 4000,
                pledged=kvpt * 1500, accounting=0, truncate=True)
    sched = _sched(spec, n)
    h = sched.schedule(lens, cls).to_host()
    assert (h["req_batch"] == -1).sum() > 30_000  # the blocked buckets stay pending
    _check_vs_oracle(spec, lens, cls, h)
    sched.close()
