"""The CPU oracle (oracle/bso.c) against the reference golden fixtures.

Each fixture was produced by the unmodified reference (bucketsim) composing
BucketSet.assign / adjust_buckets / BatchController.form_batch over a window
(oracle/ref_compose.py).  Bit-exact on every integer output; waste_ratio
bit-exact too (same float64 expression order, memory_model.py:98-100)."""

import os

import numpy as np
import pytest

from oracle import cpu
from oracle.canon import canonical, diff
from golden_util import fixture_names, load


def run_oracle(spec, lens, cls, **kw):
    ws = cpu.WindowSpec(l_max=spec["l_max"], n_classes=spec["n_classes"],
                        policies=spec["policies"], theta=spec["theta"], adjust=spec["adjust"],
                        max_passes=spec["max_passes"], kvpt=spec["kvpt"],
                        current_safe=spec["current_safe"], pledged=spec["pledged"],
                        accounting=spec["accounting"], truncate=spec["truncate"],
                        init_edges=spec["init_edges"])
    res = cpu.window(ws, lens, cls, **kw)
    return res, canonical(edges=res.edges, bucket=res.bucket, perm=res.perm,
                          req_batch=res.req_batch, req_row=res.req_row, batches=res.batches,
                          n_max=res.summary["n_max"], changes=res.changes,
                          n_passes=res.summary["n_passes"])


@pytest.mark.parametrize("name", fixture_names())
def test_oracle_matches_reference_fixture(name):
    spec, lens, cls, ref = load(name)
    res, got = run_oracle(spec, lens, cls)
    errs = diff(got, ref, bit_exact_waste=True)
    assert not errs, f"{name}: " + "; ".join(errs)
    # summary bookkeeping agrees with the canonical view
    s = res.summary
    assert s["n_batches"] == len(ref["batch_meta"])
    assert s["n_rejected"] == len(ref["rejected"])
    assert s["n_pending"] == len(ref["pending"])


def test_fixture_set_is_nontrivial():
    names = fixture_names()
    assert len(names) >= 25
    total_batches = sum(len(load(n)[3]["batch_meta"]) for n in names)
    assert total_batches > 5000


def dispatch_sequence(req_batch, req_row, emit_order):
    """Plans in dispatch order as (flat request ids, offsets) — the reference shape."""
    req_batch = np.asarray(req_batch, np.int64)
    adm = np.nonzero(req_batch >= 0)[0]
    order = adm[np.lexsort((np.asarray(req_row)[adm], req_batch[adm]))]
    starts = np.searchsorted(req_batch[order], np.arange(int(req_batch.max(initial=-1)) + 2))
    seq, off = [], [0]
    for b in np.asarray(emit_order, np.int64):
        seq.extend(order[starts[b]:starts[b + 1]].tolist())
        off.append(len(seq))
    return np.array(seq, np.int64), np.array(off, np.int64)


DISPATCH_FIXTURES = [n for n in fixture_names() if "disp_ids" in load(n)[3]]


@pytest.mark.parametrize("name", DISPATCH_FIXTURES)
def test_oracle_dispatch_matches_reference(name):
    """f3: Simulator._next_plan repeated (pd_sim.py:448-462) — the plan sequence,
    rejections and still-queued requests equal the live reference's."""
    spec, lens, cls, ref = load(name)
    res, _ = run_oracle(spec, lens, cls)
    ws = cpu.WindowSpec(l_max=spec["l_max"], n_classes=spec["n_classes"],
                        policies=spec["policies"], theta=spec["theta"], adjust=spec["adjust"],
                        max_passes=spec["max_passes"], kvpt=spec["kvpt"],
                        current_safe=spec["current_safe"], pledged=spec["pledged"],
                        accounting=spec["accounting"], truncate=spec["truncate"],
                        init_edges=spec["init_edges"])
    d = cpu.dispatch(ws, lens, res)
    seq, off = dispatch_sequence(d.req_batch, d.req_row, d.emit_order)
    assert np.array_equal(seq, ref["disp_ids"]) and np.array_equal(off, ref["disp_off"])
    assert np.array_equal(np.nonzero(d.req_batch == cpu.REQ_REJECTED)[0], ref["disp_rejected"])
    assert np.array_equal(np.nonzero(d.req_batch == cpu.REQ_PENDING)[0], ref["disp_pending"])


def test_dispatch_fixtures_cover_the_hazards():
    assert len(DISPATCH_FIXTURES) >= 28
    reordered = pending_differs = 0
    for n in DISPATCH_FIXTURES:
        ref = load(n)[3]
        reordered += not np.array_equal(ref["disp_ids"], ref["batch_ids"])
        pending_differs += len(ref["disp_pending"]) != len(ref["pending"])
    assert reordered >= 10 and pending_differs >= 3


FULLSIZE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                        "fullsize_reference.json")


@pytest.mark.parametrize("idx", [0, 1])
def test_oracle_matches_reference_at_benchmarked_size(idx):
    """The oracle pinned to the unmodified reference at the bench's own C2 window (1M
    requests, seed 1234; the reference takes ~40 s on it) and a C1 window: the sha256 of
    every canonical result array equals the reference's (oracle/gen_fullsize_hashes.py,
    run where the reference is importable)."""
    import json

    from oracle.gen_fullsize_hashes import digest, spec_of
    from paper_2507_17120_b200 import workloads as W
    w = json.load(open(FULLSIZE))["windows"][idx]
    cfg, lens, cls = W.make_window(w["config"], n=w["n"], seed=w["seed"])
    sp = spec_of(cfg)
    ws = cpu.WindowSpec(l_max=sp["l_max"], n_classes=sp["n_classes"], policies=sp["policies"],
                        theta=sp["theta"], adjust=sp["adjust"], init_edges=sp["init_edges"],
                        kvpt=sp["kvpt"], current_safe=sp["current_safe"],
                        accounting=sp["accounting"])
    res = cpu.window(ws, lens, cls)
    got = canonical(edges=res.edges, bucket=res.bucket, perm=res.perm, req_batch=res.req_batch,
                    req_row=res.req_row, batches=res.batches, n_max=res.summary["n_max"],
                    changes=res.changes)
    assert len(got["batch_meta"]) == w["batches"]
    assert digest(got) == w["sha256"]
