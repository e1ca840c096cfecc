"""The CPU oracle (oracle/bso.c) against the reference golden fixtures.

Each fixture was produced by the unmodified reference (bucketsim) composing
BucketSet.assign / adjust_buckets / BatchController.form_batch over a window
(oracle/ref_compose.py).  Bit-exact on every integer output; waste_ratio
bit-exact too (same float64 expression order, memory_model.py:98-100)."""

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
