"""Monitor statistics against the live reference's golden vectors.

tests/golden/monitor.json.gz was written by oracle/gen_monitor_golden.py from the
UNMODIFIED reference: LengthHistogram.from_samples(lengths, bins, (0, L))
(memory_model.py:125-130, as pd_sim.py:829-831 calls it every tick) and
expected_waste (memory_model.py:160-191) on integer length sets, bin counts that do
and do not divide L, and partitions including malformed ones (the reference's
ValueError texts).  The host object API (LengthHistogram, expected_waste) is checked
bit-exact on CPU; the K8 kernel (bs_monitor: bins + expected_waste in one launch over
the per-length histogram) bit-exact on the GPU."""

import gzip
import json
import os

import numpy as np
import pytest

from golden_util import GOLDEN_DIR
from paper_2507_17120_b200.memory_model import LengthHistogram, expected_waste

with gzip.open(os.path.join(GOLDEN_DIR, "monitor.json.gz"), "rt") as fh:
    CASES = json.load(fh)
IDS = [f"L{c['L']}_b{c['bins']}_{c['dist']}_{i}" for i, c in enumerate(CASES)]


def _dense_counts(case):
    out = np.zeros(case["bins"], np.int64)
    out[case["counts_i"]] = case["counts_c"]
    return out


def _per_length(case):
    h = np.zeros(case["L"], np.int64)
    h[case["hist_x"]] = case["hist_c"]
    return h


def _parts(edges):
    return list(zip(edges[:-1], edges[1:])) if edges else []


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_host_length_histogram_and_expected_waste(case):
    samples = np.repeat(np.asarray(case["hist_x"], np.int64), case["hist_c"])
    h = LengthHistogram.from_samples(samples.tolist(), bins=case["bins"],
                                     value_range=(0, case["L"]))
    assert np.array_equal(h.counts, _dense_counts(case))
    assert float(np.sum(h.edges)) == case["edges_sum"]
    assert h.total_count == case["total"]
    # the GPU path wraps device bin counts on np.histogram's edges: same object
    g = LengthHistogram.from_bin_counts(_dense_counts(case), case["bins"], (0, case["L"]))
    assert np.array_equal(g.edges, h.edges) and np.array_equal(g.mids, h.mids)
    if "support" in case:
        assert list(h.support()) == case["support"]
    else:
        with pytest.raises(ValueError, match=case["support_error"]):
            h.support()
    for part in case["parts"]:
        ps = _parts(part["edges"])
        m = len(part["mass_in"])
        assert [h.mass_in(lo, up) for lo, up in ps[:m]] == part["mass_in"]
        assert [h.conditional_mean(lo, up) for lo, up in ps[:m]] == part["cond_mean"]
        if "error" in part:
            with pytest.raises(ValueError) as ei:
                expected_waste(h, ps)
            assert str(ei.value) == part["error"]
        else:
            assert expected_waste(h, ps) == part["expected_waste"]  # bit-exact


def test_fixtures_cover_non_dividing_bins():
    """bins that do not divide L (np.histogram's float edges, corrected on the device
    exactly as numpy corrects them) are part of the fixture set, with mass."""
    assert sum(1 for c in CASES if c["L"] % c["bins"] and c["hist_x"] and c["L"] > 1) >= 30


@pytest.mark.gpu
def test_device_monitor_matches_reference():
    torch = pytest.importorskip("torch")
    from paper_2507_17120_b200.window import WindowScheduler
    scheds = {}
    for case, cid in zip(CASES, IDS):
        L = case["L"]
        s = scheds.get(L)
        if s is None:
            s = scheds[L] = WindowScheduler(max_requests=1, max_seq_len=L, n_classes=1,
                                            policies=(0,), kv_bytes_per_token=1, current_safe=0,
                                            truncate=False, device=torch.device("cuda", 0))
        hist = _per_length(case)
        for part in case["parts"]:
            if not part["edges"] or part["edges"][0] != 0 or part["edges"][-1] != L:
                continue  # the device API takes a partition of [0, L)
            if any(a >= b for a, b in zip(part["edges"], part["edges"][1:])):
                continue
            if "error" in part:
                with pytest.raises(ValueError) as ei:
                    s.monitor_from_hist(hist, part["edges"], bins=case["bins"])
                assert str(ei.value) == part["error"], cid
                continue
            h, w = s.monitor_from_hist(hist, part["edges"], bins=case["bins"])
            assert np.array_equal(h.counts, _dense_counts(case)), cid
            assert w == part["expected_waste"], (cid, w, part["expected_waste"])
    for s in scheds.values():
        s.close()


@pytest.mark.gpu
def test_bucketset_monitor_equals_host_restatement():
    """BucketSet.length_histogram / expected_waste (the simulator's per-tick monitor
    over the incremental histogram) vs the host object API on the queued lengths."""
    pytest.importorskip("torch")
    from paper_2507_17120_b200.compat import BucketSet
    from paper_2507_17120_b200.types import Request, TaskClass
    rng = np.random.default_rng(17)
    bs = BucketSet(4096)
    for i in range(30_000):
        bs.assign(Request(i, float(i), int(min(4095, rng.lognormal(5.5, 1.1))), 1,
                          TaskClass.OFFLINE if i % 3 else TaskClass.ONLINE))
        if i % 7000 == 6999:
            bs.adjust_buckets(600)
    lens = [r.input_len for r in bs.iter_requests()]
    ref_h = LengthHistogram.from_samples(lens, bins=64, value_range=(0, 4096))
    ref_w = expected_waste(ref_h, [(b.low, b.up) for b in bs.buckets])
    assert np.array_equal(bs.length_histogram().counts, ref_h.counts)
    assert bs.expected_waste() == ref_w
