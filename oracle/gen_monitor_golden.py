"""Golden vectors for the monitor statistics from the UNMODIFIED reference.

TEST INFRASTRUCTURE.  Run in the build container (needs /root/reference):
    python -m oracle.gen_monitor_golden
Every case is a set of integer lengths in [0, L), a bin count and a bucket partition
of [0, L).  The reference's own LengthHistogram.from_samples(lengths, bins,
value_range=(0, L)) (memory_model.py:125-130, the call pd_sim.py:829-831 makes every
tick) gives the counts, support, mass_in / conditional_mean of every bucket, and
expected_waste(hist, partition) (memory_model.py:160-191) the monitor value — or the
ValueError text where the reference raises.  The fixture stores the per-length
histogram (what the GPU holds; sparse: hist_x, hist_c) rather than the samples.

Cases: the reference's own test shapes (test_memory_model.py:95-138), the simulator's
64 bins at L = 4096 / 131072 / 100 / 2048 / 3000, bin counts that do not divide L
(7, 100, 1000, 4095 — np.histogram's float edge correction), empty and single-length
queues, fine and coarse partitions."""

from __future__ import annotations

import gzip
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden", "monitor.json.gz")
REF_SRC = os.environ.get("BUCKETSIM_REF_SRC", "/root/reference/pkg/src")


def _partition(rng, L, kind):
    if kind == "one":
        return [0, L]
    if kind == "halves":
        return sorted({0, L // 2, L}) if L > 1 else [0, L]
    k = int(rng.integers(1, min(L, 600) + 1))
    inner = rng.choice(np.arange(1, L), size=min(k, L - 1), replace=False) if L > 1 else []
    return [0] + sorted(int(x) for x in inner) + [L]


def main():
    if not os.path.isdir(os.path.join(REF_SRC, "bucketsim")):
        raise SystemExit("reference not available")
    sys.path.insert(0, REF_SRC)
    sys.dont_write_bytecode = True
    from bucketsim.memory_model import LengthHistogram, expected_waste

    rng = np.random.default_rng(2507)
    specs = []
    for L in (4096, 131072, 100, 2048, 3000, 7, 1):
        for bins in (64, 7, 100, 1000, 4095, 1):
            for dist in ("lognormal", "uniform", "single", "empty", "tail"):
                specs.append((L, bins, dist))
    cases = []
    for k, (L, bins, dist) in enumerate(specs):
        n = int(rng.integers(1, 8_000))
        if dist == "lognormal":
            lens = np.clip(np.rint(rng.lognormal(np.log(max(L, 2)) - 2.5, 1.1, n)), 0, L - 1)
        elif dist == "uniform":
            lens = rng.integers(0, L, n)
        elif dist == "single":
            lens = np.full(n, int(rng.integers(0, L)))
        elif dist == "tail":
            lens = np.concatenate([rng.integers(0, max(1, L // 50), n), rng.integers(L - max(1, L // 20), L, 40)])
        else:
            lens = np.zeros(0, np.int64)
        lens = lens.astype(np.int64)
        hx, hc = np.unique(lens, return_counts=True)
        hist = LengthHistogram.from_samples([int(x) for x in lens], bins=bins, value_range=(0, L))
        nz = np.nonzero(hist.counts)[0]
        case = {"L": L, "bins": bins, "dist": dist, "hist_x": hx.tolist(), "hist_c": hc.tolist(),
                "counts_i": nz.tolist(), "counts_c": [int(c) for c in hist.counts[nz]],
                "edges_sum": float(np.sum(hist.edges)), "total": hist.total_count, "parts": []}
        try:
            case["support"] = list(hist.support())
        except ValueError as e:
            case["support_error"] = str(e)
        for pk in ("one", "halves", "random"):
            edges = _partition(rng, L, pk)
            parts = list(zip(edges[:-1], edges[1:]))
            part = {"edges": edges,
                    "mass_in": [hist.mass_in(lo, up) for lo, up in parts[:50]],
                    "cond_mean": [hist.conditional_mean(lo, up) for lo, up in parts[:50]]}
            try:
                part["expected_waste"] = expected_waste(hist, parts)
            except ValueError as e:
                part["error"] = str(e)
            case["parts"].append(part)
        cases.append(case)
    # partitions that do not cover the support / are malformed (reference errors)
    hist_lens = rng.integers(10, 90, 500)
    hist = LengthHistogram.from_samples([int(x) for x in hist_lens], bins=64, value_range=(0, 100))
    nz = np.nonzero(hist.counts)[0]
    hx, hc = np.unique(hist_lens, return_counts=True)
    case = {"L": 100, "bins": 64, "dist": "bad_partition", "hist_x": hx.tolist(),
            "hist_c": hc.tolist(), "counts_i": nz.tolist(),
            "counts_c": [int(c) for c in hist.counts[nz]], "edges_sum": float(np.sum(hist.edges)),
            "total": hist.total_count, "support": list(hist.support()), "parts": []}
    for edges in ([0, 50], [20, 100], [0, 50, 50, 100], [0, 60, 40, 100], []):
        parts = list(zip(edges[:-1], edges[1:])) if edges else []
        part = {"edges": edges, "mass_in": [], "cond_mean": []}
        try:
            part["expected_waste"] = expected_waste(hist, parts)
        except ValueError as e:
            part["error"] = str(e)
        case["parts"].append(part)
    cases.append(case)
    with gzip.open(OUT, "wt") as fh:
        json.dump(cases, fh)
    print(f"{len(cases)} cases -> {OUT}")


if __name__ == "__main__":
    main()
