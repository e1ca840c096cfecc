"""Canonical (reference-shaped) view of a window result — TEST INFRASTRUCTURE.

Both the CPU oracle and the CUDA path return the same SoA layout (perm,
req_batch, req_row, batch descriptors).  canonical() turns it into the shape
oracle/ref_compose.reference_window() produces from the live reference, so
one comparison covers oracle-vs-reference and GPU-vs-oracle.
"""

from __future__ import annotations

import numpy as np

REQ_PENDING, REQ_REJECTED = -1, -2


def canonical(*, edges, bucket, perm, req_batch, req_row, batches, n_max, changes, n_passes=None):
    perm = np.asarray(perm, np.int64)
    req_batch = np.asarray(req_batch, np.int64)
    req_row = np.asarray(req_row, np.int64)
    n = len(perm)
    adm = np.nonzero(req_batch >= 0)[0]
    order = adm[np.lexsort((req_row[adm], req_batch[adm]))]
    nb = len(batches)
    counts = np.asarray(batches["n"], np.int64) if nb else np.zeros(0, np.int64)
    off = np.zeros(nb + 1, np.int64)
    np.cumsum(counts, out=off[1:])
    rej_mask = req_batch[perm] == REQ_REJECTED if n else np.zeros(0, bool)
    out = dict(
        n_max=np.int64(n_max),
        edges=np.asarray(edges, np.int64),
        changes=np.asarray(changes, np.int64).reshape(-1, 4),
        bucket=np.asarray(bucket, np.int64),
        batch_ids=order.astype(np.int64),
        batch_off=off,
        batch_meta=np.stack([np.asarray(batches[f], np.int64) for f in
                             ("segment", "n", "max_input_len", "token_sum", "footprint")],
                            axis=1) if nb else np.zeros((0, 5), np.int64),
        batch_waste=np.asarray(batches["waste"], np.float64) if nb else np.zeros(0),
        rejected=perm[rej_mask] if n else np.zeros(0, np.int64),
        pending=np.sort(np.nonzero(req_batch == REQ_PENDING)[0]).astype(np.int64),
    )
    if n_passes is not None:
        out["n_passes"] = np.int64(n_passes)
    return out


EXACT_KEYS = ("n_max", "edges", "changes", "bucket", "batch_ids", "batch_off", "batch_meta",
              "rejected", "pending")


def diff(got: dict, want: dict, waste_rtol: float = 1e-6, bit_exact_waste: bool = False):
    """List of human-readable mismatches (empty == parity)."""
    errs = []
    for k in EXACT_KEYS:
        if k not in want:
            continue
        a, b = np.asarray(got[k]), np.asarray(want[k])
        if a.shape != b.shape or not np.array_equal(a, b):
            where = ""
            if a.shape == b.shape and a.size:
                bad = np.argwhere(a != b)
                where = f" first mismatch at {bad[0].tolist()}: {a[tuple(bad[0])]} vs {b[tuple(bad[0])]}"
            errs.append(f"{k}: shape {a.shape} vs {b.shape}{where}")
    if "batch_waste" in want:
        a, b = np.asarray(got["batch_waste"]), np.asarray(want["batch_waste"])
        if a.shape != b.shape:
            errs.append(f"batch_waste shape {a.shape} vs {b.shape}")
        elif bit_exact_waste:
            if not np.array_equal(a, b, equal_nan=True):
                errs.append("batch_waste not bit-exact")
        elif a.size and not np.allclose(a, b, rtol=waste_rtol, atol=0, equal_nan=True):
            errs.append(f"batch_waste beyond rtol {waste_rtol}")
    if "n_passes" in want and "n_passes" in got and int(got["n_passes"]) != int(want["n_passes"]):
        errs.append(f"n_passes {got['n_passes']} vs {want['n_passes']}")
    return errs
