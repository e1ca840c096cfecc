"""Pin the oracle to the UNMODIFIED reference at a benchmarked size: run the reference's
window composition (oracle/ref_compose.py) on the bench's own C2 window
(1M requests, seed 1234) and on a C1 window, and store the sha256 of every canonical
result array (oracle/canon.py shape) in tests/golden/fullsize_reference.json.

TEST INFRASTRUCTURE.  Run where the reference is importable (/root/reference or its
baseline/_ref install):
    python -m oracle.gen_fullsize_hashes        (~30 s for the 1M window)
tests/test_oracle_golden.py checks the oracle against these hashes on every CPU run,
tests/test_gpu_parity.py the CUDA path."""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle.canon import EXACT_KEYS  # noqa: E402
from oracle.ref_compose import available, reference_window  # noqa: E402
from paper_2507_17120_b200 import workloads as W  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "fullsize_reference.json")
WINDOWS = (("c2", 1_000_000, 1234), ("c1", 1000, 1234))


def digest(res: dict) -> dict:
    """sha256 per canonical key: integer arrays as little-endian int64, waste_ratio as
    the float64 bit patterns (bit-exact)."""
    out = {}
    for k in EXACT_KEYS:
        a = np.ascontiguousarray(np.asarray(res[k]).astype("<i8"))
        out[k] = hashlib.sha256(a.tobytes()).hexdigest()
    w = np.ascontiguousarray(np.asarray(res["batch_waste"], "<f8"))
    out["batch_waste"] = hashlib.sha256(w.tobytes()).hexdigest()
    return out


def spec_of(cfg):
    return dict(l_max=cfg.l_max, n_classes=cfg.n_classes, policies=cfg.policies,
                theta=cfg.theta, adjust=cfg.adjust, init_edges=cfg.init_edges,
                kvpt=cfg.kvpt, current_safe=cfg.current_safe, accounting=cfg.accounting)


def main():
    if not available():
        raise SystemExit("reference not available")
    doc = {"what": "sha256 of the reference's canonical window result (oracle/canon.py keys) "
                   "on workloads.make_window(config, n, seed)", "windows": []}
    for name, n, seed in WINDOWS:
        cfg, lens, cls = W.make_window(name, n=n, seed=seed)
        t0 = time.perf_counter()
        ref = reference_window(lens, cls, **spec_of(cfg))
        dt = time.perf_counter() - t0
        doc["windows"].append({"config": name, "n": n, "seed": seed,
                               "batches": int(len(ref["batch_meta"])),
                               "reference_seconds": round(dt, 1), "sha256": digest(ref)})
        print(name, n, len(ref["batch_meta"]), f"{dt:.1f} s")
    with open(OUT, "w") as f:
        json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
