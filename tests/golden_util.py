"""Loading of the reference golden fixtures (tests/golden/*.npz, made by oracle/gen_golden.py)."""

from __future__ import annotations

import glob
import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def fixture_names():
    return sorted(os.path.splitext(os.path.basename(p))[0]
                  for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz")))


def load(name):
    z = np.load(os.path.join(GOLDEN_DIR, f"{name}.npz"))
    init = z["init_edges"]
    spec = dict(
        l_max=int(z["l_max"]), n_classes=int(z["n_classes"]),
        policies=tuple(int(v) for v in z["policies"]), theta=float(z["theta"]),
        adjust=bool(int(z["adjust"])), max_passes=int(z["max_passes"]),
        init_edges=tuple(int(v) for v in init) if len(init) else None,
        kvpt=int(z["kvpt"]), current_safe=int(z["current_safe"]), pledged=int(z["pledged"]),
        accounting=int(z["accounting"]), truncate=bool(int(z["truncate"])),
    )
    ref = {k[4:]: z[k] for k in z.files if k.startswith("ref_")}
    return spec, z["lens"], z["cls"], ref
