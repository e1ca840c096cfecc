"""Time the UNMODIFIED reference (bucketsim, pure Python, one thread) on the window
path — the composition of SURVEY §3.4 through oracle/ref_compose.reference_window —
at growing window sizes of the C1 / C2 configurations.  Needs /root/reference (build
container only); the numbers are a labelled CPU reference point beside the oracle-port
arm that bench.py times on the GPU box.

    python tools/ref_python_bench.py [--sizes 1000 10000 100000 1000000]
Prints one JSON line per (config, size)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ref_compose  # noqa: E402
from paper_2507_17120_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", type=int, nargs="+", default=[1_000, 10_000, 100_000, 1_000_000])
a = ap.parse_args()
assert ref_compose.available(), "needs the reference under /root/reference"

runs = [("c1", 1_000)] + [("c2", n) for n in a.sizes]
for name, n in runs:
    cfg, lens, cls = W.make_window(name, n=n, seed=1234)
    t0 = time.perf_counter()
    r = ref_compose.reference_window(lens, cls, l_max=cfg.l_max, n_classes=cfg.n_classes,
                                     policies=cfg.policies, theta=cfg.theta, adjust=cfg.adjust,
                                     init_edges=cfg.init_edges, kvpt=cfg.kvpt,
                                     current_safe=cfg.current_safe, accounting=cfg.accounting)
    dt = time.perf_counter() - t0
    print(json.dumps({"impl": "reference (bucketsim, pure Python, 1 thread)", "config": name,
                      "requests": n, "seconds": round(dt, 3), "requests_per_s": round(n / dt, 1),
                      "batches": int(len(r["batch_meta"])),
                      "host": os.uname().nodename, "cpus": os.cpu_count()}), flush=True)
