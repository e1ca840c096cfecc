"""Trace ingestion throughput: native bs_trace_parse vs the reference's load_trace.

    python tools/trace_bench.py [--n 4000000] [--ref-n 200000]
Generates a C2-shaped CSV / JSONL trace in memory (lognormal lengths, Poisson
arrivals), parses it with the native parser (all host threads) and, when the
reference is importable (build container only), a sample with bucketsim's own
load_trace.  Prints one JSON line."""
import argparse
import io
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_17120_b200 import trace as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4_000_000)
ap.add_argument("--ref-n", type=int, default=200_000)
a = ap.parse_args()
rng = np.random.default_rng(5)


def make(n):
    arr = np.cumsum(rng.exponential(1e-3, n))
    tr = T.TraceArrays(id=np.arange(n), arrival=arr,
                       input_len=np.clip(np.rint(rng.lognormal(5.5, 1.1, n)), 1, 4095).astype(np.int64),
                       output_len=np.clip(np.rint(rng.normal(128, 40, n)), 1, 512).astype(np.int64),
                       cls=(rng.random(n) < 0.5).astype(np.uint8))
    out = {}
    for fmt in ("csv", "jsonl"):
        buf = io.StringIO()
        T.save_trace(tr, buf, fmt)
        out[fmt] = buf.getvalue().encode()
    return out


res = {"n": a.n, "threads": os.cpu_count()}
texts = make(a.n)
for fmt, data in texts.items():
    T.parse_trace(data[: 1 << 16].rsplit(b"\n", 1)[0], fmt)
    t0 = time.perf_counter()
    tr = T.parse_trace(data, fmt)
    dt = time.perf_counter() - t0
    assert len(tr) == a.n
    res[f"native_{fmt}_Mrec_s"] = a.n / dt / 1e6
    res[f"native_{fmt}_MB_s"] = len(data) / dt / 1e6
ref = "/root/reference/pkg/src"
if os.path.isdir(ref):
    sys.path.insert(0, ref)
    sys.dont_write_bytecode = True
    from bucketsim import workload as wl
    small = make(a.ref_n)
    for fmt, data in small.items():
        t0 = time.perf_counter()
        wl.load_trace(io.StringIO(data.decode()), wl.TraceFormat(fmt))
        dt = time.perf_counter() - t0
        res[f"reference_{fmt}_Mrec_s"] = a.ref_n / dt / 1e6
print(json.dumps(res))
