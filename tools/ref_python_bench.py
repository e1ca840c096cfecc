"""Time the UNMODIFIED reference (bucketsim, pure Python, one thread on one pinned
core) on the window path — the composition of SURVEY §3.4 through
oracle/ref_compose.reference_window — at the C1 and C2 configurations, on whatever host
runs it (BASELINE.md §4.1 asks for the GPU box's host).  The reference comes from
/root/reference (build container) or its unmodified pip install in baseline/_ref
(__graft_entry__.build(); travels to the GPU box).  Each window's result is checked
against the oracle port (oracle/bso.c) with the parity comparison the tests use, so
the timed reference is the same computation the B200 arm performs.

    python tools/ref_python_bench.py [--sizes 1000 10000 100000 1000000] [--repeats 5]
Prints one JSON line per (config, size).  TEST / MEASUREMENT INFRASTRUCTURE ONLY."""
import argparse
import json
import os
import platform
import statistics
import sys
import time

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import cpu, ref_compose  # noqa: E402
from oracle.canon import canonical, diff  # noqa: E402
from paper_2507_17120_b200 import workloads as W  # noqa: E402


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def _check(cfg, lens, cls, ref):
    ws = cpu.WindowSpec(l_max=cfg.l_max, n_classes=cfg.n_classes, policies=cfg.policies,
                        theta=cfg.theta, adjust=cfg.adjust, kvpt=cfg.kvpt,
                        current_safe=cfg.current_safe, accounting=cfg.accounting,
                        init_edges=cfg.init_edges)
    o = cpu.window(ws, lens, cls)
    got = canonical(edges=o.edges, bucket=o.bucket, perm=o.perm, req_batch=o.req_batch,
                    req_row=o.req_row, batches=o.batches, n_max=o.summary["n_max"],
                    changes=o.changes)
    return diff(got, ref, bit_exact_waste=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", type=int, nargs="+", default=[1_000, 10_000, 100_000, 1_000_000])
    ap.add_argument("--repeats", type=int, default=5, help="runs per window below 100k requests")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--out", default=None, help="also append the lines to this file")
    ap.add_argument("--window", default=None, metavar="CONFIG:N",
                    help="time only this window (e.g. c2:1000000), one run")
    a = ap.parse_args()
    assert ref_compose.available(), ("needs the reference: /root/reference or baseline/_ref "
                                     "(run __graft_entry__.build() in the build container)")
    core = sorted(os.sched_getaffinity(0))[0]
    os.sched_setaffinity(0, {core})                 # one core, as BASELINE.md §4.1 states
    runs = [("c1", 1_000)] + [("c2", n) for n in a.sizes]
    if a.window:
        name, n = a.window.split(":")
        runs = [(name, int(n))]
        a.repeats = 1
    out = open(a.out, "a") if a.out else None
    for name, n in runs:
        cfg, lens, cls = W.make_window(name, n=n, seed=1234)
        reps = a.repeats if n < 100_000 else 1
        times, ref = [], None
        for _ in range(reps):
            t0 = time.perf_counter()
            ref = ref_compose.reference_window(
                lens, cls, l_max=cfg.l_max, n_classes=cfg.n_classes, policies=cfg.policies,
                theta=cfg.theta, adjust=cfg.adjust, init_edges=cfg.init_edges, kvpt=cfg.kvpt,
                current_safe=cfg.current_safe, accounting=cfg.accounting)
            times.append(time.perf_counter() - t0)
        dt = statistics.median(times)
        errs = None if a.no_check else _check(cfg, lens, cls, ref)
        line = {"impl": "reference (bucketsim, unmodified, pure Python, 1 thread on 1 core)",
                "config": name, "requests": n, "runs": reps, "seconds": round(dt, 4),
                "requests_per_s": round(n / dt, 1), "batches": int(len(ref["batch_meta"])),
                "oracle_parity": None if errs is None else (not errs),
                "reference_src": ref_compose.REF_SRC, "host": platform.node(),
                "nproc": os.cpu_count(), "cpu": _cpu_model(), "core": core,
                "python": platform.python_version()}
        s = json.dumps(line)
        print(s, flush=True)
        if out:
            out.write(s + "\n")
            out.flush()
        if errs:
            raise SystemExit(f"{name} {n}: reference != oracle: " + "; ".join(errs[:3]))


if __name__ == "__main__":
    main()
