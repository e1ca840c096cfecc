"""Per-call latency of the stateful drop-in at queue sizes the
simulator reaches: adjust_buckets (one Alg. 1 pass, K1 + K2 on the GPU) and form_batch
(K4 + K5 on the GPU) on a BucketSet holding Q queued requests, against the reference's
own classes (from /root/reference, or its unmodified install in baseline/_ref, which
ships to the GPU box), so both run on the same host.

    python tools/compat_bench.py [--q 10000 100000] [--reps 20]
Prints one JSON line per queue size."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--q", type=int, nargs="+", default=[10_000, 100_000])
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
a = ap.parse_args()

if a.impl == "reference":
    from oracle.ref_compose import REF_SRC
    sys.path.insert(0, REF_SRC)
    sys.dont_write_bytecode = True
    from bucketsim.batch_controller import BatchController, DispatchPolicy, MemoryAccounting
    from bucketsim.bucket_manager import BucketSet
    from bucketsim.memory_model import GpuConfig, ModelConfig
    from bucketsim.workload import Request, TaskClass
else:
    import torch
    from paper_2507_17120_b200 import GpuConfig, ModelConfig
    from paper_2507_17120_b200.compat import BatchController, BucketSet
    from paper_2507_17120_b200.types import DispatchPolicy, MemoryAccounting, Request, TaskClass


def build(q, seed=3):
    rng = np.random.default_rng(seed)
    lens = np.clip(np.rint(rng.lognormal(5.5, 1.1, q)), 1, 4095).astype(int)
    cls = rng.random(q) < 0.5
    model = ModelConfig(32, 32, 128, 2, 4096)
    gpu = GpuConfig(180 * 2 ** 30, 14 * 2 ** 30, 0.10)
    bs = BucketSet(4096, 0.5)
    for i in range(q):
        bs.assign(Request(i, float(i), int(lens[i]), 16,
                          TaskClass.ONLINE if cls[i] else TaskClass.OFFLINE))
    return bs, BatchController(model, gpu, MemoryAccounting.PADDED)


for q in a.q:
    t_adj, t_form, t_steady, t_drain, nb, calls = [], [], [], [], 0, 0
    for rep in range(a.reps):
        bs, ctl = build(q, seed=3 + rep)
        n_max = ctl.current_n_max(bs)
        while True:  # adjust_buckets to the fixpoint (the first pass is timed)
            t0 = time.perf_counter()
            ch = bs.adjust_buckets(n_max)
            if not t_adj or len(t_adj) <= rep:
                t_adj.append(time.perf_counter() - t0)
            if not any(c.kind == "split" for c in ch):
                break
        t0 = time.perf_counter()  # steady state: a pass at the fixpoint (no change)
        bs.adjust_buckets(n_max)
        t_steady.append(time.perf_counter() - t0)
        # one form_batch on the bucket holding the most offline requests
        big = max(range(len(bs.buckets)), key=lambda k: sum(
            1 for r in bs.buckets[k].requests if r.task_class is TaskClass.OFFLINE))
        t0 = time.perf_counter()
        plan = ctl.form_batch(bs.buckets[big], DispatchPolicy.SJF, task_class=TaskClass.OFFLINE)
        t_form.append(time.perf_counter() - t0)
        nb = len(plan) if plan is not None else 0
        # the rest of that bucket's offline drain, call by call (the simulator's pattern)
        calls = 1
        t0 = time.perf_counter()
        while plan is not None:
            plan = ctl.form_batch(bs.buckets[big], DispatchPolicy.SJF, task_class=TaskClass.OFFLINE)
            calls += 1
        t_drain.append(time.perf_counter() - t0)
    print(json.dumps({"impl": a.impl, "queue": q, "buckets": len(bs.buckets),
                      "adjust_first_pass_ms_median": 1e3 * float(np.median(t_adj)),
                      "adjust_steady_ms_median": 1e3 * float(np.median(t_steady)),
                      "form_batch_ms_median": 1e3 * float(np.median(t_form)),
                      "batch_size": nb, "drain_calls": calls,
                      "drain_rest_ms_median": 1e3 * float(np.median(t_drain)),
                      "reps": a.reps, "host": os.uname().nodename, "nproc": os.cpu_count()}),
          flush=True)
