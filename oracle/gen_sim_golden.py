"""Call logs of the reference simulator's scheduling path.

TEST INFRASTRUCTURE.  Run in the build container (needs /root/reference):
    python -m oracle.gen_sim_golden
Runs the UNMODIFIED reference Simulator (pd_sim.py) on mixed workloads with logging
subclasses of its BucketSet / BatchController injected into pd_sim's namespace, and
records every call the simulator makes on the scheduling path, in order, with its
inputs and results:

  assign(request)                  -> bucket index        (pd_sim.py:406)
  current_n_max(bucket_set)        -> n_max               (pd_sim.py:435)
  adjust_buckets(n_max)            -> changes, edges      (pd_sim.py:438)
  select_bucket(bucket_set, cls)   -> index | None        (pd_sim.py:451)
  form_batch(bucket[idx], policy, pledged, task_class)
                                   -> plan | None, rejections (pd_sim.py:454-467)
  snapshot (monitor, every tick)   -> bucket partition, expected_waste of the 64-bin
                                      LengthHistogram of the queue (pd_sim.py:828-833)

Workloads: four synthetic mixes (BucketServe SJF / LJF+EXACT / tight memory, the
continuous no-bucket proxy) and the reference's own scenario files run exactly as
`bucketsim run` runs them (pkg/scenarios/smoke.yaml, mixed_longtail.yaml through
config.load_scenario -> Scenario.simulator, cli.py:37-48); for those the sha256 of the
JSON report `bucketsim run --format json` prints is stored too.  Since the simulator
touches the scheduling path only through these calls, a drop-in that reproduces every
logged result reproduces the run (and its report) byte for byte.

tests/test_compat_sim_replay.py replays each log against the GPU-backed drop-in
(paper_2507_17120_b200.compat) and requires identical results at every call — the
stateful drop-in exercised with the simulator's real call pattern (per-arrival
assign, one adjust pass per tick on the current edges, per-dispatch select + form).
"""

from __future__ import annotations

import gzip
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden", "sim_calls.json.gz")
REF_SRC = os.environ.get("BUCKETSIM_REF_SRC", "/root/reference/pkg/src")


def main():
    if not os.path.isdir(os.path.join(REF_SRC, "bucketsim")):
        raise SystemExit("reference not available")
    sys.path.insert(0, REF_SRC)
    sys.dont_write_bytecode = True
    from bucketsim import pd_sim
    from bucketsim import bucket_manager as bm
    from bucketsim import batch_controller as bc
    from bucketsim import workload as wl
    from bucketsim.baselines import BucketServePolicy, ContinuousNoBucketPolicy
    from bucketsim.config import load_scenario
    from bucketsim.memory_model import MODEL_PRESETS, GpuConfig
    from bucketsim.metrics import emit_report
    import hashlib

    log: list = []

    def req_rec(r):
        return [r.id, r.arrival_time, r.input_len, r.task_class.value]

    class LogBucketSet(bm.BucketSet):
        def assign(self, request):
            idx = super().assign(request)
            log.append({"op": "assign", "req": req_rec(request), "out": idx})
            return idx

        def adjust_buckets(self, n_max):
            ch = super().adjust_buckets(n_max)
            log.append({"op": "adjust", "n_max": n_max,
                        "out": [[c.kind, c.parent_low, c.parent_up, c.midpoint] for c in ch],
                        "edges": [b.low for b in self.buckets] + [self.buckets[-1].up],
                        "dirty": self.dirty})
            return ch

    class LogController(bc.BatchController):
        def current_n_max(self, bucket_set):
            v = super().current_n_max(bucket_set)
            log.append({"op": "n_max", "out": v})
            return v

        def select_bucket(self, bucket_set, task_class):
            v = super().select_bucket(bucket_set, task_class)
            log.append({"op": "select", "cls": task_class.value, "out": v})
            return v

        def form_batch(self, bucket, policy, *, pledged=0, task_class=None, now=0.0):
            before = len(self.rejections)
            idx = next(i for i, b in enumerate(self._bs.buckets) if b is bucket)
            plan = super().form_batch(bucket, policy, pledged=pledged, task_class=task_class,
                                      now=now)
            rej = [r.request.id for r in self.rejections[before:]]
            log.append({"op": "form", "bucket": idx, "policy": policy.value, "pledged": pledged,
                        "cls": None if task_class is None else task_class.value,
                        "out": None if plan is None else
                        [list(plan.request_ids), plan.max_input_len, plan.token_sum,
                         plan.footprint],
                        "rejected": rej})
            return plan

    orig_ew = pd_sim.expected_waste

    def log_expected_waste(hist, partition):
        v = orig_ew(hist, partition)
        log.append({"op": "snapshot", "edges": [lo for lo, _ in partition] + [partition[-1][1]],
                    "total": hist.total_count, "out": v})
        return v

    orig_bs, orig_bc = pd_sim.BucketSet, pd_sim.BatchController
    pd_sim.BucketSet = LogBucketSet
    pd_sim.BatchController = LogController
    pd_sim.expected_waste = log_expected_waste
    cases = []
    gib = 2 ** 30
    scenarios = [
        ("bucketserve_sjf", BucketServePolicy(), bc.DispatchPolicy.SJF, bc.MemoryAccounting.PADDED,
         MODEL_PRESETS["llama2-13b-like"], GpuConfig(40 * gib, 26 * gib, 0.10), 0.5, 800, 400.0),
        ("bucketserve_ljf_exact", BucketServePolicy(), bc.DispatchPolicy.LJF,
         bc.MemoryAccounting.EXACT, MODEL_PRESETS["llama2-13b-like"],
         GpuConfig(40 * gib, 26 * gib, 0.10), 0.4, 600, 700.0),
        ("bucketserve_tight_mem", BucketServePolicy(), bc.DispatchPolicy.FCFS,
         bc.MemoryAccounting.PADDED, MODEL_PRESETS["llama2-13b-like"],
         GpuConfig(29 * gib, 26 * gib, 0.10), 0.5, 500, 300.0),
        ("continuous_nobucket", ContinuousNoBucketPolicy(), bc.DispatchPolicy.SJF,
         bc.MemoryAccounting.PADDED, MODEL_PRESETS["llama2-13b-like"],
         GpuConfig(40 * gib, 26 * gib, 0.10), 0.5, 500, 500.0),
    ]
    try:
        for k, (name, policy, off, acc, model, gpu, theta, nreq, rate) in enumerate(scenarios):
            log.clear()
            spec = wl.WorkloadSpec(
                arrival=wl.PoissonArrivals(rate),
                length_dist=wl.Mixture((wl.ShortNormal(83, 40, cap=4095),
                                        wl.LongTailLogNormal(7.0, 0.8, cap=4095)), (0.7, 0.3)),
                output_dist=wl.ShortNormal(64, 20), horizon=wl.Horizon(requests=nreq),
                online_fraction=0.5, seed=100 + k)
            trace = wl.gen_synthetic(spec)
            # one prefill worker and a slow prefill so queues build up and buckets split /
            # merge (the simcases STANDARD_COST figures)
            cluster = pd_sim.ClusterConfig(prefill_workers=1, decode_workers=2, gpu=gpu)
            cost = pd_sim.CostModel(prefill_base=0.004, prefill_per_token=2e-5,
                                    decode_step_base=0.002, decode_per_kv_byte=1e-12,
                                    transfer_bandwidth=300e9, transfer_latency=2e-4)
            sim = pd_sim.Simulator(trace, model=model, cluster=cluster, cost=cost,
                                   policy=policy, offline_policy=off, accounting=acc,
                                   split_threshold=theta)
            sim.controller._bs = sim.bucket_set
            sim.run()
            cases.append({
                "name": name,
                "max_seq_len": model.max_seq_len,
                "split_threshold": sim.bucket_set.split_threshold,
                "model": [model.layers, model.heads, model.head_dim, model.bytes_per_elem,
                          model.max_seq_len],
                "gpu": [gpu.total_mem, gpu.model_mem, gpu.reserve_fraction],
                "accounting": acc.value,
                "calls": list(log),
            })
            ops = {}
            for e in log:
                ops[e["op"]] = ops.get(e["op"], 0) + 1
            print(f"{name:24s} calls={len(log):6d} {ops}")
        scen_dir = os.path.join(os.path.dirname(REF_SRC), "scenarios")
        for fname in ("smoke.yaml", "mixed_longtail.yaml"):
            log.clear()
            sc = load_scenario(os.path.join(scen_dir, fname))
            sim = sc.simulator()
            sim.controller._bs = sim.bucket_set
            report = sim.run()
            m = sc.model
            cases.append({
                "name": "scenario_" + fname.split(".")[0],
                "max_seq_len": m.max_seq_len,
                "split_threshold": sim.bucket_set.split_threshold,
                "model": [m.layers, m.heads, m.head_dim, m.bytes_per_elem, m.max_seq_len],
                "gpu": [sc.cluster.gpu.total_mem, sc.cluster.gpu.model_mem,
                        sc.cluster.gpu.reserve_fraction],
                "accounting": sc.accounting.value,
                "report_sha256": hashlib.sha256(emit_report(report, "json").encode()).hexdigest(),
                "calls": list(log),
            })
            ops = {}
            for e in log:
                ops[e["op"]] = ops.get(e["op"], 0) + 1
            print(f"{cases[-1]['name']:24s} calls={len(log):6d} {ops}")
        # acceptance criterion 7 (test_acceptance.py:264-282): theta = 1.0 + FCFS +
        # EXACT BucketServe vs the continuous no-bucket proxy on 20 seeded traces of the
        # standard scenario; the reference's batch schedules are identical per seed
        from dataclasses import replace as _replace
        base = load_scenario(os.path.join(scen_dir, "mixed_longtail.yaml"))
        for seed in range(20):
            spec = _replace(base.workload.spec, horizon=wl.Horizon(requests=100),
                            arrival=wl.PoissonArrivals(30.0), seed=seed)
            trace = wl.gen_synthetic(spec)
            for kind in ("bucket", "continuous"):
                log.clear()
                if kind == "bucket":
                    sim = pd_sim.Simulator(
                        trace, model=base.model, cluster=base.cluster, cost=base.cost,
                        policy=BucketServePolicy(), offline_policy=bc.DispatchPolicy.FCFS,
                        accounting=bc.MemoryAccounting.EXACT, split_threshold=1.0,
                        tick_interval=base.tick_interval)
                else:
                    sim = pd_sim.Simulator(
                        trace, model=base.model, cluster=base.cluster, cost=base.cost,
                        policy=ContinuousNoBucketPolicy(), accounting=bc.MemoryAccounting.EXACT,
                        tick_interval=base.tick_interval)
                sim.controller._bs = sim.bucket_set
                sim.run()
                m = base.model
                cases.append({
                    "name": f"reduction_{kind}_seed{seed}",
                    "max_seq_len": m.max_seq_len,
                    "split_threshold": sim.bucket_set.split_threshold,
                    "model": [m.layers, m.heads, m.head_dim, m.bytes_per_elem, m.max_seq_len],
                    "gpu": [base.cluster.gpu.total_mem, base.cluster.gpu.model_mem,
                            base.cluster.gpu.reserve_fraction],
                    "accounting": "exact",
                    "calls": list(log),
                })
        print(f"reduction pairs: 20 seeds, {sum(len(c['calls']) for c in cases[-40:])} calls")
    finally:
        pd_sim.BucketSet, pd_sim.BatchController = orig_bs, orig_bc
        pd_sim.expected_waste = orig_ew
    with gzip.open(OUT, "wt") as fh:
        json.dump(cases, fh)


if __name__ == "__main__":
    main()
