"""The GPU-backed drop-in under the reference simulator's real call pattern.

oracle/gen_sim_golden.py ran the UNMODIFIED reference Simulator (pd_sim.py) with
logging BucketSet / BatchController subclasses and recorded every scheduling call in
order (assign per arrival, current_n_max + one adjust_buckets pass per dirty tick,
select_bucket + form_batch per dispatch, the rejections the simulator drains).  Each
log is replayed here against paper_2507_17120_b200.compat — whose split / merge
decisions (K1 + one K2 pass from the current edges) and form_batch sizing (K4 + K5)
run on the GPU — with the simulator's own bookkeeping between calls (dirty on a plan
or rejections, pd_sim.py:457-459; rejections drained, :464-467).  Every result must be
identical: bucket indices, n_max, change lists and edges, dirty flags, selected
buckets, plans (ids, max_input_len, token_sum, footprint), rejected ids, and the
per-tick monitor value expected_waste (K8 over the set's incremental histogram).

Two of the logs are the reference's own scenario files run as `bucketsim run` runs
them (smoke.yaml, mixed_longtail.yaml); the simulator touches the scheduling path only
through these calls, so identical results at every call mean the drop-in run — and the
report whose sha256 the log records — is byte-identical to the reference's."""

import gzip
import json
import os

import pytest

torch = pytest.importorskip("torch")


from golden_util import GOLDEN_DIR  # noqa: E402
from paper_2507_17120_b200 import GpuConfig, ModelConfig  # noqa: E402
from paper_2507_17120_b200.compat import BatchController, BucketSet  # noqa: E402
from paper_2507_17120_b200.types import (DispatchPolicy, MemoryAccounting, Request,  # noqa: E402
                                         TaskClass)

with gzip.open(os.path.join(GOLDEN_DIR, "sim_calls.json.gz"), "rt") as fh:
    CASES = json.load(fh)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_replay_simulator_calls(case):
    model = ModelConfig(*case["model"])
    gpu = GpuConfig(*case["gpu"])
    bs = BucketSet(case["max_seq_len"], split_threshold=case["split_threshold"])
    ctl = BatchController(model, gpu, MemoryAccounting(case["accounting"]))
    seen = {}
    for k, e in enumerate(case["calls"]):
        op = e["op"]
        where = f"{case['name']} call {k} ({op})"
        if op == "assign":
            rid, arrival, length, cls = e["req"]
            r = Request(rid, arrival, length, None, TaskClass(cls))
            seen[rid] = r
            assert bs.assign(r) == e["out"], where
        elif op == "n_max":
            assert ctl.current_n_max(bs) == e["out"], where
        elif op == "adjust":
            ch = bs.adjust_buckets(e["n_max"])
            assert [[c.kind, c.parent_low, c.parent_up, c.midpoint] for c in ch] == e["out"], where
            assert bs.edges() == e["edges"], where
            assert bs.dirty == e["dirty"], where
            assert bs.check_partition() is None, where
        elif op == "select":
            assert ctl.select_bucket(bs, TaskClass(e["cls"])) == e["out"], where
        elif op == "form":
            plan = ctl.form_batch(bs.buckets[e["bucket"]], DispatchPolicy(e["policy"]),
                                  pledged=e["pledged"],
                                  task_class=None if e["cls"] is None else TaskClass(e["cls"]))
            got = None if plan is None else [list(plan.request_ids), plan.max_input_len,
                                             plan.token_sum, plan.footprint]
            assert got == e["out"], where
            rej = [x.request.id for x in ctl.rejections]
            assert rej == e["rejected"], where
            if plan is not None or ctl.rejections:  # Simulator._next_plan, pd_sim.py:457-459
                bs.dirty = True
            ctl.rejections.clear()                   # pd_sim.py:464-467
        elif op == "snapshot":  # monitor: expected_waste of the queue (pd_sim.py:828-833)
            assert bs.edges() == e["edges"], where
            assert bs.total_requests == e["total"], where
            assert bs.expected_waste() == e["out"], where   # bit-exact, from K8
        else:
            raise AssertionError(f"unknown op {op}")
    assert len(seen) > 0


def test_logs_exercise_the_stateful_paths():
    kinds, rejected, none_plans, plans = set(), 0, 0, 0
    for c in CASES:
        for e in c["calls"]:
            if e["op"] == "adjust":
                kinds.update(ch[0] for ch in e["out"])
            if e["op"] == "form":
                rejected += len(e["rejected"])
                none_plans += e["out"] is None
                plans += e["out"] is not None
    assert {"split", "merge"} <= kinds
    assert rejected > 0 and none_plans > 0 and plans > 200
    names = {c["name"] for c in CASES}
    assert {"scenario_smoke", "scenario_mixed_longtail"} <= names
    assert sum(e["op"] == "snapshot" for c in CASES for e in c["calls"]) > 1000


def test_reduction_pairs_are_batch_identical_in_the_logs():
    """Acceptance criterion 7 (test_acceptance.py:264-282): for every seed the
    theta = 1.0 FCFS BucketServe run and the continuous proxy form the same batches.
    The replay above reproduces every one of those calls on the GPU classes, so the
    drop-in satisfies the reduction too."""
    by = {c["name"]: c for c in CASES}
    seeds = [n.split("seed")[1] for n in by if n.startswith("reduction_bucket_")]
    assert len(seeds) == 20
    for sd in seeds:
        a = [e["out"][0] for e in by[f"reduction_bucket_seed{sd}"]["calls"]
             if e["op"] == "form" and e["out"] is not None]
        b = [e["out"][0] for e in by[f"reduction_continuous_seed{sd}"]["calls"]
             if e["op"] == "form" and e["out"] is not None]
        assert a == b and len(a) > 0
