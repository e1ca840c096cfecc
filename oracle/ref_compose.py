"""Run the UNMODIFIED reference (bucketsim) on a window — golden-vector generator.

TEST INFRASTRUCTURE ONLY; needs /root/reference (present in the build container,
absent on the GPU box) or its unmodified pip install under baseline/_ref (made by
__graft_entry__.build(), git-ignored, shipped to the GPU box).  It composes the reference's own public classes exactly
as SURVEY §3.4 describes the window:

  1. BucketSet(L_max, split_threshold[, buckets])           bucket_manager.py:79-97
  2. assign every request in arrival order                    bucket_manager.py:110-131
  3. n_max = BatchController.current_n_max(bucket_set)        batch_controller.py:93-104
     adjust_buckets(n_max) until a pass yields no split       bucket_manager.py:133-191
  4. for each bucket (left to right), for each class in priority order,
     form_batch(bucket, policy, pledged, task_class) until None
                                                              batch_controller.py:141-191

Classes: class 0 = TaskClass.ONLINE, class 1 = TaskClass.OFFLINE; classes >= 2
are opaque sentinel objects — form_batch's filter is an identity test
(`r.task_class is task_class`, batch_controller.py:155), so the reference's own
code drains them (the 4-class generalisation pinned to reference code).
"""

from __future__ import annotations

import os
import sys
import copy
from collections import deque

import numpy as np

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# the reference sources in the build container, else the unmodified package installed
# by `pip install --target baseline/_ref` (git-ignored; it travels to the GPU box)
REF_SRC = os.environ.get("BUCKETSIM_REF_SRC") or next(
    (p for p in ("/root/reference/pkg/src", os.path.join(_ROOT, "baseline", "_ref"))
     if os.path.isdir(os.path.join(p, "bucketsim"))), "/root/reference/pkg/src")


def available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "bucketsim"))


def _import():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    sys.dont_write_bytecode = True
    import bucketsim  # noqa: F401
    from bucketsim import batch_controller, bucket_manager, memory_model, workload
    return bucket_manager, batch_controller, memory_model, workload


class _Cls:
    def __init__(self, i):
        self.i = i

    def __repr__(self):
        return f"Class{self.i}"


def reference_window(lens, cls, *, l_max, n_classes=2, policies=(0, 1), theta=0.5,
                     adjust=True, max_passes=0, init_edges=None, model=None, gpu=None,
                     kvpt=None, current_safe=None, accounting=0, pledged=0, truncate=True,
                     dispatch=False):
    """Returns a dict of numpy arrays describing the reference's window result.

    Memory can be given as (model, gpu) reference objects, or as raw
    (kvpt, current_safe) — the latter builds a ModelConfig with
    kv_bytes_per_token == kvpt when possible and overrides current_safe through
    BatchController.on_memory_change (batch_controller.py:83-88)."""
    bm, bc, mm, wl = _import()
    TaskClass = wl.TaskClass
    class_objs = [TaskClass.ONLINE, TaskClass.OFFLINE] + [_Cls(i) for i in range(2, n_classes)]
    class_objs = class_objs[:n_classes]
    pol_map = {0: bc.DispatchPolicy.FCFS, 1: bc.DispatchPolicy.SJF, 2: bc.DispatchPolicy.LJF}
    acc = bc.MemoryAccounting.PADDED if accounting == 0 else bc.MemoryAccounting.EXACT

    if model is None:
        # kv_bytes_per_token = 2*L*H*D*B; pick L=kvpt/2 with H=D=B=1 when even,
        # else B=... kvpt must be even for a ModelConfig; callers use even kvpt.
        assert kvpt is not None and kvpt % 2 == 0
        model = mm.ModelConfig(layers=kvpt // 2, heads=1, head_dim=1, bytes_per_elem=1,
                               max_seq_len=max(l_max, 1))
        gpu = mm.GpuConfig(total_mem=max(current_safe, 0), model_mem=0, reserve_fraction=0.0)
    ctl = bc.BatchController(model, gpu, acc)
    if current_safe is not None and current_safe != ctl.current_safe:
        ctl.on_memory_change(current_safe)

    reqs = []
    for i, (x, c) in enumerate(zip(np.asarray(lens).tolist(), np.asarray(cls).tolist())):
        if truncate and x >= l_max:          # pd_sim.py:382-383
            x = l_max - 1
        reqs.append(wl.Request(i, float(i), int(x), 1, class_objs[int(c)]))
    buckets = None
    if init_edges is not None:
        buckets = [bm.Bucket(int(lo), int(up)) for lo, up in zip(init_edges[:-1], init_edges[1:])]
    bs = bm.BucketSet(l_max, theta, buckets=buckets)
    for r in reqs:
        bs.assign(r)
    n_max = ctl.current_n_max(bs)
    changes = []
    passes = 0
    if adjust:
        while True:
            ch = bs.adjust_buckets(n_max)
            passes += 1
            changes.extend(ch)
            if not any(c.kind == "split" for c in ch):
                break
            if max_passes and passes >= max_passes:
                break
    edges = [b.low for b in bs.buckets] + [bs.buckets[-1].up]
    bucket_of = np.full(len(reqs), -1, np.int64)
    for bi, b in enumerate(bs.buckets):
        for r in b.requests:
            bucket_of[r.id] = bi

    dispatch_bs = dispatch_ctl = None
    if dispatch:
        # the simulator's dispatch loop runs on its own copy of the adjusted buckets
        dispatch_bs = copy.deepcopy(bs)
        dispatch_ctl = bc.BatchController(model, gpu, acc)
        if current_safe is not None and current_safe != dispatch_ctl.current_safe:
            dispatch_ctl.on_memory_change(current_safe)

    kind_code = {"split": 1, "merge": 2, "skip": 3}
    ch_arr = np.array([[kind_code[c.kind], c.parent_low, c.parent_up,
                        -1 if c.midpoint is None else c.midpoint] for c in changes],
                      dtype=np.int64).reshape(-1, 4)

    batch_ids, batch_off, meta, waste = [], [0], [], []
    for bi, b in enumerate(bs.buckets):
        for ci, cobj in enumerate(class_objs):
            while True:
                plan = ctl.form_batch(b, pol_map[policies[ci]], pledged=pledged, task_class=cobj)
                if plan is None:
                    break
                batch_ids.extend(plan.request_ids)
                batch_off.append(len(batch_ids))
                meta.append((bi * n_classes + ci, len(plan), plan.max_input_len, plan.token_sum,
                             plan.footprint))
                try:
                    waste.append(mm.waste_ratio([r.input_len for r in plan.requests]))
                except ValueError:
                    waste.append(np.nan)
    rejected = [rej.request.id for rej in ctl.rejections]
    pending = sorted(r.id for r in bs.iter_requests())
    if dispatch_bs is not None:
        extra = _dispatch_loop(dispatch_bs, dispatch_ctl, class_objs, pol_map, policies, pledged,
                               TaskClass)
    else:
        extra = {}
    return dict(
        **extra,
        n_max=np.int64(n_max), edges=np.array(edges, np.int64), changes=ch_arr,
        n_passes=np.int64(passes), bucket=bucket_of,
        batch_ids=np.array(batch_ids, np.int64), batch_off=np.array(batch_off, np.int64),
        batch_meta=np.array(meta, np.int64).reshape(-1, 5),
        batch_waste=np.array(waste, np.float64),
        rejected=np.array(rejected, np.int64), pending=np.array(pending, np.int64),
        current_safe=np.int64(ctl.current_safe), kvpt=np.int64(ctl.kv_per_token),
    )


def _dispatch_loop(bs, ctl, class_objs, pol_map, policies, pledged, TaskClass):
    """Simulator._next_plan (pd_sim.py:448-462) repeated while it makes progress:
    for each class in priority order, select_bucket (batch_controller.py:106-134)
    then form_batch on that bucket; the first plan ends the call.  Progress = a plan
    or new rejections (the simulator marks the set dirty and would call again,
    pd_sim.py:457-459).  Two classes only: select_bucket knows ONLINE / OFFLINE."""
    assert len(class_objs) == 2, "the reference's select_bucket has two classes"
    seq, off, rejected = [], [0], []
    while True:
        plan, progressed = None, False
        for ci, cobj in enumerate(class_objs):
            idx = ctl.select_bucket(bs, cobj)
            if idx is None:
                continue
            plan = ctl.form_batch(bs.buckets[idx], pol_map[policies[ci]], pledged=pledged,
                                  task_class=cobj)
            if ctl.rejections:
                progressed = True
                rejected.extend(rej.request.id for rej in ctl.rejections)
                ctl.rejections.clear()
            if plan is not None:
                break
        if plan is not None:
            seq.extend(plan.request_ids)
            off.append(len(seq))
            continue
        if not progressed:
            break
    return dict(disp_ids=np.array(seq, np.int64), disp_off=np.array(off, np.int64),
                disp_rejected=np.array(sorted(rejected), np.int64),
                disp_pending=np.array(sorted(r.id for r in bs.iter_requests()), np.int64))
