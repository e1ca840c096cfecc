"""Generate tests/golden/*.npz from the UNMODIFIED reference (bucketsim).

TEST INFRASTRUCTURE.  Run in the build container (needs /root/reference):
    python -m oracle.gen_golden
Each fixture stores the window inputs, its parameters and the reference's
result in the canonical shape of oracle/canon.py.  The cases cover the
BASELINE configs at reduced N plus every edge case the reference tests pin
(SURVEY §8c): fixed edges, adaptive fixpoint, theta float hazard
(test P6: 0.29), width/merge/skip, LJF/SJF/FCFS, EXACT/PADDED, oversize
rejection, pledged headroom blocking, zero headroom, empty and tiny windows,
truncation, zero lengths, four classes.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle.ref_compose import available, reference_window  # noqa: E402
from paper_2507_17120_b200 import workloads as W  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def _case(name, lens, cls, **spec):
    return name, np.asarray(lens, np.int32), np.asarray(cls, np.uint8), spec


def cases():
    out = []
    rng = np.random.default_rng(20261017)
    # --- BASELINE configs at fixture scale --------------------------------------
    for cname, n in (("c1", 1000), ("c2", 30000), ("c3", 20000), ("c4", 6000)):
        cfg, lens, cls = W.make_window(cname, n=n, seed=7)
        out.append(_case(f"{cname}_n{n}", lens, cls, l_max=cfg.l_max, n_classes=cfg.n_classes,
                         policies=cfg.policies, theta=cfg.theta, adjust=cfg.adjust,
                         init_edges=cfg.init_edges, kvpt=cfg.kvpt, current_safe=cfg.current_safe,
                         accounting=cfg.accounting))
    # C2 distribution, EXACT accounting, LJF offline
    cfg, lens, cls = W.make_window("c2", n=20000, seed=11)
    out.append(_case("c2_exact_ljf", lens, cls, l_max=4096, n_classes=2, policies=(0, 2),
                     kvpt=cfg.kvpt, current_safe=cfg.current_safe, accounting=1))
    # C2 distribution, FCFS both (continuous proxy ordering, pd_sim.py:312-313), theta 1.0
    out.append(_case("c2_fcfs_theta1", lens[:8000], cls[:8000], l_max=4096, n_classes=2,
                     policies=(0, 0), theta=1.0, kvpt=cfg.kvpt, current_safe=cfg.current_safe))
    # theta float hazard values
    for th in (0.29, 0.57, 0.7):
        l = np.clip(np.rint(rng.lognormal(4.0, 1.0, size=3000)), 1, 999)
        c = rng.integers(0, 2, size=3000)
        out.append(_case(f"theta_{th}", l, c, l_max=1000, n_classes=2, policies=(0, 1), theta=th,
                         kvpt=2, current_safe=2 * 30000))
    # tiny l_max, deep splits, zero lengths, LJF, small budgets -> rejections
    for L in (2, 7, 64, 100):
        l = np.minimum(rng.geometric(3.0 / L if L > 3 else 0.5, size=2000) - 1, L - 1)
        c = rng.integers(0, 2, size=2000)
        out.append(_case(f"tiny_L{L}_ljf_exact", l, c, l_max=L, n_classes=2, policies=(0, 2),
                         theta=0.3, kvpt=4, current_safe=4 * 3 * L, accounting=1))
        out.append(_case(f"tiny_L{L}_sjf_padded", l, c, l_max=L, n_classes=2, policies=(0, 1),
                         theta=0.5, kvpt=4, current_safe=4 * 5 * L, accounting=0))
    # oversize rejection heavy: budget below many lengths
    l = rng.integers(1, 4096, size=5000)
    c = rng.integers(0, 2, size=5000)
    for acc in (0, 1):
        out.append(_case(f"reject_heavy_acc{acc}", l, c, l_max=4096, n_classes=2, policies=(1, 2),
                         kvpt=6, current_safe=6 * 1500 + 5, accounting=acc))
    # pledged > 0: drains stop at a request that does not fit the headroom
    for acc in (0, 1):
        out.append(_case(f"pledged_acc{acc}", l[:3000], c[:3000], l_max=4096, n_classes=2,
                         policies=(0, 1), kvpt=2, current_safe=2 * 4000, pledged=2 * 1500 + 1,
                         accounting=acc))
    # zero headroom -> nothing scheduled, nothing rejected
    out.append(_case("zero_headroom", l[:500], c[:500], l_max=4096, n_classes=2, policies=(0, 1),
                     kvpt=2, current_safe=0))
    # empty window and single request
    out.append(_case("empty", [], [], l_max=4096, n_classes=2, policies=(0, 1), kvpt=2,
                     current_safe=2 * 10000))
    out.append(_case("single", [17], [1], l_max=4096, n_classes=2, policies=(0, 1), kvpt=2,
                     current_safe=2 * 10000))
    # truncation of over-long inputs (pd_sim.py:382-383)
    lt = rng.integers(1, 6000, size=3000)
    out.append(_case("truncate", lt, c[:3000], l_max=4096, n_classes=2, policies=(0, 1), kvpt=2,
                     current_safe=2 * 20000))
    # identical lengths (equal-length SJF runs)
    out.append(_case("equal_lengths", np.full(5000, 333), c[:5000], l_max=4096, n_classes=2,
                     policies=(0, 1), kvpt=2, current_safe=2 * 333 * 37 + 1))
    # 4 classes mixed policies, EXACT
    l4 = rng.integers(1, 2048, size=8000)
    c4 = rng.integers(0, 4, size=8000)
    out.append(_case("four_class_exact", l4, c4, l_max=2048, n_classes=4, policies=(0, 1, 2, 0),
                     kvpt=2, current_safe=2 * 50000, accounting=1))
    # stateful forms: one pass from given edges (merge and split branches)
    out.append(_case("one_pass_split", l[:4000], c[:4000], l_max=4096, n_classes=2,
                     policies=(0, 1), init_edges=(0, 1024, 2048, 4096), max_passes=1, kvpt=2,
                     current_safe=2 * 20000))
    out.append(_case("one_pass_merge", l[:40], c[:40], l_max=4096, n_classes=2, policies=(0, 1),
                     init_edges=(0, 100, 1024, 4096), max_passes=1, kvpt=2,
                     current_safe=2 * 10 ** 6))
    out.append(_case("fixed_edges_no_adjust", l[:4000], c[:4000], l_max=4096, n_classes=2,
                     policies=(0, 1), init_edges=(0, 256, 1024, 4096), adjust=False, kvpt=2,
                     current_safe=2 * 20000))
    # f3 dispatch-order stress: whole buckets of oversize ONLINE requests (null calls
    # that cascade to OFFLINE inside one _next_plan), equal offline masses (ties to
    # the lower bucket), and a blocked ONLINE drain under pledged memory
    ld = rng.integers(1, 4096, size=6000)
    cd = (rng.random(6000) < 0.3).astype(np.uint8)
    out.append(_case("dispatch_online_rejects", ld, cd, l_max=4096, n_classes=2, policies=(0, 1),
                     init_edges=(0, 512, 1024, 2048, 3072, 4096), adjust=False, kvpt=2,
                     current_safe=2 * 1800))
    lt = np.repeat(np.array([100, 700, 1500, 2500], np.int32), 50)
    ct = np.ones(len(lt), np.uint8)
    ct[::7] = 0
    out.append(_case("dispatch_mass_ties", lt, ct, l_max=4096, n_classes=2, policies=(0, 2),
                     init_edges=(0, 512, 1024, 2048, 4096), adjust=False, kvpt=2,
                     current_safe=2 * 2600, accounting=1))
    out.append(_case("dispatch_pledged_block", ld[:2500], cd[:2500], l_max=4096, n_classes=2,
                     policies=(0, 1), kvpt=2, current_safe=2 * 4000, pledged=2 * 1200 + 1))
    return out


def main():
    if not available():
        raise SystemExit("reference not available (needs /root/reference)")
    os.makedirs(OUT, exist_ok=True)
    for name, lens, cls, spec in cases():
        spec = dict(spec)
        # the simulator's global dispatch sequence (f3) where the reference defines it
        ref = reference_window(lens, cls, dispatch=spec.get("n_classes", 2) == 2, **spec)
        init = spec.get("init_edges")
        np.savez_compressed(
            os.path.join(OUT, f"{name}.npz"), lens=lens, cls=cls,
            l_max=spec["l_max"], n_classes=spec.get("n_classes", 2),
            policies=np.array(spec.get("policies", (0, 1)), np.int32),
            theta=spec.get("theta", 0.5), adjust=int(spec.get("adjust", True)),
            max_passes=spec.get("max_passes", 0),
            init_edges=np.array(init if init is not None else [], np.int32),
            kvpt=spec["kvpt"], current_safe=spec["current_safe"],
            pledged=spec.get("pledged", 0), accounting=spec.get("accounting", 0),
            truncate=int(spec.get("truncate", True)),
            **{f"ref_{k}": v for k, v in ref.items()})
        print(f"{name:28s} N={len(lens):6d} K={len(ref['edges']) - 1:4d} "
              f"batches={len(ref['batch_meta']):5d} rej={len(ref['rejected']):5d} "
              f"pend={len(ref['pending']):5d}")


if __name__ == "__main__":
    main()
