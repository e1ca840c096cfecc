"""C1 over the library's own NCCL communicator (bs_nccl_* / bs_set_nccl).

A box here has one GPU, and NCCL refuses two ranks on one device, so the
communicator is exercised at world size 1 — the all-reduce is then the identity and
the point is the plumbing: the collective is issued by bs_window_schedule between
K1 and K2 on the window's stream and is captured, with the rest of the window, into
one CUDA graph.  The multi-rank host logic runs under gloo (tests/test_dist_gloo.py,
and bench.py --gpus 2 --share-gpus below)."""

import ctypes as C
import json
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2507_17120_b200 import _native as N  # noqa: E402
from paper_2507_17120_b200 import workloads as W  # noqa: E402
from paper_2507_17120_b200.window import WindowScheduler  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sched(cfg, n, **kw):
    return WindowScheduler(max_requests=n, max_seq_len=cfg.l_max, n_classes=cfg.n_classes,
                           policies=cfg.policies, kv_bytes_per_token=cfg.kvpt,
                           current_safe=cfg.current_safe, device=torch.device("cuda", 0), **kw)


def _host(res):
    h = res.to_host()
    return {k: h[k] for k in ("edges", "perm", "bucket", "req_batch", "req_row", "changes")}, h


def test_nccl_world1_window_in_graph_equals_plain():
    cfg, lens, cls = W.make_window("c2", n=200_000, seed=5)
    tok_off, tokens = W.token_store(lens)
    d = lambda x: torch.as_tensor(x).cuda(0)  # noqa: E731
    dl, dc, do, dt = d(lens), d(cls), d(tok_off), d(tokens)
    plain = _sched(cfg, len(lens))
    ref, ref_h = _host(plain.schedule(dl, dc, do, dt))
    s = _sched(cfg, len(lens))
    s.attach_nccl(0, 1, WindowScheduler.nccl_unique_id())
    for graph in (False, True, True):
        res = s.schedule(dl, dc, do, dt, graph=graph)
        got, h = _host(res)
        for k in ref:
            assert np.array_equal(got[k], ref[k]), (graph, k)
        assert np.array_equal(h["batches"], ref_h["batches"])
        m = int(h["summary"]["packed_elems"])
        assert np.array_equal(h["out_tokens"][:m], ref_h["out_tokens"][:m])
        assert torch.equal(s.hist_global, s.hist)
    # the exchange stage is recorded between K1 and K2
    s.ctx.profile_enable(3)
    for _ in range(3):
        s.schedule(dl, dc, do, dt, sync=False, check=False)
    torch.cuda.synchronize()
    ms, steps = s.ctx.profile_read()
    assert steps == 3 and ms["exchange"] > 0 and ms["pack"] > 0
    s.close()
    plain.close()


def test_nccl_allreduce_and_detach_through_the_c_abi():
    lib = N.load()
    cfg, lens, cls = W.make_window("c1", n=1000, seed=2)
    s = _sched(cfg, len(lens))
    s.attach_nccl(0, 1, WindowScheduler.nccl_unique_id())
    h = s.histogram(lens, cls)
    out = torch.zeros_like(s.hist)
    with torch.cuda.device(0):
        N.check(lib.bs_nccl_allreduce(s.ctx.ptr, C.c_void_p(s.hist.data_ptr()), C.byref(s._params),
                                      C.c_void_p(out.data_ptr()),
                                      C.c_void_p(torch.cuda.current_stream().cuda_stream)),
                s.ctx.ptr)
    torch.cuda.synchronize()
    assert torch.equal(out.view_as(h), h.cuda())
    # detach: the fused call no longer runs C1 and then needs no hist_global
    N.check(lib.bs_set_nccl(s.ctx.ptr, None, 0, 0), s.ctx.ptr)
    with pytest.raises(ValueError):
        lib_rc = lib.bs_nccl_allreduce(s.ctx.ptr, C.c_void_p(s.hist.data_ptr()), C.byref(s._params),
                                       C.c_void_p(out.data_ptr()), None)
        N.check(lib_rc, s.ctx.ptr)
    s.close()


def test_bench_spawns_ranks_on_shared_gpu():
    """`bench.py --gpus 2` on a one-GPU box: refused without --share-gpus, and with it two
    ranks (gloo, ranks sharing the GPU) print one line with n_gpus 2 and the C1 time."""
    base = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
            "--warmup", "3", "--requests", "50000", "--no-e2e", "--no-cpu-baseline"]
    if torch.cuda.device_count() < 2:
        r = subprocess.run(base, capture_output=True, text=True, timeout=600, cwd=ROOT)
        assert r.returncode == 0 and "unavailable" in json.loads(r.stdout.strip().splitlines()[-1])
    r = subprocess.run(base + ["--share-gpus"], capture_output=True, text=True, timeout=900,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["c1"]["ms_per_window"] > 0
