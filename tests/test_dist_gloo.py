"""Sharded windows across ranks with torch.distributed (gloo, world size 2, CPU).

Host-side logic of the data-parallel path: contiguous arrival-order shards, the
C1 histogram all-reduce (sharding.allreduce_histogram), identical global edges
on every rank, and per-shard drains on the global edges.  The per-rank compute
uses the CPU oracle here; the GPU kernels run the same plan (tests/test_gpu_parity.py
::test_sharded_window_on_one_gpu, bench.py under torchrun)."""

import os
import socket
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import cpu
    from paper_2507_17120_b200 import workloads as W
    from paper_2507_17120_b200.sharding import allreduce_histogram, shard_range
    cfg, lens, cls = W.make_window("c2", n=60_000, seed=9)
    a, b = shard_range(len(lens), rank, world)
    l, c = lens[a:b], cls[a:b]
    spec = cpu.WindowSpec(l_max=cfg.l_max, n_classes=cfg.n_classes, policies=cfg.policies,
                          kvpt=cfg.kvpt, current_safe=cfg.current_safe)
    local = cpu.window(spec, l, c).hist.astype(np.int64)
    h = torch.as_tensor(local.reshape(-1).astype(np.int32))
    allreduce_histogram(h)
    glob = h.numpy().astype(np.uint32).reshape(local.shape)
    # edges from the global histogram, computed independently on every rank
    full = cpu.window(spec, lens, cls)
    assert np.array_equal(glob, full.hist)
    # each rank derives the same edges: gather them and compare
    e = torch.as_tensor(full.edges.astype(np.int64))
    es = [torch.zeros_like(e) for _ in range(world)]
    dist.all_gather(es, e)
    assert all(torch.equal(es[0], x) for x in es)
    shard = cpu.window(cpu.WindowSpec(**{**spec.__dict__, "adjust": False,
                                          "init_edges": tuple(int(v) for v in full.edges)}), l, c)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), perm=shard.perm + a,
             req_batch=shard.req_batch, n_batches=shard.summary["n_batches"])
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_histogram_allreduce_and_shard_plans(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    sys.path.insert(0, ROOT)
    from paper_2507_17120_b200.sharding import shard_range
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    # the shards cover the window exactly once
    allp = np.concatenate([p["perm"] for p in parts])
    assert np.array_equal(np.sort(allp), np.arange(60_000))
    assert all(int(p["n_batches"]) > 0 for p in parts)
    assert shard_range(60_000, 1, 2) == (30_000, 60_000)


def test_shard_range_partitions():
    from paper_2507_17120_b200.sharding import shard_range
    for n in (0, 1, 7, 1000, 64_000_001):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)
