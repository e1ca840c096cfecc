"""C1 over peer memory (bs_peer_*): two ranks exchange their length histograms through
CUDA IPC mappings of each other's exchange buffers — on an HGX node that is NVLink
peer memory; here both processes share one B200, which exercises the same IPC mapping,
device-side epochs, system-scope flags and double-buffered slots.  Every window must
equal the torch.distributed all-reduce path (gloo here, NCCL on a multi-GPU box),
eagerly and when the whole window (K1 + exchange + K2..K6) replays as one CUDA graph."""

import os
import socket
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu

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
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    from paper_2507_17120_b200 import workloads as W
    from paper_2507_17120_b200.window import WindowScheduler
    cfg, lens, cls = W.make_window("c2", n=200_000, seed=31, shard=(rank, world))
    tok_off, tokens = W.token_store(lens)
    t = [torch.as_tensor(x).to(dev) for x in (lens, cls, tok_off, tokens)]

    def mk(collective):
        return WindowScheduler(max_requests=len(lens), max_seq_len=cfg.l_max,
                               n_classes=cfg.n_classes, policies=cfg.policies,
                               kv_bytes_per_token=cfg.kvpt, current_safe=cfg.current_safe,
                               device=dev, process_group=dist.group.WORLD, collective=collective)

    ref = mk("torch").schedule(*t).to_host()
    peer = mk("peer")
    outs = [peer.schedule(*t).to_host()]
    for _ in range(4):  # several epochs through both exchange slots, as one CUDA graph each
        outs.append(peer.schedule(*t, graph=True).to_host())
    ok = True
    for h in outs:
        for k in ("edges", "perm", "req_batch", "req_row", "out_tokens", "out_mask"):
            ok &= bool(np.array_equal(h[k], ref[k]))
        ok &= int(h["summary"]["total_global"]) == 200_000
        ok &= int(h["summary"]["flags"]) == 0
    with open(os.path.join(out_dir, f"rank{rank}.txt"), "w") as fh:
        fh.write("ok" if ok else "mismatch")
    dist.barrier()
    dist.destroy_process_group()


def test_peer_histogram_exchange_two_ranks(tmp_path):
    if torch.cuda.device_count() < 1:
        pytest.skip("needs a GPU")
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        assert (tmp_path / f"rank{r}.txt").read_text() == "ok"
