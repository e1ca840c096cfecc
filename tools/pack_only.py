"""Back-to-back packs of already-scheduled C2 windows on 1-4 streams (bs_pack only, no
scheduling kernels): the in-flight pipeline's pack throughput without the co-running
scheduling of the next windows.  usage: python tools/pack_only.py [--streams 1 2 4]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import torch  # noqa: E402

from paper_2507_17120_b200 import _native as N  # noqa: E402
from paper_2507_17120_b200 import workloads as W  # noqa: E402
from paper_2507_17120_b200.window import WindowScheduler, _ptr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--streams", type=int, nargs="+", default=[1, 2, 4])
ap.add_argument("--steps", type=int, default=100)
a = ap.parse_args()
dev = torch.device("cuda", 0)
cfg, lens_np, cls_np = W.make_window("c2", seed=1234)
lens = torch.as_tensor(lens_np).to(dev)
cls = torch.as_tensor(cls_np).to(dev)
tok_off, tokens = W.token_store_device(lens)
lib = N.load()
S = max(a.streams)
scheds, streams = [], []
for q in range(S):
    s = WindowScheduler(max_requests=len(lens_np), max_seq_len=cfg.l_max, n_classes=cfg.n_classes,
                        policies=cfg.policies, kv_bytes_per_token=cfg.kvpt,
                        current_safe=cfg.current_safe, device=dev)
    r = s.schedule(lens, cls, tok_off, tokens)
    scheds.append(s)
    streams.append(torch.cuda.Stream(dev))
elems = int(r.summary()["packed_elems"])


def pack(q):
    s = scheds[q]
    N.check(lib.bs_pack(s.ctx.ptr, _ptr(lens), _ptr(s.perm), _ptr(tok_off), _ptr(tokens),
                        C.byref(s._params), _ptr(s.batches_raw), 0, -1, _ptr(s.out_tokens),
                        _ptr(s.out_mask), s.pack_capacity, _ptr(s.summary),
                        C.c_void_p(streams[q].cuda_stream)), s.ctx.ptr)


for ns in a.streams:
    for i in range(4 * ns):
        pack(i % ns)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for st in streams[:ns]:
        st.wait_stream(torch.cuda.current_stream())
    for i in range(a.steps):
        pack(i % ns)
    for st in streams[:ns]:
        torch.cuda.current_stream().wait_stream(st)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    print(f"streams {ns}: {ms:.4f} ms per window pack, {4.0037e9 / (ms * 1e-3) / 1e9:.0f} GB/s "
          f"({elems} packed elements)", flush=True)
