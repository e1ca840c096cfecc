"""One-window latency (CUDA graph replay, one window at a time) and per-stage times
for tuning-hook settings read by bs_create.  usage:
  python tools/latency_sweep.py --config c2 --env BS_CHAIN_WALK=16,32,128 [--no-pack]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2507_17120_b200 import workloads as W  # noqa: E402
from paper_2507_17120_b200.window import WindowScheduler  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--env", action="append", default=[], help="NAME=v1,v2,...")
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--no-pack", action="store_true")
a = ap.parse_args()
cfg, lens_np, cls_np = W.make_window(a.config, n=a.n, seed=1234)
dev = torch.device("cuda", 0)
lens = torch.as_tensor(lens_np).to(dev)
cls = torch.as_tensor(cls_np).to(dev)
tok_off = tokens = None
if not a.no_pack:
    tok_off, tokens = W.token_store_device(lens)
combos = [{}]
for spec in a.env:
    name, vals = spec.split("=")
    combos = [dict(c, **{name: v}) for c in combos for v in vals.split(",")]
ref = None
for env in combos:
    for k, v in env.items():
        os.environ[k] = v
    s = WindowScheduler(max_requests=len(lens_np), max_seq_len=cfg.l_max, n_classes=cfg.n_classes,
                        policies=cfg.policies, split_threshold=cfg.theta, adjust=cfg.adjust,
                        buckets=cfg.init_edges, kv_bytes_per_token=cfg.kvpt,
                        current_safe=cfg.current_safe, accounting=cfg.accounting, device=dev)
    for k in env:
        del os.environ[k]
    r = s.schedule(lens, cls, tok_off, tokens)
    h = r.summary()
    key = (h["n_batches"], h["packed_elems"], int(r.req_batch.sum().item()))
    ref = ref or key
    for _ in range(3):
        s.schedule(lens, cls, tok_off, tokens, sync=False, graph=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        s.schedule(lens, cls, tok_off, tokens, sync=False, check=False, graph=True)
    e1.record()
    torch.cuda.synchronize()
    lat = e0.elapsed_time(e1) / a.steps * 1000
    s.ctx.profile_enable(a.steps)
    for _ in range(a.steps):
        s.schedule(lens, cls, tok_off, tokens, sync=False, check=False)
    torch.cuda.synchronize()
    ms, k = s.ctx.profile_read()
    st = {kk: round(v / k * 1000, 1) for kk, v in ms.items() if v}
    print(json.dumps({"config": a.config, "env": env, "graph_latency_us": round(lat, 1),
                      "stage_us": st, "same_result": key == ref}), flush=True)
    s.close()
