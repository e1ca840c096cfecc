"""Per-stage device times of the fused window (CUDA events inside the library)."""
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
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--no-pack", action="store_true")
ap.add_argument("--dispatch", action="store_true")
ap.add_argument("--no-mask", action="store_true")
ap.add_argument("--policies", default=None, help="override, e.g. fcfs,sjf,sjf,sjf")
a = ap.parse_args()
cfg, lens_np, cls_np = W.make_window(a.config, n=a.n, seed=1234)
dev = torch.device("cuda", 0)
lens = torch.as_tensor(lens_np).to(dev)
cls = torch.as_tensor(cls_np).to(dev)
tok_off = tokens = None
if not a.no_pack:
    tok_off, tokens = W.token_store_device(lens)
pol = cfg.policies
if a.policies:
    names = {"fcfs": 0, "sjf": 1, "ljf": 2}
    pol = tuple(names[x] for x in a.policies.split(","))
s = WindowScheduler(max_requests=len(lens_np), max_seq_len=cfg.l_max, n_classes=cfg.n_classes,
                    policies=pol, split_threshold=cfg.theta, adjust=cfg.adjust,
                    buckets=cfg.init_edges, kv_bytes_per_token=cfg.kvpt,
                    current_safe=cfg.current_safe, accounting=cfg.accounting, device=dev,
                    dispatch=a.dispatch, with_mask=not a.no_mask)
r = s.schedule(lens, cls, tok_off, tokens)
for _ in range(3):
    s.schedule(lens, cls, tok_off, tokens, sync=False)
torch.cuda.synchronize()
s.ctx.profile_enable(a.steps)
for _ in range(a.steps):
    s.schedule(lens, cls, tok_off, tokens, sync=False)
torch.cuda.synchronize()
ms, k = s.ctx.profile_read()
out = {kk: round(v / k * 1000, 1) for kk, v in ms.items()}
print(json.dumps({"config": a.config, "n": len(lens_np), "stage_us": out,
                  "total_us": round(sum(out.values()), 1), "summary": r.summary()}))
