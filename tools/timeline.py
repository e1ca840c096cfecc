"""Device timeline of windows in flight (the bench's pipelined loop) from CUPTI kernel
records (torch.profiler), to see how the scheduling kernels of one window overlap the
pack of another.  Usage: python tools/timeline.py [--config c2] [--inflight 4] [--windows 12]
Writes gpurun_out/timeline_<config>.json (kernel, stream, start, duration in us) and prints
per-window spans and the pack-busy fraction of the traced interval."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2507_17120_b200 import workloads as W  # noqa: E402
from paper_2507_17120_b200.window import WindowScheduler  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--inflight", type=int, default=4)
ap.add_argument("--windows", type=int, default=12)
ap.add_argument("--no-graph", action="store_true")
ap.add_argument("--out", default=None)
a = ap.parse_args()
cfg, lens_np, cls_np = W.make_window(a.config, n=a.n, seed=1234)
dev = torch.device("cuda", 0)
lens = torch.as_tensor(lens_np).to(dev)
cls = torch.as_tensor(cls_np).to(dev)
tok_off, tokens = W.token_store_device(lens)
mk = lambda cap=None: WindowScheduler(  # noqa: E731
    max_requests=len(lens_np), max_seq_len=cfg.l_max, n_classes=cfg.n_classes,
    policies=cfg.policies, split_threshold=cfg.theta, adjust=cfg.adjust, buckets=cfg.init_edges,
    kv_bytes_per_token=cfg.kvpt, current_safe=cfg.current_safe, accounting=cfg.accounting,
    device=dev, pack_capacity=cap)
s0 = mk()
s0.schedule(lens, cls, tok_off, tokens)
scheds = [s0] + [mk(s0.pack_capacity) for _ in range(a.inflight - 1)]
streams = [torch.cuda.Stream(dev) for _ in range(a.inflight)]


def run(k):
    cur = torch.cuda.current_stream(dev)
    for st in streams:
        st.wait_stream(cur)
    for i in range(k):
        q = i % a.inflight
        with torch.cuda.stream(streams[q]):
            scheds[q].schedule(lens, cls, tok_off, tokens, sync=False, check=False,
                               graph=not a.no_graph)
    for st in streams:
        cur.wait_stream(st)


run(2 * a.inflight)
torch.cuda.synchronize(dev)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run(a.windows)
    torch.cuda.synchronize(dev)
out = a.out or os.path.join("gpurun_out", f"timeline_{a.config}.json")
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
tmp = out + ".trace"
prof.export_chrome_trace(tmp)
ev = json.load(open(tmp))["traceEvents"]
os.remove(tmp)
ks = [e for e in ev if e.get("cat") == "kernel"]
ks.sort(key=lambda e: e["ts"])
t0 = ks[0]["ts"]
rows = [{"k": e["name"].split("(")[0].replace("void ", "").replace("bsk::", "")[:40],
         "stream": e.get("args", {}).get("stream"), "t": round(e["ts"] - t0, 2),
         "d": round(e["dur"], 2)} for e in ks]
json.dump(rows, open(out, "w"))
span = rows[-1]["t"] + rows[-1]["d"]
# pack-busy: union of intervals of the pack kernels
iv = sorted((r["t"], r["t"] + r["d"]) for r in rows if "k_pack" in r["k"] and "rowprep" not in r["k"])
busy, cs, ce = 0.0, None, None
for s, e in iv:
    if cs is None or s > ce:
        if cs is not None:
            busy += ce - cs
        cs, ce = s, e
    else:
        ce = max(ce, e)
if cs is not None:
    busy += ce - cs
print(f"{len(rows)} kernels over {span:.1f} us ({span / a.windows:.1f} us/window); "
      f"pack busy {busy:.1f} us = {100 * busy / span:.1f}%")
for r in rows:
    print(f"{r['t']:9.1f} {r['d']:8.1f}  s{r['stream']}  {r['k']}")
