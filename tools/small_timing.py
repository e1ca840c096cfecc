"""K0 (k_window_small) phase times from its in-kernel timestamps.
usage: python tools/small_timing.py [1|2]   (1: globaltimer ns, 2: SM cycles -> us at the
current SM clock, 1965 MHz on the B200 pool)"""
import os
import sys

mode = sys.argv[1] if len(sys.argv) > 1 else "2"
os.environ["BS_SMALL_TIMING"] = mode
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_17120_b200 import workloads as W  # noqa: E402
from paper_2507_17120_b200.window import WindowScheduler  # noqa: E402

scale = 1000.0 if mode == "1" else 1965.0
for name, n in (("c1", 1000), ("c2", 2000), ("c2", 500)):
    cfg, lens, cls = W.make_window(name, n=n, seed=1234)
    s = WindowScheduler(max_requests=n, max_seq_len=cfg.l_max, n_classes=cfg.n_classes,
                        policies=cfg.policies, split_threshold=cfg.theta, adjust=cfg.adjust,
                        buckets=cfg.init_edges, kv_bytes_per_token=cfg.kvpt,
                        current_safe=cfg.current_safe, device=torch.device("cuda", 0))
    for _ in range(5):
        r = s.schedule(lens, cls)
    raw = s.summary.cpu().numpy().view(np.int64)
    t = raw[18:30]
    print(name, n, "phase us:", [float(round((t[i + 1] - t[i]) / scale, 2)) for i in range(7)],
          "total", round((t[7] - t[0]) / scale, 2), r.summary()["n_batches"],
          "| K5-A: prep", round((t[8] - t[4]) / scale, 2), "scan", round((t[9] - t[8]) / scale, 2),
          "walk", round((t[5] - t[9]) / scale, 2), "| K3", round((t[10] - t[2]) / scale, 2),
          "K4 pass0", round((t[11] - t[10]) / scale, 2), "pass1", round((t[3] - t[11]) / scale, 2),
          flush=True)
