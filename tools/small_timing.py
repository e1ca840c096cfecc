import os, sys, torch, numpy as np
os.environ["BS_SMALL_TIMING"]="1"
sys.path.insert(0, os.getcwd())
from paper_2507_17120_b200 import workloads as W
from paper_2507_17120_b200.window import WindowScheduler
for name, n in (("c1", 1000), ("c2", 2000), ("c2", 500)):
    cfg, lens, cls = W.make_window(name, n=n, seed=1234)
    s = WindowScheduler(max_requests=n, max_seq_len=cfg.l_max, n_classes=cfg.n_classes, policies=cfg.policies,
                        split_threshold=cfg.theta, adjust=cfg.adjust, buckets=cfg.init_edges,
                        kv_bytes_per_token=cfg.kvpt, current_safe=cfg.current_safe, device=torch.device("cuda", 0))
    for _ in range(5):
        r = s.schedule(lens, cls)
    raw = s.summary.cpu().numpy().view(np.int64)
    t = raw[18:26]
    print(name, n, "phase us:", [round((t[i+1]-t[i])/1000, 2) for i in range(7)], "total", (t[7]-t[0])/1000, r.summary()["n_batches"])
