import numpy as np, torch, sys
sys.path.insert(0,'.')
from paper_2507_17120_b200 import workloads as W
from paper_2507_17120_b200.window import WindowScheduler
for name in ("c2","c4"):
    cfg, lens, cls = W.make_window(name, seed=1234)
    dev=torch.device("cuda",0)
    s = WindowScheduler(max_requests=len(lens), max_seq_len=cfg.l_max, n_classes=cfg.n_classes, policies=cfg.policies,
        split_threshold=cfg.theta, adjust=cfg.adjust, buckets=cfg.init_edges, kv_bytes_per_token=cfg.kvpt,
        current_safe=cfg.current_safe, accounting=cfg.accounting, device=dev)
    L=torch.as_tensor(lens).to(dev); C=torch.as_tensor(cls).to(dev)
    for _ in range(3): r=s.schedule(L,C)
    raw = s.summary.cpu().numpy().view(np.int64)[18:]
    t = raw[:5]
    print(name, "levels", raw[7], "phase us:", np.diff(t)/1000.0, "chain_blocks", s.ctx.ptr)
