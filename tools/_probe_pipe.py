import sys, os, numpy as np, torch
sys.path.insert(0, '.')
from paper_2507_17120_b200 import workloads as W
from paper_2507_17120_b200.window import WindowScheduler
cfg, lens, cls = W.make_window("c2", seed=1234)
dev = torch.device("cuda", 0)
L = torch.as_tensor(lens).to(dev); C = torch.as_tensor(cls).to(dev)
tok_off, tokens = W.token_store_device(L)
mk = lambda: WindowScheduler(max_requests=len(lens), max_seq_len=cfg.l_max, n_classes=2, policies=cfg.policies,
                             kv_bytes_per_token=cfg.kvpt, current_safe=cfg.current_safe, device=dev)
streams = [torch.cuda.Stream() for _ in range(3)]
scheds = []
for k in range(3):
    with torch.cuda.stream(streams[k]):
        s = mk(); s.schedule(L, C, tok_off, tokens)
        for _ in range(3): s.schedule(L, C, tok_off, tokens, sync=False, check=False, graph=True)
        scheds.append(s)
torch.cuda.synchronize()
K = 100
res = []
for infl in (1, 2, 3):
    cur = torch.cuda.current_stream()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for st in streams: st.wait_stream(cur)
    for i in range(K):
        k = i % infl
        with torch.cuda.stream(streams[k]):
            scheds[k].schedule(L, C, tok_off, tokens, sync=False, check=False, graph=True)
    for st in streams: cur.wait_stream(st)
    e1.record(cur); torch.cuda.synchronize()
    res.append(round(e0.elapsed_time(e1) / K, 4))
print(os.environ.get("BS_PACK_VARIANT", "default"), "inflight 1/2/3 ms:", res)
