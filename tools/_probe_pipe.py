import sys, os, ctypes as Cc, numpy as np, torch
sys.path.insert(0, '.')
from paper_2507_17120_b200 import workloads as W, _native as N
from paper_2507_17120_b200.window import WindowScheduler, _ptr
cfg, lens, cls = W.make_window("c2", seed=1234)
dev = torch.device("cuda", 0)
L = torch.as_tensor(lens).to(dev); C = torch.as_tensor(cls).to(dev)
tok_off, tokens = W.token_store_device(L)
lib = N.load()
mk = lambda: WindowScheduler(max_requests=len(lens), max_seq_len=cfg.l_max, n_classes=2, policies=cfg.policies,
                             kv_bytes_per_token=cfg.kvpt, current_safe=cfg.current_safe, device=dev)
S = [torch.cuda.Stream(priority=-1), torch.cuda.Stream(priority=-1)]
P = [torch.cuda.Stream(priority=0), torch.cuda.Stream(priority=0)]
scheds = []
for k in range(2):
    s = mk(); s.schedule(L, C, tok_off, tokens); scheds.append(s)
torch.cuda.synchronize()

def window(k, split):
    s = scheds[k]
    if not split:
        with torch.cuda.stream(S[k]):
            S[k].wait_stream(P[k])
            s.schedule(L, C, tok_off, tokens, sync=False, check=False)
        return
    with torch.cuda.stream(S[k]):
        S[k].wait_stream(P[k])
        s.schedule(L, C, sync=False, check=False)
    P[k].wait_stream(S[k])
    N.check(lib.bs_pack(s.ctx.ptr, _ptr(L), _ptr(s.perm), _ptr(tok_off), _ptr(tokens), Cc.byref(s._params),
                        _ptr(s.batches_raw), 0, -1, _ptr(s.out_tokens), _ptr(s.out_mask), s.pack_capacity,
                        _ptr(s.summary), Cc.c_void_p(P[k].cuda_stream)), s.ctx.ptr)

K = 100
out = []
for mode in ("serial", "pipe2", "pipe2_split"):
    for _ in range(4): window(0, False)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    e0.record(cur)
    for st in S + P: st.wait_stream(cur)
    for i in range(K):
        k = 0 if mode == "serial" else i % 2
        window(k, mode == "pipe2_split")
    for st in S + P: cur.wait_stream(st)
    e1.record(cur); torch.cuda.synchronize()
    out.append(round(e0.elapsed_time(e1) / K, 4))
print(os.environ.get("BS_PACK_VARIANT", "default"), "serial/pipe2/pipe2_split ms:", out)
