"""Small windows through every stage (K1..K7, all pack paths: 128-byte, 16-byte and
unaligned token stores, long-context TMA pack, four classes), for compute-sanitizer:

    compute-sanitizer --tool memcheck  --error-exitcode 9 python tools/sanitize_window.py
    compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_window.py --small
    compute-sanitizer --tool memcheck  --error-exitcode 9 python tools/sanitize_window.py --paths
    compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_window.py --k0
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2507_17120_b200 import workloads as W  # noqa: E402
from paper_2507_17120_b200.window import WindowScheduler  # noqa: E402

cases = [("c2", 30000, 32), ("c2", 20000, 1), ("c4", 2000, 32), ("c3", 40000, 4)]
if "--paths" in sys.argv:
    # the rarer K5 paths: every chain longer than 2 calls through K5c's doubling CTAs, and
    # K5e's drain-order outcomes scattered in three request-id ranges
    os.environ["BS_CHAIN_WALK"] = "2"
    os.environ["BS_OUTCOME_PARTS"] = "3"
    cases = [("c2", 30000, 32), ("c3", 40000, 4)]
if "--small" in sys.argv:
    # + windows of <= 2048 requests, which take K0 (k_window_small)
    cases = [("c2", 3000, 32), ("c3", 3000, 1), ("c4", 300, 32), ("c1", 1000, 32), ("c2", 2000, 4)]
if "--k0" in sys.argv:
    # K0 (k_window_small) at the edges of its range: 2048 requests with l_max 8192
    # (largest shared-memory layout), eight classes, the exact accounting, tiny l_max
    import numpy as np
    rng = np.random.default_rng(5)
    for (n, L, C, pol, kvpt, budget, acc) in [
            (2048, 8192, 2, (0, 1), 2, 8192 * 40, 0), (2048, 2048, 8, (0, 1, 2, 1, 0, 2, 1, 1), 2, 2048 * 3, 1),
            (1500, 4096, 2, (1, 1), 2, 4096 * 200, 0), (2000, 100, 4, (2, 0, 1, 1), 6, 300, 0)]:
        lens = np.clip(rng.lognormal(np.log(L / 6), 1.2, n).astype(np.int32), 0, L - 1)
        cls = rng.integers(0, C, n).astype(np.uint8)
        tok_off, tokens = W.token_store(lens)
        s = WindowScheduler(max_requests=n, max_seq_len=L, n_classes=C, policies=pol,
                            kv_bytes_per_token=kvpt, current_safe=kvpt * budget, accounting=acc,
                            device=torch.device("cuda", 0))
        r = s.schedule(*(torch.as_tensor(a).cuda() for a in (lens, cls, tok_off, tokens)))
        assert s.ctx.launches <= 3  # K0 + the row copy
        print("k0", n, L, C, r.summary()["n_batches"])
        s.close()
    cases = []
for name, n, align in cases:
    cfg, lens, cls = W.make_window(name, n=n, seed=11)
    tok_off, tokens = W.token_store(lens, align=align)
    s = WindowScheduler(max_requests=n, max_seq_len=cfg.l_max, n_classes=cfg.n_classes,
                        policies=cfg.policies, kv_bytes_per_token=cfg.kvpt,
                        current_safe=cfg.current_safe, device=torch.device("cuda", 0),
                        dispatch=not (n <= 2048 and cfg.l_max <= 8192))  # K0 has no K7
    h = s.schedule(*(torch.as_tensor(a).cuda() for a in (lens, cls, tok_off, tokens))).to_host()
    assert int(h["summary"]["flags"]) == 0
    print(name, n, align, int(h["summary"]["n_batches"]))
    s.close()
