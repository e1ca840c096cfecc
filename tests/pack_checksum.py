"""Device-side checksum of a packed window (test infrastructure): the same
position-weighted sums mod 2^64 as oracle/bso.c:bso_pack_checksum, computed with torch
ops in bounded chunks on the GPU, so packed outputs of tens of GB (C3's 16M-request
window, C4's long-context window) are compared with the oracle without a host copy."""

import torch

from oracle.cpu import CK

M64 = (1 << 64) - 1


def _s64(v):
    return v - (1 << 64) if v >= 1 << 63 else v


def device_checksum(out_tokens, out_mask, m: int, chunk: int = 1 << 27):
    dev = out_tokens.device
    a1, b1, a2, b2 = (_s64(v) for v in CK)
    st = torch.zeros((), dtype=torch.int64, device=dev)
    sm = torch.zeros((), dtype=torch.int64, device=dev)
    for a in range(0, m, chunk):
        b = min(m, a + chunk)
        e = torch.arange(a, b, dtype=torch.int64, device=dev)
        st += (out_tokens[a:b].to(torch.int64) * (e * a1 + b1)).sum()
        sm += (out_mask[a:b].to(torch.int64) * (e * a2 + b2)).sum()
        del e
    return int(st.item()) & M64, int(sm.item()) & M64
