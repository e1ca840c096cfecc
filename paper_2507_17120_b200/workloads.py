"""Synthetic windows for the five BASELINE.json configs (shared by tests, bench, golden).

Pure numpy; the generator is ours (the reference draws per-request in a Python
loop, workload.py:264-282) but follows the reference's distributions:
rounded, clamped to [1, cap] (workload.py:54-60); LongTailLogNormal
(workload.py:89-110); ShortNormal (:63-86); Mixture (:113-135).  Windows are
arrival-sorted, so the arrival rank is the index (workload.py:389-399).

Used by bench.py, the tests and oracle/gen_golden.py; it never touches oracle/.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

GIB = 2 ** 30

FCFS, SJF, LJF = 0, 1, 2
PADDED, EXACT = 0, 1


def kv_bytes_per_token(layers, heads, head_dim, bytes_per_elem):
    """ModelConfig.kv_bytes_per_token, memory_model.py:36-39."""
    return 2 * layers * heads * head_dim * bytes_per_elem


def safe_memory(total, model, reserve=0.10):
    """memory_model.py:194-197: floor((1 - r) * (total - model)) in float64."""
    return math.floor((1.0 - reserve) * (total - model))


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    l_max: int
    n_classes: int
    policies: tuple
    kvpt: int
    current_safe: int
    accounting: int = PADDED
    theta: float = 0.5
    adjust: bool = True
    init_edges: tuple | None = None
    dist: str = "lognormal"
    note: str = ""


# Llama-2-7B: 32 layers, 32 heads, 128 dim, fp16 -> 524,288 B/token (test_memory_model.py:157-159)
LLAMA2_7B = kv_bytes_per_token(32, 32, 128, 2)
# llama2-13b-like preset: 40/40/128/2 -> 819,200 B/token (memory_model.py:45-46)
LLAMA2_13B = kv_bytes_per_token(40, 40, 128, 2)
# Llama-3-8B GQA: 32 layers, 8 KV heads, 128 dim, fp16 -> 131,072 B/token
LLAMA3_8B = kv_bytes_per_token(32, 8, 128, 2)

CONFIGS = {
    # pkg/scenarios default: 1k uniform 32-2048, fixed buckets, 2 classes (PAPER.md:98 edges)
    "c1": Config("c1", 1_000, 4096, 2, (FCFS, SJF), LLAMA2_13B,
                 safe_memory(40 * GIB, 26 * GIB), adjust=False, init_edges=(0, 256, 1024, 4096),
                 dist="uniform", note="uniform 32-2048, fixed edges [0,256,1024,4096]"),
    # 1M ShareGPT-like lognormal, adaptive, Llama-2-7B on one B200 (180 GiB / 14 GiB weights)
    "c2": Config("c2", 1_000_000, 4096, 2, (FCFS, SJF), LLAMA2_7B,
                 safe_memory(180 * GIB, 14 * GIB), note="lognormal(5.5,1.1) cap 4095"),
    # 16M, 4 priority classes (class 0 FCFS, 1-3 SJF), bursty Poisson arrivals
    "c3": Config("c3", 16_000_000, 4096, 4, (FCFS, SJF, SJF, SJF), LLAMA2_7B,
                 safe_memory(180 * GIB, 14 * GIB), note="lognormal, 4 classes, bursty arrivals"),
    # long-context tail to 128k, Llama-3-8B on 180 GB, pack [B, L]
    "c4": Config("c4", 262_144, 131072, 2, (FCFS, SJF), LLAMA3_8B,
                 safe_memory(180 * 10 ** 9, 16 * 10 ** 9), dist="longctx",
                 note="0.7 N(83,40) + 0.3 lognormal(ln 41417, 1.0), cap 131071"),
    # 64M sharded over 2/4/8 GPUs (C2 distribution)
    "c5": Config("c5", 64_000_000, 4096, 2, (FCFS, SJF), LLAMA2_7B,
                 safe_memory(180 * GIB, 14 * GIB), note="C2 distribution, sharded"),
}


def gen_lengths(cfg: Config, n: int, rng: np.random.Generator) -> np.ndarray:
    cap = cfg.l_max - 1
    if cfg.dist == "uniform":
        return rng.integers(32, 2049, size=n).astype(np.int32)
    if cfg.dist == "lognormal":
        x = rng.lognormal(5.5, 1.1, size=n)
    elif cfg.dist == "longctx":
        comp = rng.random(n) < 0.7
        a = rng.normal(83.0, 40.0, size=n)
        b = rng.lognormal(math.log(41417.0), 1.0, size=n)
        x = np.where(comp, a, b)
    else:
        raise ValueError(cfg.dist)
    return np.clip(np.rint(x), 1, cap).astype(np.int32)


def gen_classes(cfg: Config, n: int, rng: np.random.Generator) -> np.ndarray:
    return rng.integers(0, cfg.n_classes, size=n).astype(np.uint8)


def gen_arrivals(cfg: Config, n: int, rng: np.random.Generator, rate: float = 1000.0):
    """Bursty Poisson arrivals (bursts of geometric size, exponential gaps).
    Sorted, so the scheduler's arrival rank is the index; kept for completeness."""
    if n == 0:
        return np.zeros(0)
    burst = rng.geometric(1 / 16.0, size=n)
    gaps = rng.exponential(1.0 / rate, size=n)
    starts = np.repeat(np.cumsum(gaps), burst)[:n]
    return np.sort(starts)


_HASH_MUL = 2654435761


def token_store(lens: np.ndarray, rng: np.random.Generator | None = None, vocab: int = 32000,
                align: int = 32, seed: int = 0):
    """CSR token store: row i starts at tok_off[i] (multiple of `align` tokens: with the
    default 32 every row starts on a 128-byte line, the TMA-friendly layout SURVEY §8f
    recommends; measured 790 vs 798 us for C2's pack against 16-byte alignment) and
    holds lens[i] synthetic ids.
    Token at global slot p is ((p * 2654435761 + seed) mod 2^32) mod vocab."""
    lens = np.asarray(lens, np.int64)
    pitch = (lens + align - 1) // align * align
    tok_off = np.zeros(len(lens) + 1, np.int64)
    np.cumsum(pitch, out=tok_off[1:])
    total = int(tok_off[-1])
    pos = np.arange(total, dtype=np.uint32)
    pos *= np.uint32(_HASH_MUL)
    pos += np.uint32(seed & 0xFFFFFFFF)
    pos %= np.uint32(vocab)
    return tok_off, pos.view(np.int32)


def token_store_device(lens, vocab: int = 32000, align: int = 32, seed: int = 0):
    """Same store as token_store(), generated on the GPU (torch tensors)."""
    import torch
    lens = lens.to(torch.int64)
    pitch = (lens + align - 1) // align * align
    tok_off = torch.zeros(lens.numel() + 1, dtype=torch.int64, device=lens.device)
    torch.cumsum(pitch, 0, out=tok_off[1:])
    total = int(tok_off[-1].item())
    tokens = torch.empty(total, dtype=torch.int32, device=lens.device)
    chunk = 1 << 28  # bounded int64 temporaries (C3's store holds ~7e9 slots)
    for a in range(0, total, chunk):
        b = min(total, a + chunk)
        pos = torch.arange(a, b, dtype=torch.int64, device=lens.device)
        tokens[a:b] = (((pos * _HASH_MUL + (seed & 0xFFFFFFFF)) & 0xFFFFFFFF) % vocab).to(torch.int32)
        del pos
    return tok_off, tokens


def make_window(name: str, n: int | None = None, seed: int = 1234, shard: tuple | None = None):
    """Returns (cfg, lens, cls).  shard=(rank, world) takes the contiguous
    arrival-order slice [r*N/P, (r+1)*N/P) of the full trace."""
    cfg = CONFIGS[name]
    n = cfg.n if n is None else n
    rng = np.random.default_rng(seed)
    lens = gen_lengths(cfg, n, rng)
    cls = gen_classes(cfg, n, rng)
    if shard is not None:
        r, w = shard
        a, b = r * n // w, (r + 1) * n // w
        lens, cls = lens[a:b].copy(), cls[a:b].copy()
    return cfg, lens, cls
