"""ctypes wrapper over oracle/bso.c (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py)."""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libbso.so")

FCFS, SJF, LJF = 0, 1, 2
PADDED, EXACT = 0, 1
REQ_PENDING, REQ_REJECTED = -1, -2


class Params(C.Structure):
    _fields_ = [("l_max", C.c_int32), ("n_classes", C.c_int32), ("policy", C.c_int32 * 8),
                ("theta", C.c_double), ("adjust", C.c_int32), ("max_passes", C.c_int32),
                ("n_max", C.c_int64), ("kvpt", C.c_int64), ("current_safe", C.c_int64),
                ("pledged", C.c_int64), ("accounting", C.c_int32), ("truncate", C.c_int32),
                ("pad_id", C.c_int32), ("reserved", C.c_int32)]


class Summary(C.Structure):
    _fields_ = [(k, C.c_int64) for k in (
        "n_requests", "total_global", "sum_len_global", "n_max", "k_buckets", "n_changes",
        "n_passes", "n_batches", "n_rejected", "n_pending", "admitted_tokens",
        "padded_tokens", "packed_elems", "peak_footprint")] + [
        ("waste_sum", C.c_double), ("sort_passes", C.c_int64), ("flags", C.c_int64),
        ("reserved", C.c_int64 * 15)]


BATCH_DTYPE = np.dtype([("segment", "<i4"), ("start", "<i4"), ("end", "<i4"), ("n", "<i4"),
                        ("max_input_len", "<i4"), ("pitch", "<i4"), ("token_sum", "<i8"),
                        ("footprint", "<i8"), ("out_offset", "<i8"), ("waste", "<f8"),
                        ("row_base", "<i8")])
assert BATCH_DTYPE.itemsize == 64


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH) or \
            os.path.getmtime(LIB_PATH) < os.path.getmtime(os.path.join(HERE, "bso.c")):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.bso_n_max.restype = C.c_int64
        _lib.bso_n_max.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_int64,
                                   C.POINTER(C.c_int64)]
        _lib.bso_num_threads.restype = C.c_int
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


@dataclass
class WindowSpec:
    """Scheduling parameters of one window (mirrors bs_window_params)."""
    l_max: int
    n_classes: int = 2
    policies: tuple = (FCFS, SJF)
    theta: float = 0.5
    adjust: bool = True
    max_passes: int = 0
    n_max: int = 0
    kvpt: int = 1
    current_safe: int = 0
    pledged: int = 0
    accounting: int = PADDED
    truncate: bool = True
    pad_id: int = 0
    init_edges: tuple | None = None

    def params(self) -> Params:
        p = Params()
        p.l_max, p.n_classes = self.l_max, self.n_classes
        for i, v in enumerate(self.policies):
            p.policy[i] = int(v)
        p.theta, p.adjust, p.max_passes = self.theta, int(self.adjust), self.max_passes
        p.n_max, p.kvpt, p.current_safe, p.pledged = self.n_max, self.kvpt, self.current_safe, self.pledged
        p.accounting, p.truncate, p.pad_id = int(self.accounting), int(self.truncate), self.pad_id
        return p


@dataclass
class WindowResult:
    hist: np.ndarray
    edges: np.ndarray
    changes: np.ndarray
    perm: np.ndarray
    seg_off: np.ndarray
    bucket: np.ndarray
    batches: np.ndarray
    req_batch: np.ndarray
    req_row: np.ndarray
    summary: dict
    out_tokens: np.ndarray | None = None
    out_mask: np.ndarray | None = None
    extra: dict = field(default_factory=dict)


def window(spec: WindowSpec, lens, cls, tok_off=None, tokens=None, threads: int = 0,
           out_capacity: int | None = None) -> WindowResult:
    """Run the whole window on the CPU restatement."""
    L = lib()
    if threads:
        L.bso_set_threads(int(threads))
    lens = np.ascontiguousarray(lens, dtype=np.int32)
    cls = np.ascontiguousarray(cls, dtype=np.uint8)
    n = len(lens)
    p = spec.params()
    hist = np.zeros(spec.n_classes * spec.l_max, np.uint32)
    edges = np.zeros(spec.l_max + 1, np.int32)
    k = C.c_int32(0)
    cap = 4 * spec.l_max + 64
    changes = np.zeros((cap, 4), np.int32)
    perm = np.zeros(max(n, 1), np.int32)
    seg_off = np.zeros(spec.l_max * spec.n_classes + 1, np.int32)
    bcap = max(n, 1)
    batches = np.zeros(bcap, BATCH_DTYPE)
    req_batch = np.zeros(max(n, 1), np.int32)
    req_row = np.zeros(max(n, 1), np.int32)
    init = None
    kinit = 0
    if spec.init_edges is not None:
        init = np.ascontiguousarray(spec.init_edges, dtype=np.int32)
        kinit = len(init) - 1
    pack = tok_off is not None and tokens is not None
    out_tokens = out_mask = None
    if pack:
        tok_off = np.ascontiguousarray(tok_off, dtype=np.int64)
        tokens = np.ascontiguousarray(tokens, dtype=np.int32)
        if out_capacity is None:
            out_capacity = 0  # two-phase: size first
    s = Summary()
    if pack and out_capacity == 0:
        # size-only pass to learn the packed extent, then pack
        rc = L.bso_window(_ptr(lens), _ptr(cls), C.c_int64(n), None, None, C.byref(p),
                          _ptr(init), C.c_int32(kinit), _ptr(hist), _ptr(edges), C.byref(k),
                          _ptr(changes), C.c_int32(cap), _ptr(perm), _ptr(seg_off),
                          _ptr(batches), C.c_int64(bcap), _ptr(req_batch), _ptr(req_row),
                          None, None, C.c_int64(0), C.byref(s))
        if rc != 0:
            raise ValueError("malformed init edges")
        out_capacity = int(s.packed_elems)
    if pack:
        out_tokens = np.zeros(max(out_capacity, 1), np.int32)
        out_mask = np.zeros(max(out_capacity, 1), np.uint8)
    rc = L.bso_window(_ptr(lens), _ptr(cls), C.c_int64(n), _ptr(tok_off) if pack else None,
                      _ptr(tokens) if pack else None, C.byref(p), _ptr(init), C.c_int32(kinit),
                      _ptr(hist), _ptr(edges), C.byref(k), _ptr(changes), C.c_int32(cap),
                      _ptr(perm), _ptr(seg_off), _ptr(batches), C.c_int64(bcap),
                      _ptr(req_batch), _ptr(req_row), _ptr(out_tokens), _ptr(out_mask),
                      C.c_int64(out_capacity or 0), C.byref(s))
    if rc != 0:
        raise ValueError("malformed init edges")
    K = k.value
    summary = {f: getattr(s, f) for f, _ in Summary._fields_ if f != "reserved"}
    nb = int(summary["n_batches"])
    bucket = np.zeros(max(n, 1), np.int32)
    fl = C.c_int64(0)
    L.bso_assign(_ptr(lens), C.c_int64(n), C.byref(p), _ptr(edges), C.c_int32(K), _ptr(bucket),
                 C.byref(fl))
    return WindowResult(hist=hist.reshape(spec.n_classes, spec.l_max), edges=edges[:K + 1].copy(),
                        changes=changes[:min(int(summary["n_changes"]), cap)].copy(),
                        perm=perm[:n].copy(), seg_off=seg_off[:K * spec.n_classes + 1].copy(),
                        bucket=bucket[:n].copy(), batches=batches[:nb].copy(),
                        req_batch=req_batch[:n].copy(), req_row=req_row[:n].copy(),
                        summary=summary, out_tokens=out_tokens, out_mask=out_mask)


def boundaries(spec: WindowSpec, hist) -> tuple[np.ndarray, np.ndarray, dict]:
    """K2 alone on a given (global) per-(class, length) histogram: (edges, change log,
    summary) of bso_boundaries (BucketSet.adjust_buckets to the fixpoint on the counts;
    n_max from the histogram's moments unless spec.n_max is set)."""
    L = lib()
    h = np.ascontiguousarray(np.asarray(hist).reshape(-1), dtype=np.uint32)
    p = spec.params()
    edges = np.zeros(spec.l_max + 1, np.int32)
    k = C.c_int32(0)
    cap = 4 * spec.l_max + 64
    changes = np.zeros((cap, 4), np.int32)
    init = None if spec.init_edges is None else np.ascontiguousarray(spec.init_edges, np.int32)
    s = Summary()
    rc = L.bso_boundaries(_ptr(h), C.byref(p), _ptr(init), C.c_int32(0 if init is None else len(init) - 1),
                          _ptr(edges), C.byref(k), _ptr(changes), C.c_int32(cap), C.byref(s))
    if rc != 0:
        raise ValueError("malformed init edges")
    summary = {f: getattr(s, f) for f, _ in Summary._fields_ if f != "reserved"}
    return edges[:k.value + 1].copy(), changes[:min(int(s.n_changes), cap)].copy(), summary


CK = (0x9E3779B97F4A7C15, 0x632BE59BD9B4E019, 0xD6E8FEB86659FD93, 0xA0761D6478BD642F)
HASH_MUL = 2654435761


def pack_checksum(spec: WindowSpec, lens, res: WindowResult, tok_off, tokens=None,
                  seed: int = 0, vocab: int = 32000) -> tuple[int, int]:
    """(token sum, mask sum) of the window's packed output (bso_pack_checksum) from the
    oracle's own plan, without materialising it; tokens=None regenerates the synthetic
    store's ids from its hash (workloads.token_store)."""
    L = lib()
    lens = np.ascontiguousarray(lens, dtype=np.int32)
    p = spec.params()
    out = np.zeros(2, np.uint64)
    tok_off = np.ascontiguousarray(tok_off, dtype=np.int64)
    tk = None if tokens is None else np.ascontiguousarray(tokens, dtype=np.int32)
    b = np.ascontiguousarray(res.batches)
    L.bso_pack_checksum(_ptr(lens), _ptr(res.perm), _ptr(res.req_batch), _ptr(res.req_row),
                        _ptr(tok_off), _ptr(tk), C.c_uint32(HASH_MUL), C.c_uint32(seed & 0xFFFFFFFF),
                        C.c_uint32(vocab), C.byref(p), _ptr(b), C.c_int64(len(b)), _ptr(out))
    return int(out[0]), int(out[1])


def checksum_arrays(out_tokens, out_mask, m: int) -> tuple[int, int]:
    """The same checksum over materialised packed arrays (numpy, for cross-checks)."""
    e = np.arange(m, dtype=np.uint64)
    with np.errstate(over="ignore"):
        w1 = e * np.uint64(CK[0]) + np.uint64(CK[1])
        w2 = e * np.uint64(CK[2]) + np.uint64(CK[3])
        st = np.sum(out_tokens[:m].astype(np.uint32).astype(np.uint64) * w1, dtype=np.uint64)
        sm = np.sum(out_mask[:m].astype(np.uint64) * w2, dtype=np.uint64)
    return int(st), int(sm)


def n_max(total: int, sum_len: int, current_safe: int, kvpt: int) -> int:
    fl = C.c_int64(0)
    return int(lib().bso_n_max(total, sum_len, current_safe, kvpt, C.byref(fl)))


def monitor_bins(hist: np.ndarray, l_max: int, bins: int = 64) -> np.ndarray:
    h = np.ascontiguousarray(hist, dtype=np.uint32).reshape(-1)
    p = Params()
    p.l_max, p.n_classes = l_max, h.size // l_max
    out = np.zeros(bins, np.uint64)
    lib().bso_monitor_bins(_ptr(h), C.byref(p), C.c_int32(bins), _ptr(out))
    return out


@dataclass
class DispatchResult:
    emit_order: np.ndarray   # batch index of the t-th plan
    batch_emit: np.ndarray   # t of batch b, or -1
    req_batch: np.ndarray    # dispatch outcome per request
    req_row: np.ndarray
    n_emitted: int
    n_rejected: int
    n_pending: int


def dispatch(spec: WindowSpec, lens, res: WindowResult) -> DispatchResult:
    """f3: the simulator's global dispatch sequence over a window result
    (bso_dispatch; Simulator._next_plan repeated, pd_sim.py:448-462)."""
    L = lib()
    L.bso_dispatch.restype = C.c_int64
    lens = np.ascontiguousarray(lens, dtype=np.int32)
    n = len(lens)
    p = spec.params()
    nb = len(res.batches)
    batches = np.ascontiguousarray(res.batches)
    rb = res.req_batch.copy()
    rr = res.req_row.copy()
    emit = np.full(max(nb, 1), -1, np.int32)
    bemit = np.full(max(nb, 1), -1, np.int32)
    s = Summary()
    t = L.bso_dispatch(_ptr(lens), _ptr(res.perm), _ptr(res.seg_off),
                       C.c_int64(len(res.seg_off) - 1), C.c_int64(n), C.byref(p), _ptr(batches),
                       C.c_int64(nb), _ptr(rb), _ptr(rr), _ptr(emit), _ptr(bemit), C.byref(s))
    return DispatchResult(emit_order=emit[:t].copy(), batch_emit=bemit[:nb].copy(), req_batch=rb,
                          req_row=rr, n_emitted=int(t), n_rejected=int(s.n_rejected),
                          n_pending=int(s.n_pending))
