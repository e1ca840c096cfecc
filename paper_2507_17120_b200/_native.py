"""ctypes binding of the C-ABI library (include/bucketserve.h).

The product path has exactly one implementation: the sm_100a kernels in
_lib/libbucketserve.so.  There is no CPU fallback — if the library or a B200 is
missing, every entry point raises (NativeUnavailable).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import ConfigError, SimulationError

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "_lib", "libbucketserve.so")

BS_OK = 0
BS_ERR_INVALID_ARG = -1
BS_ERR_CONFIG = -2
BS_ERR_CUDA = -3
BS_ERR_CAPACITY = -4
BS_ERR_NOT_BUILT = -5

FLAG_LEN_RANGE = 0x1
FLAG_CLASS_RANGE = 0x2
FLAG_ZERO_MEAN = 0x4
FLAG_CHANGES_TRUNC = 0x8
FLAG_PACK_CAPACITY = 0x10
FLAG_NONPOS_LEN = 0x20
FLAG_BATCH_CAP = 0x40
FLAG_BAD_EDGES = 0x80
FLAG_DISPATCH_RANGE = 0x100
FLAG_PEER_TIMEOUT = 0x200
PEER_HANDLE_BYTES = 64
NCCL_ID_BYTES = 128

POLICY_FCFS, POLICY_SJF, POLICY_LJF = 0, 1, 2
ACCOUNTING_PADDED, ACCOUNTING_EXACT = 0, 1
CHANGE_SPLIT, CHANGE_MERGE, CHANGE_SKIP = 1, 2, 3
REQ_PENDING, REQ_REJECTED = -1, -2
MAX_CLASSES = 8
PACK_ALIGN = 16

EXPORTS = ("bs_abi_version", "bs_last_error", "bs_scratch_bytes", "bs_create", "bs_destroy",
           "bs_histogram", "bs_boundaries", "bs_assign", "bs_order", "bs_size", "bs_pack",
           "bs_window_schedule", "bs_window_from_hist", "bs_monitor_bins", "bs_monitor",
           "bs_profile_enable",
           "bs_profile_read", "bs_launch_count", "bs_dispatch", "bs_trace_parse",
           "bs_trace_write_bst", "bs_trace_read_bst", "bs_peer_export", "bs_peer_connect",
           "bs_peer_reduce", "bs_nccl_unique_id", "bs_nccl_connect", "bs_set_nccl",
           "bs_nccl_allreduce")
STAGES = ("histogram", "exchange", "boundaries", "order", "size.prep", "size.next", "size.chain",
          "size.describe", "size.outcome", "dispatch", "pack")


class NativeUnavailable(RuntimeError):
    """The CUDA library or a B200 (sm_100) device is not available."""


class WindowParams(C.Structure):
    _fields_ = [("l_max", C.c_int32), ("n_classes", C.c_int32), ("policy", C.c_int32 * 8),
                ("split_threshold", C.c_double), ("adjust", C.c_int32), ("max_passes", C.c_int32),
                ("n_max", C.c_int64), ("kv_bytes_per_token", C.c_int64),
                ("current_safe", C.c_int64), ("pledged", C.c_int64), ("accounting", C.c_int32),
                ("truncate", C.c_int32), ("pad_id", C.c_int32), ("dispatch", C.c_int32)]


class WindowIO(C.Structure):
    _fields_ = [("len", C.c_void_p), ("cls", C.c_void_p), ("tok_off", C.c_void_p),
                ("tokens", C.c_void_p), ("n", C.c_int64), ("init_edges", C.c_void_p),
                ("k_init", C.c_int32), ("changes_cap", C.c_int32), ("batches_cap", C.c_int32),
                ("reserved0", C.c_int32), ("out_capacity", C.c_int64), ("hist", C.c_void_p),
                ("hist_global", C.c_void_p), ("edges", C.c_void_p), ("changes", C.c_void_p),
                ("bucket", C.c_void_p), ("perm", C.c_void_p), ("seg_off", C.c_void_p),
                ("batches", C.c_void_p), ("req_batch", C.c_void_p), ("req_row", C.c_void_p),
                ("out_tokens", C.c_void_p), ("out_mask", C.c_void_p), ("summary", C.c_void_p),
                ("emit_order", C.c_void_p), ("batch_emit", C.c_void_p)]


BATCH_DTYPE = np.dtype([("segment", "<i4"), ("start", "<i4"), ("end", "<i4"), ("n", "<i4"),
                        ("max_input_len", "<i4"), ("pitch", "<i4"), ("token_sum", "<i8"),
                        ("footprint", "<i8"), ("out_offset", "<i8"), ("waste", "<f8"),
                        ("row_base", "<i8")])
SUMMARY_FIELDS = ("n_requests", "total_global", "sum_len_global", "n_max", "k_buckets",
                  "n_changes", "n_passes", "n_batches", "n_rejected", "n_pending",
                  "admitted_tokens", "padded_tokens", "packed_elems", "peak_footprint",
                  "waste_sum", "sort_passes", "flags", "n_dispatched")
SUMMARY_DTYPE = np.dtype([(f, "<f8" if f == "waste_sum" else "<i8") for f in SUMMARY_FIELDS] +
                         [("reserved", "<i8", (14,))])
assert BATCH_DTYPE.itemsize == 64 and SUMMARY_DTYPE.itemsize == 256

_lib = None


def lib_path() -> str:
    return LIB_PATH


def load():
    """Load libbucketserve.so (raises NativeUnavailable when absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(
            f"{LIB_PATH} is missing: run `python -m paper_2507_17120_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    P = C.POINTER(WindowParams)
    sig = {
        "bs_abi_version": (C.c_int, []),
        "bs_last_error": (C.c_char_p, [vp]),
        "bs_scratch_bytes": (i64, [vp]),
        "bs_create": (C.c_int, [C.POINTER(vp), C.c_int, i64, i32, i32]),
        "bs_destroy": (C.c_int, [vp]),
        "bs_histogram": (C.c_int, [vp, vp, vp, i64, P, vp, vp, vp]),
        "bs_boundaries": (C.c_int, [vp, vp, vp, P, vp, i32, vp, vp, i32, vp, vp]),
        "bs_assign": (C.c_int, [vp, vp, i64, P, vp, vp]),
        "bs_order": (C.c_int, [vp, vp, vp, i64, P, vp, vp, vp, vp, vp]),
        "bs_size": (C.c_int, [vp, vp, vp, vp, i64, P, vp, i32, vp, vp, vp, vp]),
        "bs_pack": (C.c_int, [vp, vp, vp, vp, vp, P, vp, i64, i64, vp, vp, i64, vp, vp]),
        "bs_window_schedule": (C.c_int, [vp, C.POINTER(WindowIO), P, vp]),
        "bs_window_from_hist": (C.c_int, [vp, C.POINTER(WindowIO), P, vp]),
        "bs_monitor_bins": (C.c_int, [vp, vp, P, i32, vp, vp]),
        "bs_monitor": (C.c_int, [vp, vp, P, i32, vp, i32, vp, vp, vp]),
        "bs_profile_enable": (C.c_int, [vp, i32]),
        "bs_profile_read": (C.c_int, [vp, C.POINTER(C.c_float), C.POINTER(i32)]),
        "bs_launch_count": (i64, [vp]),
        "bs_dispatch": (C.c_int, [vp, vp, vp, i64, P, vp, i32, vp, vp, vp, vp, vp, vp]),
        "bs_peer_export": (C.c_int, [vp, vp]),
        "bs_peer_connect": (C.c_int, [vp, i32, i32, vp]),
        "bs_peer_reduce": (C.c_int, [vp, vp, P, vp, vp, vp]),
        "bs_nccl_unique_id": (C.c_int, [vp]),
        "bs_nccl_connect": (C.c_int, [vp, i32, i32, vp]),
        "bs_set_nccl": (C.c_int, [vp, vp, i32, i32]),
        "bs_nccl_allreduce": (C.c_int, [vp, vp, P, vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, ctx=None):
    """Map a BS_* status to the reference's exception taxonomy (errors.py)."""
    if rc == BS_OK:
        return
    msg = (_lib.bs_last_error(ctx) or b"").decode(errors="replace") if _lib else ""
    if rc in (BS_ERR_INVALID_ARG, BS_ERR_CAPACITY):
        raise ValueError(msg or f"bucketserve status {rc}")
    if rc == BS_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == BS_ERR_NOT_BUILT:
        raise NativeUnavailable(msg)
    raise SimulationError(f"CUDA failure in bucketserve: {msg}")


def raise_for_flags(flags: int, l_max: int | None = None):
    """Device-latched data errors -> the exception the reference raises."""
    if flags & FLAG_LEN_RANGE:
        raise ValueError(f"input_len outside [0, {l_max}); truncation should have been applied")
    if flags & FLAG_CLASS_RANGE:
        raise ValueError("task class id outside [0, n_classes)")
    if flags & FLAG_BAD_EDGES:
        raise ValueError("initial bucket edges must increase strictly from 0 to max_seq_len")
    if flags & FLAG_ZERO_MEAN:
        raise ZeroDivisionError("float floor division by zero (mean queued length is 0)")
    if flags & FLAG_BATCH_CAP:
        raise SimulationError("batch descriptor capacity exceeded")
    if flags & FLAG_PACK_CAPACITY:
        raise ValueError("packed output buffer too small")
    if flags & FLAG_PEER_TIMEOUT:
        raise SimulationError("a peer rank's histogram did not arrive (peer-memory C1 timeout)")
    if flags & FLAG_DISPATCH_RANGE:
        raise ValueError("dispatch order: queued token mass or bucket count out of range")


def make_params(*, l_max, n_classes, policies, split_threshold, adjust, max_passes, n_max,
                kv_bytes_per_token, current_safe, pledged, accounting, truncate, pad_id,
                dispatch=False):
    p = WindowParams()
    p.l_max, p.n_classes = int(l_max), int(n_classes)
    for i, v in enumerate(policies):
        p.policy[i] = int(v)
    p.split_threshold = float(split_threshold)
    p.adjust, p.max_passes = int(bool(adjust)), int(max_passes)
    p.n_max = int(n_max or 0)
    p.kv_bytes_per_token = int(kv_bytes_per_token)
    p.current_safe, p.pledged = int(current_safe), int(pledged)
    p.accounting, p.truncate, p.pad_id = int(accounting), int(bool(truncate)), int(pad_id)
    p.dispatch = int(bool(dispatch))
    return p


class Context:
    """Owns one bs_ctx (scratch for windows up to max_n requests on a device)."""

    def __init__(self, device: int, max_n: int, l_max_cap: int, max_classes: int):
        self._lib = load()
        self.ptr = C.c_void_p()
        rc = self._lib.bs_create(C.byref(self.ptr), int(device), int(max_n), int(l_max_cap),
                                 int(max_classes))
        check(rc, None)
        self.device, self.max_n, self.l_max_cap, self.max_classes = device, max_n, l_max_cap, max_classes

    @property
    def scratch_bytes(self) -> int:
        return int(self._lib.bs_scratch_bytes(self.ptr))

    @property
    def launches(self) -> int:
        """Kernels launched through this context so far."""
        return int(self._lib.bs_launch_count(self.ptr))

    def profile_enable(self, max_steps: int):
        check(self._lib.bs_profile_enable(self.ptr, int(max_steps)), self.ptr)

    def profile_read(self) -> tuple[dict, int]:
        """(summed ms per stage, steps) of the profiled fused calls since the last read."""
        ms = (C.c_float * len(STAGES))()
        steps = C.c_int32(0)
        check(self._lib.bs_profile_read(self.ptr, ms, C.byref(steps)), self.ptr)
        return {k: float(ms[i]) for i, k in enumerate(STAGES)}, int(steps.value)

    def close(self):
        if self.ptr:
            self._lib.bs_destroy(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
