"""Trace ingestion for the window path.

`load_trace(stream, fmt)` / `load_trace_path(path)` keep the reference's signatures
and semantics (bucketsim/workload.py:343-437) but parse with the native
multi-threaded parser in the C-ABI library (`bs_trace_parse`) into structure-of-
arrays (`TraceArrays`) instead of a list of Python objects: records in arrival order
(stable sort, ids = file order), the reference's validation, and TraceFormatError
with the reference's line number and text on the first malformed record.
`TraceArrays.window()` gives the (lengths, classes) a WindowScheduler consumes;
`TraceArrays.requests()` materialises reference-shaped `Request` objects.

`save_binary` / `load_binary` use the .bst SoA format (bs_trace_write_bst /
bs_trace_read_bst) for reloading 64M-request traces without re-parsing text.
The parser is host code: no GPU is needed.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from enum import Enum
from pathlib import Path

import numpy as np

from . import _native as N
from .errors import ConfigError, TraceFormatError
from .types import Request, TaskClass


class TraceFormat(Enum):
    """workload.py:321-323."""
    CSV = "csv"
    JSONL = "jsonl"


class _Trace(C.Structure):
    _fields_ = [("n", C.c_int64), ("id", C.POINTER(C.c_int64)), ("arrival", C.POINTER(C.c_double)),
                ("input_len", C.POINTER(C.c_int64)), ("output_len", C.POINTER(C.c_int64)),
                ("cls", C.POINTER(C.c_uint8)), ("err_line", C.c_int64),
                ("err_msg", C.c_char * 256)]


_bound = False


def _lib():
    global _bound
    lib = N.load()
    if not _bound:
        P = C.POINTER(_Trace)
        lib.bs_trace_parse.restype = C.c_int
        lib.bs_trace_parse.argtypes = [C.c_char_p, C.c_int64, C.c_int32, C.c_int32, P]
        lib.bs_trace_free.restype = None
        lib.bs_trace_free.argtypes = [P]
        lib.bs_trace_write_bst.restype = C.c_int
        lib.bs_trace_write_bst.argtypes = [C.c_char_p, P]
        lib.bs_trace_read_bst.restype = C.c_int
        lib.bs_trace_read_bst.argtypes = [C.c_char_p, P]
        _bound = True
    return lib


@dataclass
class TraceArrays:
    """A parsed trace as structure of arrays, ordered by arrival (workload.py:215-237)."""
    id: np.ndarray          # int64, file order
    arrival: np.ndarray     # float64, non-decreasing
    input_len: np.ndarray   # int64 >= 1
    output_len: np.ndarray  # int64, -1 where the record omitted it (None)
    cls: np.ndarray         # uint8, 0 online / 1 offline

    def __len__(self) -> int:
        return len(self.id)

    def window(self, max_seq_len: int | None = None):
        """(lengths int32, classes uint8) in arrival order for WindowScheduler.schedule;
        lengths >= max_seq_len are truncated to max_seq_len - 1 as the simulator does
        (pd_sim.py:382-383)."""
        lens = self.input_len
        if max_seq_len is not None:
            lens = np.minimum(lens, max_seq_len - 1)
        return lens.astype(np.int32), self.cls.copy()

    def requests(self) -> list:
        """Reference-shaped Request objects (workload.py:30-51)."""
        classes = (TaskClass.ONLINE, TaskClass.OFFLINE)
        return [Request(int(i), float(a), int(x), None if o < 0 else int(o), classes[int(c)])
                for i, a, x, o, c in zip(self.id, self.arrival, self.input_len, self.output_len,
                                         self.cls)]

    def validate(self) -> None:
        """Trace.validate (workload.py:226-237)."""
        if len(self.arrival) and np.any(np.diff(self.arrival) < 0):
            raise ConfigError("trace arrival times must be non-decreasing")
        if len(np.unique(self.id)) != len(self.id):
            raise ConfigError("duplicate request id")


def _take(t: _Trace) -> TraceArrays:
    n = int(t.n)

    def arr(p, dt):
        return np.ctypeslib.as_array(p, shape=(n,)).astype(dt, copy=True) if n else np.zeros(0, dt)

    return TraceArrays(id=arr(t.id, np.int64), arrival=arr(t.arrival, np.float64),
                       input_len=arr(t.input_len, np.int64), output_len=arr(t.output_len, np.int64),
                       cls=arr(t.cls, np.uint8))


def parse_trace(data: bytes | str, fmt: TraceFormat, threads: int = 0) -> TraceArrays:
    """Parse trace text (CSV or JSON lines) with the native parser."""
    if isinstance(data, str):
        data = data.encode("utf-8")
    fmt = TraceFormat(fmt)
    lib = _lib()
    t = _Trace()
    rc = lib.bs_trace_parse(data, len(data), 0 if fmt is TraceFormat.CSV else 1, int(threads),
                            C.byref(t))
    try:
        if rc == N.BS_ERR_CONFIG and t.err_line >= 0:
            msg = t.err_msg.decode("utf-8", errors="replace")
            prefix = f"line {int(t.err_line)}: "
            raise TraceFormatError(int(t.err_line), msg[len(prefix):] if msg.startswith(prefix) else msg)
        N.check(rc)
        return _take(t)
    finally:
        lib.bs_trace_free(C.byref(t))


def load_trace(stream, fmt: TraceFormat) -> TraceArrays:
    """workload.py:422-431 (stream: a text or binary file object, or str / bytes)."""
    data = stream if isinstance(stream, (str, bytes)) else stream.read()
    return parse_trace(data, fmt)


def format_for_path(path) -> TraceFormat:
    """workload.py:434-441."""
    suffix = Path(path).suffix.lower()
    if suffix == ".csv":
        return TraceFormat.CSV
    if suffix == ".jsonl":
        return TraceFormat.JSONL
    raise ConfigError(f"cannot infer trace format from extension {suffix!r} (use .csv or .jsonl)")


def load_trace_path(path, threads: int = 0) -> TraceArrays:
    """workload.py:444-447; .bst files load through load_binary."""
    if Path(path).suffix.lower() == ".bst":
        return load_binary(path)
    fmt = format_for_path(path)
    with open(path, "rb") as fh:
        return parse_trace(fh.read(), fmt, threads)


def save_binary(trace: TraceArrays, path) -> None:
    """Write the .bst SoA format."""
    t = _Trace()
    n = len(trace)
    keep = [np.ascontiguousarray(trace.id, np.int64), np.ascontiguousarray(trace.arrival, np.float64),
            np.ascontiguousarray(trace.input_len, np.int64),
            np.ascontiguousarray(trace.output_len, np.int64), np.ascontiguousarray(trace.cls, np.uint8)]
    t.n = n
    t.id = keep[0].ctypes.data_as(C.POINTER(C.c_int64))
    t.arrival = keep[1].ctypes.data_as(C.POINTER(C.c_double))
    t.input_len = keep[2].ctypes.data_as(C.POINTER(C.c_int64))
    t.output_len = keep[3].ctypes.data_as(C.POINTER(C.c_int64))
    t.cls = keep[4].ctypes.data_as(C.POINTER(C.c_uint8))
    N.check(_lib().bs_trace_write_bst(os.fsencode(str(path)), C.byref(t)))


def load_binary(path) -> TraceArrays:
    """Read the .bst SoA format."""
    lib = _lib()
    t = _Trace()
    rc = lib.bs_trace_read_bst(os.fsencode(str(path)), C.byref(t))
    try:
        if rc != N.BS_OK:
            raise ConfigError(f"{path}: not a readable .bst trace")
        return _take(t)
    finally:
        lib.bs_trace_free(C.byref(t))


def save_trace(trace: TraceArrays, stream, fmt: TraceFormat) -> None:
    """workload.py:450-466 (writes the reference's text formats)."""
    fmt = TraceFormat(fmt)
    cls_name = ("online", "offline")
    if fmt is TraceFormat.CSV:
        stream.write("arrival_s,input_tokens,output_tokens,class\n")
        for a, x, o, c in zip(trace.arrival.tolist(), trace.input_len.tolist(),
                              trace.output_len.tolist(), trace.cls.tolist()):
            stream.write(f"{a!r},{x},{'' if o < 0 else o},{cls_name[c]}\n")
    else:
        import json
        for a, x, o, c in zip(trace.arrival.tolist(), trace.input_len.tolist(),
                              trace.output_len.tolist(), trace.cls.tolist()):
            obj = {"arrival_s": a, "input_tokens": x}
            if o >= 0:
                obj["output_tokens"] = o
            obj["class"] = cls_name[c]
            stream.write(json.dumps(obj) + "\n")


__all__ = ["TraceFormat", "TraceArrays", "parse_trace", "load_trace", "load_trace_path",
           "format_for_path", "save_binary", "load_binary", "save_trace", "TraceFormatError"]

