"""Window scheduling on the B200: the data-parallel hot path of BucketServe.

One call takes a window of pending requests (arrival order, structure of
arrays) and returns, bit-exact with the reference composition of
BucketSet.assign / adjust_buckets / BatchController.form_batch:

  bucket boundaries + change log   (BucketSet.adjust_buckets, bucket_manager.py:133-191)
  bucket id per request            (BucketSet.assign, bucket_manager.py:110-131)
  drain order                      (order_requests per class, batch_controller.py:33-41)
  batches + outcomes               (BatchController.form_batch, batch_controller.py:141-191)
  packed [n, pitch] tokens + mask  (no reference; padding stats = waste_ratio)

Everything runs in sm_100a kernels behind the C-ABI (include/bucketserve.h);
PyTorch only allocates device buffers, provides the stream, and (for sharded
windows) all-reduces the length histogram over NCCL.
"""

from __future__ import annotations

import collections
import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError
from .memory_model import GpuConfig, ModelConfig, safe_memory
from .sharding import allreduce_histogram
from .types import (CHANGE_KIND, DispatchPolicy, MemoryAccounting, StructuralChange,
                    accounting_code, policy_code)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _stream_handle(device):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _as_device(x, dtype, device):
    if isinstance(x, torch.Tensor):
        if x.device != device or x.dtype != dtype:
            x = x.to(device=device, dtype=dtype)
        return x.contiguous()
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype).to(device)


@dataclass
class WindowConfig:
    """The scheduling knobs of one window (bs_window_params)."""
    max_seq_len: int
    n_classes: int = 2
    policies: tuple = (DispatchPolicy.EARLIEST_ARRIVAL, DispatchPolicy.SJF)
    split_threshold: float = 0.5
    adjust: bool = True
    max_passes: int = 0
    n_max: int | None = None
    kv_bytes_per_token: int = 1
    current_safe: int = 0
    pledged: int = 0
    accounting: MemoryAccounting = MemoryAccounting.PADDED
    truncate: bool = True
    pad_id: int = 0
    dispatch: bool = False

    def params(self) -> N.WindowParams:
        if len(self.policies) != self.n_classes:
            raise ValueError("need one dispatch policy per class")
        if not 0.0 < self.split_threshold <= 1.0:
            raise ValueError("split_threshold must be in (0, 1]")
        if self.max_seq_len < 1:
            raise ValueError("max_seq_len must be >= 1")
        return N.make_params(
            l_max=self.max_seq_len, n_classes=self.n_classes,
            policies=[policy_code(p) for p in self.policies],
            split_threshold=self.split_threshold, adjust=self.adjust, max_passes=self.max_passes,
            n_max=self.n_max, kv_bytes_per_token=self.kv_bytes_per_token,
            current_safe=self.current_safe, pledged=self.pledged,
            accounting=accounting_code(self.accounting), truncate=self.truncate,
            pad_id=self.pad_id, dispatch=self.dispatch)


class WindowResult:
    """Device-resident result of one window; host views are pulled lazily."""

    def __init__(self, sched: "WindowScheduler", n: int, packed: bool):
        self._s = sched
        self.n = n
        self.packed = packed
        self._summary = None

    # ---- device tensors (valid until the scheduler runs the next window) ----
    @property
    def perm(self):
        return self._s.perm[:self.n]

    @property
    def bucket(self):
        return self._s.bucket[:self.n]

    @property
    def req_batch(self):
        return self._s.req_batch[:self.n]

    @property
    def req_row(self):
        return self._s.req_row[:self.n]

    @property
    def hist(self):
        s = self._s
        return s.hist.view(s.cfg.n_classes, s.cfg.max_seq_len)

    @property
    def out_tokens(self):
        return self._s.out_tokens

    @property
    def out_mask(self):
        return self._s.out_mask

    # ---- host views --------------------------------------------------------
    def summary(self) -> dict:
        if self._summary is None:
            raw = self._s.summary.cpu().numpy().view(N.SUMMARY_DTYPE)[0]
            self._summary = {f: (float(raw[f]) if f == "waste_sum" else int(raw[f]))
                             for f in N.SUMMARY_FIELDS}
        return self._summary

    def check(self):
        """Raise the reference's exception for any device-latched data error."""
        N.raise_for_flags(self.summary()["flags"], self._s.cfg.max_seq_len)
        return self

    @property
    def k(self) -> int:
        return self.summary()["k_buckets"]

    @property
    def n_batches(self) -> int:
        return min(self.summary()["n_batches"], self._s.batches_cap)

    def edges(self) -> np.ndarray:
        return self._s.edges[:self.k + 1].cpu().numpy()

    def changes_array(self) -> np.ndarray:
        m = min(self.summary()["n_changes"], self._s.changes_cap)
        return self._s.changes[:4 * m].view(m, 4).cpu().numpy() if m else np.zeros((0, 4), np.int32)

    def changes(self) -> list:
        return [StructuralChange(CHANGE_KIND[int(k)], int(lo), int(up),
                                 None if int(k) == N.CHANGE_MERGE else int(mid))
                for k, lo, up, mid in self.changes_array()]

    def seg_off(self) -> np.ndarray:
        return self._s.seg_off[:self.k * self._s.cfg.n_classes + 1].cpu().numpy()

    def batches(self) -> np.ndarray:
        nb = self.n_batches
        raw = self._s.batches_raw[:nb * 64].cpu().numpy()
        return raw.view(N.BATCH_DTYPE).copy()

    def emit_order(self) -> np.ndarray:
        """f3: batch indices in the simulator's dispatch order (Simulator._next_plan
        repeated, pd_sim.py:448-462); needs dispatch=True."""
        if not self._s.cfg.dispatch:
            raise ValueError("the scheduler was built without dispatch=True")
        t = min(self.summary()["n_dispatched"], self._s.batches_cap)
        return self._s.emit_order[:t].cpu().numpy()

    def batch_emit(self) -> np.ndarray:
        """f3: dispatch rank of every batch, -1 for batches the loop never forms."""
        if not self._s.cfg.dispatch:
            raise ValueError("the scheduler was built without dispatch=True")
        return self._s.batch_emit[:self.n_batches].cpu().numpy()

    def mean_batch_waste(self):
        """pd_sim.py:898-899: mean of per-batch waste_ratio in emission order."""
        b = self.batches()
        return float(np.sum(b["waste"]) / len(b)) if len(b) else None

    def batch_tensors(self, i: int, batches=None):
        """(tokens [n, pitch] int32, mask [n, pitch] uint8) views of batch i."""
        if not self.packed:
            raise ValueError("window was scheduled without a token store")
        b = (batches if batches is not None else self.batches())[i]
        o, n, p = int(b["out_offset"]), int(b["n"]), int(b["pitch"])
        tok = self._s.out_tokens[o:o + n * p].view(n, p)
        msk = self._s.out_mask[o:o + n * p].view(n, p) if self._s.out_mask is not None else None
        return tok, msk

    def to_host(self) -> dict:
        """All outputs as numpy (for checking / logging)."""
        s = self.summary()
        out = dict(summary=s, edges=self.edges(), changes=self.changes_array(),
                   seg_off=self.seg_off(), batches=self.batches(),
                   perm=self.perm.cpu().numpy(), bucket=self.bucket.cpu().numpy(),
                   req_batch=self.req_batch.cpu().numpy(), req_row=self.req_row.cpu().numpy(),
                   hist=self.hist.cpu().numpy().view(np.uint32))
        if self._s.cfg.dispatch:
            out["emit_order"] = self.emit_order()
            out["batch_emit"] = self.batch_emit()
        if self.packed:
            m = int(s["packed_elems"])
            out["out_tokens"] = self._s.out_tokens[:m].cpu().numpy()
            if self._s.out_mask is not None:
                out["out_mask"] = self._s.out_mask[:m].cpu().numpy()
        return out


class WindowScheduler:
    """GPU window scheduler with preallocated buffers for up to `max_requests`.

    Memory comes either from reference objects (`model`, `gpu`: kv bytes per
    token = ModelConfig.kv_bytes_per_token, safe memory = safe_memory(gpu)) or
    from raw `kv_bytes_per_token` / `current_safe`.
    """

    def __init__(self, model: ModelConfig | None = None, gpu: GpuConfig | None = None, *,
                 max_requests: int, max_seq_len: int | None = None, n_classes: int = 2,
                 policies=None, offline_policy=DispatchPolicy.SJF,
                 accounting=MemoryAccounting.PADDED, split_threshold: float = 0.5,
                 adjust: bool = True, max_passes: int = 0, buckets=None, pledged: int = 0,
                 truncate: bool = True, pad_id: int = 0, kv_bytes_per_token: int | None = None,
                 current_safe: int | None = None, n_max: int | None = None, device=None,
                 pack_capacity: int | None = None, with_mask: bool = True,
                 changes_cap: int | None = None, batches_cap: int | None = None,
                 process_group=None, dispatch: bool = False, collective: str = "nccl"):
        if not torch.cuda.is_available():
            raise N.NativeUnavailable("no CUDA device: the window scheduler runs only on a B200")
        if max_seq_len is None:
            if model is None:
                raise ConfigError("max_seq_len or model is required")
            max_seq_len = model.max_seq_len
        kvpt = kv_bytes_per_token if kv_bytes_per_token is not None else (
            model.kv_bytes_per_token if model is not None else None)
        safe = current_safe if current_safe is not None else (
            safe_memory(gpu) if gpu is not None else None)
        if kvpt is None or safe is None:
            raise ConfigError("memory model needs (model, gpu) or (kv_bytes_per_token, current_safe)")
        if policies is None:
            policies = (DispatchPolicy.EARLIEST_ARRIVAL,) + (offline_policy,) * (n_classes - 1)
        if not 1 <= n_classes <= N.MAX_CLASSES:
            raise ValueError(f"n_classes must be in [1, {N.MAX_CLASSES}]")
        self.cfg = WindowConfig(max_seq_len=max_seq_len, n_classes=n_classes,
                                policies=tuple(policies), split_threshold=split_threshold,
                                adjust=adjust, max_passes=max_passes, n_max=n_max,
                                kv_bytes_per_token=kvpt, current_safe=safe, pledged=pledged,
                                accounting=accounting, truncate=truncate, pad_id=pad_id,
                                dispatch=dispatch)
        self._params = self.cfg.params()
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else
                                   torch.device(device).index or 0)
        self.max_requests = int(max_requests)
        self.ctx = N.Context(self.device.index, self.max_requests, max_seq_len, n_classes)
        L, Cn, Nmax = max_seq_len, n_classes, self.max_requests
        dev = self.device
        i32 = dict(dtype=torch.int32, device=dev)
        self.hist = torch.zeros(Cn * L, **i32)
        self.hist_global = torch.zeros(Cn * L, **i32) if process_group is not None else None
        self.process_group = process_group
        if collective not in ("nccl", "torch", "peer"):
            raise ValueError("collective must be 'nccl' (the library's NCCL communicator, C1 "
                             "inside the window), 'torch' (torch.distributed all-reduce between "
                             "K1 and K2) or 'peer' (CUDA-IPC peer memory)")
        self.collective = collective if process_group is not None else "none"
        self._nccl = False
        if self.collective == "peer":
            self._peer_connect()
        elif self.collective == "nccl":
            self._nccl_connect()
        self.edges = torch.zeros(L + 1, **i32)
        self.changes_cap = int(changes_cap if changes_cap is not None else 4 * L + 64)
        self.changes = torch.zeros(4 * self.changes_cap, **i32)
        self.bucket = torch.zeros(max(Nmax, 1), **i32)
        self.perm = torch.zeros(max(Nmax, 1), **i32)
        self.seg_off = torch.zeros(L * Cn + 1, **i32)
        self.batches_cap = int(batches_cap if batches_cap is not None else max(Nmax, 1))
        self.batches_raw = torch.zeros(64 * self.batches_cap, dtype=torch.uint8, device=dev)
        self.req_batch = torch.zeros(max(Nmax, 1), **i32)
        self.req_row = torch.zeros(max(Nmax, 1), **i32)
        self.summary = torch.zeros(256, dtype=torch.uint8, device=dev)
        self.emit_order = torch.zeros(self.batches_cap, **i32) if dispatch else None
        self.batch_emit = torch.zeros(self.batches_cap, **i32) if dispatch else None
        self.init_edges = None
        self.k_init = 0
        if buckets is not None:
            e = np.asarray(buckets, np.int32)
            self.init_edges = torch.as_tensor(e).to(dev)
            self.k_init = len(e) - 1
        self.with_mask = with_mask
        # captured window graphs by input buffers (a double-buffered serving loop
        # alternates two input sets), least recently used first
        self._graphs = collections.OrderedDict()
        self.out_tokens = None
        self.out_mask = None
        self.pack_capacity = 0
        if pack_capacity:
            self._ensure_pack(int(pack_capacity))

    _RECONFIGURABLE = ("policies", "split_threshold", "adjust", "max_passes", "n_max",
                       "kv_bytes_per_token", "current_safe", "pledged", "accounting",
                       "truncate", "pad_id")

    def configure(self, *, buckets=(), **fields) -> "WindowScheduler":
        """Change the per-window knobs (policies, memory, threshold, initial edges, ...)
        without reallocating: the buffers depend only on (max_requests, max_seq_len,
        n_classes, dispatch).  A captured graph is dropped when anything changed."""
        bad = set(fields) - set(self._RECONFIGURABLE)
        if bad:
            raise ValueError(f"not reconfigurable: {sorted(bad)}")
        if "policies" in fields:
            fields["policies"] = tuple(fields["policies"])
        changed = any(getattr(self.cfg, k) != v for k, v in fields.items())
        if changed:
            old = {k: getattr(self.cfg, k) for k in fields}
            for k, v in fields.items():
                setattr(self.cfg, k, v)
            try:
                self._params = self.cfg.params()
            except Exception:
                for k, v in old.items():
                    setattr(self.cfg, k, v)
                raise
        if buckets != ():
            if buckets is None:
                changed |= self.init_edges is not None
                self.init_edges, self.k_init = None, 0
            else:
                e = np.asarray(buckets, np.int32)
                same = (self.init_edges is not None and self.k_init == len(e) - 1
                        and bool(torch.equal(self.init_edges.cpu(), torch.as_tensor(e))))
                if not same:
                    self.init_edges = torch.as_tensor(e).to(self.device)
                    self.k_init = len(e) - 1
                    changed = True
        if changed:
            self._graphs.clear()
        return self

    # ------------------------------------------------------------------------
    def _peer_connect(self):
        """C1 over peer memory: share this context's exchange buffer with the other ranks
        (CUDA IPC handles gathered over the process group) and map theirs."""
        import torch.distributed as dist
        lib = N.load()
        h = (C.c_ubyte * N.PEER_HANDLE_BYTES)()
        N.check(lib.bs_peer_export(self.ctx.ptr, h), self.ctx.ptr)
        world = dist.get_world_size(self.process_group)
        rank = dist.get_rank(self.process_group)
        got = [None] * world
        dist.all_gather_object(got, bytes(h), group=self.process_group)
        allh = (C.c_ubyte * (N.PEER_HANDLE_BYTES * world)).from_buffer_copy(b"".join(got))
        N.check(lib.bs_peer_connect(self.ctx.ptr, rank, world, allh), self.ctx.ptr)

    def _nccl_connect(self):
        """C1 over the library's own NCCL communicator: rank 0 makes the unique id, the
        process group carries it to the other ranks, every rank attaches it to its
        context (bs_nccl_connect); bs_window_schedule then all-reduces the histogram
        between K1 and K2 on the window's stream — inside the window's CUDA graph."""
        import torch.distributed as dist
        rank = dist.get_rank(self.process_group)
        world = dist.get_world_size(self.process_group)
        uid = bytearray(N.NCCL_ID_BYTES)
        if rank == 0:
            uid = self.nccl_unique_id()
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(self.process_group, 0)
                                   if self.process_group is not dist.group.WORLD else 0,
                                   group=self.process_group)
        self.attach_nccl(rank, world, obj[0])

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_ubyte * N.NCCL_ID_BYTES)()
        N.check(N.load().bs_nccl_unique_id(buf), None)
        return bytes(buf)

    def attach_nccl(self, rank: int, world: int, unique_id: bytes):
        """Attach an NCCL communicator (ncclCommInitRank over `unique_id`) to this
        scheduler's context; every window then runs C1 itself (also with world = 1)."""
        buf = (C.c_ubyte * N.NCCL_ID_BYTES).from_buffer_copy(bytes(unique_id))
        with torch.cuda.device(self.device):
            N.check(N.load().bs_nccl_connect(self.ctx.ptr, int(rank), int(world), buf), self.ctx.ptr)
        self._nccl = True
        self.collective = "nccl"
        if self.hist_global is None:
            self.hist_global = torch.zeros_like(self.hist)
        self._graphs.clear()

    _GRAPHS = 4  # captured graphs kept per scheduler

    def _graph_for(self, key):
        g = self._graphs.get(key)
        if g is not None:
            self._graphs.move_to_end(key)
        return g

    def _keep_graph(self, key, g):
        self._graphs[key] = g
        while len(self._graphs) > self._GRAPHS:
            self._graphs.popitem(last=False)

    def _ensure_pack(self, cap: int):
        if cap <= self.pack_capacity:
            return
        cap = (cap + 63) // 64 * 64
        self._graphs.clear()  # captured graphs write the outputs being replaced
        self.out_tokens = torch.empty(cap, dtype=torch.int32, device=self.device)
        self.out_mask = torch.empty(cap, dtype=torch.uint8, device=self.device) if self.with_mask else None
        self.pack_capacity = cap

    def _io(self, lens, cls, n, tok_off, tokens, pack: bool) -> N.WindowIO:
        io = N.WindowIO()
        io.len, io.cls = _ptr(lens), _ptr(cls)
        io.tok_off = _ptr(tok_off) if pack else None
        io.tokens = _ptr(tokens) if pack else None
        io.n = n
        io.init_edges = _ptr(self.init_edges)
        io.k_init = self.k_init
        io.changes_cap = self.changes_cap
        io.batches_cap = self.batches_cap
        io.out_capacity = self.pack_capacity if pack else 0
        io.hist = _ptr(self.hist)
        io.hist_global = _ptr(self.hist_global) if self.hist_global is not None else None
        io.edges, io.changes = _ptr(self.edges), _ptr(self.changes)
        io.bucket, io.perm, io.seg_off = _ptr(self.bucket), _ptr(self.perm), _ptr(self.seg_off)
        io.batches = _ptr(self.batches_raw)
        io.req_batch, io.req_row = _ptr(self.req_batch), _ptr(self.req_row)
        io.out_tokens = _ptr(self.out_tokens) if pack else None
        io.out_mask = _ptr(self.out_mask) if (pack and self.out_mask is not None) else None
        io.summary = _ptr(self.summary)
        io.emit_order = _ptr(self.emit_order)
        io.batch_emit = _ptr(self.batch_emit)
        return io

    def _inputs(self, lengths, classes):
        dev = self.device
        lens = _as_device(lengths, torch.int32, dev)
        cls = _as_device(classes, torch.uint8, dev)
        n = int(lens.numel())
        if cls.numel() != n:
            raise ValueError("lengths and classes differ in length")
        if n > self.max_requests:
            raise ValueError(f"window of {n} exceeds max_requests={self.max_requests}")
        return lens, cls, n

    def histogram(self, lengths, classes, *, sync: bool = True):
        """K1 only: the window's per-(class, length) counts as an int32 [C, L] tensor
        (a copy; uint32 bit patterns).  Used to build a global histogram by hand."""
        lens, cls, n = self._inputs(lengths, classes)
        with torch.cuda.device(self.device):
            N.check(N.load().bs_histogram(self.ctx.ptr, _ptr(lens), _ptr(cls), n,
                                          C.byref(self._params), _ptr(self.hist),
                                          _ptr(self.summary), _stream_handle(self.device)),
                    self.ctx.ptr)
        out = self.hist.view(self.cfg.n_classes, self.cfg.max_seq_len).clone()
        if sync:
            torch.cuda.current_stream(self.device).synchronize()
        return out

    def schedule(self, lengths, classes, tok_off=None, tokens=None, *, sync: bool = True,
                 check: bool = True, hist_reduce=None, graph: bool = False) -> WindowResult:
        """Schedule one window.  `lengths` int32[n] and `classes` uint8[n] in arrival
        order (device tensors, or host arrays that are copied); optional CSR token
        store (`tok_off` int64[n+1], `tokens` int32[...]) enables packing.

        Sharded windows: with a process group (constructor) the local histogram is
        all-reduced across the ranks (C1: collective 'nccl' inside the fused call, or
        'peer', or 'torch' between K1 and K2); `hist_reduce(hist)` may instead transform
        the local histogram in place into the global one (e.g. in single-GPU tests).

        graph=True replays the whole fused window (16-20 kernels) as one CUDA graph,
        captured on the first call for these input buffers (serving loops reuse
        their input buffers); launch gaps between the stages disappear.  Sharded
        windows replay K2..K6 as a graph after the eager K1 + all-reduce."""
        dev = self.device
        lens, cls, n = self._inputs(lengths, classes)
        pack = tok_off is not None and tokens is not None
        if pack:
            tok_off = _as_device(tok_off, torch.int64, dev)
            tokens = _as_device(tokens, torch.int32, dev)
            if tok_off.numel() < n:
                raise ValueError("tok_off must hold at least n offsets")
        lib = N.load()
        st = _stream_handle(dev)
        p = self._params
        if pack and n == 0:
            self._ensure_pack(64)  # nothing to pack; keep the result shape uniform
        two_phase = pack and self.pack_capacity == 0
        sharded = self.process_group is not None or hist_reduce is not None or self._nccl
        # C1 inside the fused call: the library's NCCL communicator or peer memory
        fused = not sharded or (self.collective in ("nccl", "peer") and hist_reduce is None)
        if graph and fused and not two_phase:
            key = (lens.data_ptr(), cls.data_ptr(), n,
                   tok_off.data_ptr() if pack else 0, tokens.data_ptr() if pack else 0,
                   self.pack_capacity)
            g = self._graph_for(key)
            if g is None:
                torch.cuda.synchronize(dev)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, capture_error_mode="thread_local"):
                    io_g = self._io(lens, cls, n, tok_off, tokens, pack)
                    if sharded:  # NCCL / peer context: C1 runs inside the fused call
                        io_g.hist_global = _ptr(self.hist_global)
                    N.check(lib.bs_window_schedule(self.ctx.ptr, C.byref(io_g), C.byref(p),
                                                   _stream_handle(dev)), self.ctx.ptr)
                self._keep_graph(key, g)
            g.replay()
            res = WindowResult(self, n, pack)
            if sync:
                torch.cuda.current_stream(dev).synchronize()
                if check:
                    res.check()
            return res
        if sharded and self.hist_global is None:
            self.hist_global = torch.zeros_like(self.hist)
        if graph and sharded and not fused and not two_phase:
            # K1 and the histogram all-reduce (C1) run eagerly; K2..K6 on the reduced
            # histogram replay as one CUDA graph
            with torch.cuda.device(dev):
                N.check(lib.bs_histogram(self.ctx.ptr, _ptr(lens), _ptr(cls), n, C.byref(p),
                                         _ptr(self.hist), _ptr(self.summary), st), self.ctx.ptr)
                self.hist_global.copy_(self.hist)
                if hist_reduce is not None:
                    hist_reduce(self.hist_global)
                else:
                    allreduce_histogram(self.hist_global, self.process_group)
            key = ("from_hist", lens.data_ptr(), cls.data_ptr(), n,
                   tok_off.data_ptr() if pack else 0, tokens.data_ptr() if pack else 0,
                   self.pack_capacity)
            g = self._graph_for(key)
            if g is None:
                torch.cuda.synchronize(dev)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, capture_error_mode="thread_local"):
                    io_g = self._io(lens, cls, n, tok_off, tokens, pack)
                    io_g.hist_global = _ptr(self.hist_global)
                    N.check(lib.bs_window_from_hist(self.ctx.ptr, C.byref(io_g), C.byref(p),
                                                    _stream_handle(dev)), self.ctx.ptr)
                self._keep_graph(key, g)
            g.replay()
            res = WindowResult(self, n, pack)
            if sync:
                torch.cuda.current_stream(dev).synchronize()
                if check:
                    res.check()
            return res
        io = self._io(lens, cls, n, tok_off, tokens, pack and not two_phase)
        with torch.cuda.device(dev):
            if fused:
                if sharded:
                    io.hist_global = _ptr(self.hist_global)
                N.check(lib.bs_window_schedule(self.ctx.ptr, C.byref(io), C.byref(p), st), self.ctx.ptr)
            else:
                N.check(lib.bs_histogram(self.ctx.ptr, _ptr(lens), _ptr(cls), n, C.byref(p),
                                         _ptr(self.hist), _ptr(self.summary), st), self.ctx.ptr)
                self.hist_global.copy_(self.hist)
                if hist_reduce is not None:
                    hist_reduce(self.hist_global)
                else:  # C1: sum of per-rank histograms over NCCL (NVLink / NVSwitch)
                    allreduce_histogram(self.hist_global, self.process_group)
                io.hist_global = _ptr(self.hist_global)
                N.check(lib.bs_window_from_hist(self.ctx.ptr, C.byref(io), C.byref(p), st),
                        self.ctx.ptr)
            if two_phase:
                # first packed window: size the reusable output buffer from the plan
                need = int(self.summary[96:104].cpu().view(torch.int64).item())  # packed_elems
                self._ensure_pack(max(need, 64))
            if two_phase and tokens.numel() > 0:  # an empty store: every row is padding-free
                N.check(lib.bs_pack(self.ctx.ptr, _ptr(lens), _ptr(self.perm), _ptr(tok_off),
                                    _ptr(tokens), C.byref(p), _ptr(self.batches_raw), 0, -1,
                                    _ptr(self.out_tokens), _ptr(self.out_mask),
                                    self.pack_capacity, _ptr(self.summary), st), self.ctx.ptr)
        res = WindowResult(self, n, pack)
        if sync:
            torch.cuda.current_stream(dev).synchronize()
            s = res.summary()
            if pack and (s["flags"] & N.FLAG_PACK_CAPACITY):
                # the packed extent outgrew the reusable buffer: grow it and re-pack
                self._ensure_pack(int(s["packed_elems"]))
                keep = int(s["flags"]) & ~N.FLAG_PACK_CAPACITY  # flags word at byte 128
                self.summary[128:136].copy_(torch.tensor([keep], dtype=torch.int64).view(torch.uint8))
                with torch.cuda.device(dev):
                    N.check(lib.bs_pack(self.ctx.ptr, _ptr(lens), _ptr(self.perm), _ptr(tok_off),
                                        _ptr(tokens), C.byref(p), _ptr(self.batches_raw), 0, -1,
                                        _ptr(self.out_tokens), _ptr(self.out_mask),
                                        self.pack_capacity, _ptr(self.summary), st), self.ctx.ptr)
                torch.cuda.current_stream(dev).synchronize()
                res = WindowResult(self, n, pack)
            if check:
                res.check()
        return res

    def boundaries(self, lengths, classes=None, *, init_edges=None, n_max=None,
                   max_passes=None):
        """K1 + K2 only: BucketSet.adjust_buckets run `max_passes` times (None: the
        configured value) from `init_edges` (None: the configured edges) with an
        explicit split floor `n_max` (None: current_n_max from the histogram).
        Returns (edges, [StructuralChange], summary)."""
        if classes is None:
            classes = np.zeros(len(lengths), np.uint8)
        lens, cls, n = self._inputs(lengths, classes)
        p = N.WindowParams.from_buffer_copy(self._params)
        if n_max is not None:
            p.n_max = int(n_max)
        if max_passes is not None:
            p.max_passes = int(max_passes)
        ie, k_init = self.init_edges, self.k_init
        if init_edges is not None:
            e = np.asarray(init_edges, np.int32)
            ie, k_init = torch.as_tensor(e).to(self.device), len(e) - 1
        lib = N.load()
        st = _stream_handle(self.device)
        with torch.cuda.device(self.device):
            N.check(lib.bs_histogram(self.ctx.ptr, _ptr(lens), _ptr(cls), n, C.byref(p),
                                     _ptr(self.hist), _ptr(self.summary), st), self.ctx.ptr)
            N.check(lib.bs_boundaries(self.ctx.ptr, _ptr(self.hist), _ptr(self.hist), C.byref(p),
                                      _ptr(ie), k_init, _ptr(self.edges), _ptr(self.changes),
                                      self.changes_cap, _ptr(self.summary), st), self.ctx.ptr)
        torch.cuda.current_stream(self.device).synchronize()
        res = WindowResult(self, n, False)
        res.check()
        return res.edges(), res.changes(), res.summary()

    def boundaries_from_hist(self, hist, *, init_edges=None, n_max=None, max_passes=None):
        """K2 only, on a caller-maintained histogram (int [C, L] or [L] for one class):
        the incremental form SURVEY f1 asks for — the stateful BucketSet keeps per-length
        counts up to date on assign / removal and uploads C*L words per adjust instead of
        re-histogramming every queued request.  Same returns as boundaries()."""
        h = np.ascontiguousarray(np.asarray(hist).reshape(-1), dtype=np.int64)
        Cn, L = self.cfg.n_classes, self.cfg.max_seq_len
        if h.size != Cn * L:
            raise ValueError(f"histogram has {h.size} counts, expected {Cn * L}")
        if h.size and (h.min() < 0 or h.max() > 0xFFFFFFFF):
            raise ValueError("histogram counts out of range")
        p = N.WindowParams.from_buffer_copy(self._params)
        if n_max is not None:
            p.n_max = int(n_max)
        if max_passes is not None:
            p.max_passes = int(max_passes)
        ie, k_init = self.init_edges, self.k_init
        if init_edges is not None:
            e = np.asarray(init_edges, np.int32)
            ie, k_init = torch.as_tensor(e).to(self.device), len(e) - 1
        lib = N.load()
        st = _stream_handle(self.device)
        with torch.cuda.device(self.device):
            # an empty K1 initialises the summary; the counts then replace the histogram
            N.check(lib.bs_histogram(self.ctx.ptr, None, None, 0, C.byref(p), _ptr(self.hist),
                                     _ptr(self.summary), st), self.ctx.ptr)
            self.hist.copy_(torch.from_numpy(h.astype(np.uint32).view(np.int32)))
            N.check(lib.bs_boundaries(self.ctx.ptr, _ptr(self.hist), _ptr(self.hist), C.byref(p),
                                      _ptr(ie), k_init, _ptr(self.edges), _ptr(self.changes),
                                      self.changes_cap, _ptr(self.summary), st), self.ctx.ptr)
        torch.cuda.current_stream(self.device).synchronize()
        res = WindowResult(self, int(h.sum()), False)
        res.check()
        return res.edges(), res.changes(), res.summary()

    def monitor_bins(self, bins: int = 64) -> np.ndarray:
        """f2: the 64-bin LengthHistogram view of the last window (pd_sim.py:828-833)."""
        out = torch.zeros(bins, dtype=torch.int64, device=self.device)
        N.check(N.load().bs_monitor_bins(self.ctx.ptr, _ptr(self.hist_global if self.hist_global
                                                            is not None else self.hist),
                                         C.byref(self._params), bins, _ptr(out),
                                         _stream_handle(self.device)), self.ctx.ptr)
        return out.cpu().numpy()

    def monitor_from_hist(self, hist, edges, *, bins: int = 64):
        """f2 on a caller-maintained per-length histogram (int [C, L] or [L]): the
        simulator's per-tick monitor (pd_sim.py:828-833) — the LengthHistogram of the
        queued lengths (bins over [0, max_seq_len)) and expected_waste of the bucket
        partition `edges` — from one K8 launch.  Raises the reference's ValueError
        where expected_waste does (memory_model.py:167-183).
        Returns (LengthHistogram, expected_waste)."""
        from .memory_model import LengthHistogram, check_waste_partition
        h = np.ascontiguousarray(np.asarray(hist).reshape(-1), dtype=np.int64)
        Cn, L = self.cfg.n_classes, self.cfg.max_seq_len
        if h.size != Cn * L:
            raise ValueError(f"histogram has {h.size} counts, expected {Cn * L}")
        e = np.asarray(edges, np.int32)
        dev = self.device
        counts = torch.empty(bins, dtype=torch.int64, device=dev)
        stats = torch.empty(3, dtype=torch.float64, device=dev)
        d_edges = torch.as_tensor(e).to(dev)
        with torch.cuda.device(dev):
            self.hist.copy_(torch.from_numpy(h.astype(np.uint32).view(np.int32)))
            N.check(N.load().bs_monitor(self.ctx.ptr, _ptr(self.hist), C.byref(self._params),
                                        bins, _ptr(d_edges), len(e) - 1, _ptr(counts),
                                        _ptr(stats), _stream_handle(dev)), self.ctx.ptr)
        hist_obj = LengthHistogram.from_bin_counts(counts.cpu().numpy(), bins, (0, L))
        check_waste_partition(hist_obj, list(zip(e[:-1].tolist(), e[1:].tolist())))
        return hist_obj, float(stats[0].item())

    def monitor(self, *, bins: int = 64):
        """f2 for the last window: (LengthHistogram, expected_waste of its edges)."""
        res = WindowResult(self, 0, False)
        h = (self.hist_global if self.hist_global is not None else self.hist)
        hist = h.cpu().numpy().view(np.uint32).astype(np.int64)
        return self.monitor_from_hist(hist, res.edges(), bins=bins)

    def close(self):
        """Release the context scratch, the captured graph and the output buffers."""
        self.ctx.close()
        self._graphs.clear()
        self.out_tokens = self.out_mask = None
        self.pack_capacity = 0
