"""B200-native BucketServe scheduling hot path (arXiv 2507.17120).

Drop-in names of the reference package (bucketsim) for the scheduling path
(BucketSet, Bucket, BatchController, order_requests, memory-model functions; see
compat.py), with the window hot path on sm_100a kernels behind a C-ABI
(include/bucketserve.h):

    from paper_2507_17120_b200 import WindowScheduler, ModelConfig, GpuConfig
    sched = WindowScheduler(model, gpu, max_requests=1 << 20)
    res = sched.schedule(lengths, classes, tok_off, tokens)   # device tensors
    res.edges(), res.batches(), res.batch_tensors(0)

See DESIGN.md for the kernel map and INTEGRATION.md for the boundary.
"""

from .errors import ConfigError, SimulationError, TraceFormatError
from .memory_model import (MODEL_PRESETS, GpuConfig, LengthHistogram, ModelConfig,
                           expected_waste, kv_footprint_exact, kv_footprint_padded,
                           max_safe_batch, safe_memory, token_budget, waste_ratio)
from .types import (BatchPlan, DispatchPolicy, MemoryAccounting, OversizeRejection,
                    PartitionViolation, Request, StructuralChange, TaskClass)
from ._native import NativeUnavailable
from .compat import (Bucket, BucketSet, BatchController, WindowSchedule, order_requests,
                     schedule_requests)

__version__ = "0.1.0"


def __getattr__(name):
    # the CUDA-backed classes import torch lazily so the pure-host parts stay light
    if name in ("WindowScheduler", "WindowResult", "WindowConfig"):
        from . import window
        return getattr(window, name)
    raise AttributeError(name)
