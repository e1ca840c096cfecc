"""The C-ABI library: loads, exports every symbol include/bucketserve.h declares, and
its struct layouts agree with the Python binding.  No compute calls (CPU-safe)."""

import ctypes as C
import os
import re

import pytest

from paper_2507_17120_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bucketserve.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(bs_[a-z_]+)\s*\(", src, re.M)))


def test_library_built_in_tree():
    assert os.path.exists(N.LIB_PATH), "run `python -m paper_2507_17120_b200.build`"
    assert N.LIB_PATH.startswith(ROOT)


def test_exports_every_declared_symbol():
    lib = N.load()
    decl = declared_functions()
    assert len(decl) >= 15
    for name in decl:
        assert hasattr(lib, name), name
    assert set(decl) == set(N.EXPORTS)


def test_abi_version():
    assert N.load().bs_abi_version() == 2


def test_struct_layouts_match_header():
    assert C.sizeof(N.WindowParams) == 104
    assert C.sizeof(N.WindowIO) == 192
    assert N.BATCH_DTYPE.itemsize == 64
    assert N.SUMMARY_DTYPE.itemsize == 256
    src = open(HEADER).read()
    for f in ("l_max", "n_classes", "policy", "split_threshold", "adjust", "max_passes", "n_max",
              "kv_bytes_per_token", "current_safe", "pledged", "accounting", "truncate", "pad_id", "dispatch"):
        assert re.search(rf"\b{f}\b", src), f
    for f in N.BATCH_DTYPE.names:
        assert re.search(rf"\b{f}\b", src), f
    for f in N.SUMMARY_FIELDS:
        assert re.search(rf"\b{f}\b", src), f
    for f, _ in N.WindowIO._fields_:
        assert re.search(rf"\b{f}\b", src), f


def test_create_without_gpu_fails_cleanly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(N.NativeUnavailable):
        N.Context(0, 1000, 4096, 2)


def test_null_context_is_rejected():
    lib = N.load()
    p = N.make_params(l_max=16, n_classes=1, policies=[0], split_threshold=0.5, adjust=True,
                      max_passes=0, n_max=0, kv_bytes_per_token=2, current_safe=100, pledged=0,
                      accounting=0, truncate=True, pad_id=0)
    rc = lib.bs_histogram(None, None, None, 0, C.byref(p), None, None, None)
    assert rc == N.BS_ERR_INVALID_ARG
    assert b"ctx" in lib.bs_last_error(None)


def test_create_rejects_bad_capacity():
    lib = N.load()
    ctx = C.c_void_p()
    assert lib.bs_create(C.byref(ctx), 0, -5, 4096, 2) == N.BS_ERR_INVALID_ARG
    assert lib.bs_create(C.byref(ctx), 0, 10, 4096, 9) == N.BS_ERR_INVALID_ARG
