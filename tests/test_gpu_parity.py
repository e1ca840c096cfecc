"""GPU (sm_100a) window path vs the reference golden fixtures and the CPU oracle.

Bit-exact on every integer output (edges, change log, bucket ids, drain order,
batch membership / rows / sizes / footprints, rejections, pending, packed
tokens and masks); waste_ratio bit-exact as well (same float64 expression,
tolerance in north_star is 1e-6 relative, checked separately)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import cpu  # noqa: E402
from oracle.canon import canonical, diff  # noqa: E402
from golden_util import fixture_names, load  # noqa: E402
from paper_2507_17120_b200 import workloads as W  # noqa: E402
from paper_2507_17120_b200.window import WindowScheduler  # noqa: E402


def _sched(spec, n, **kw):
    return WindowScheduler(max_requests=max(n, 1), max_seq_len=spec["l_max"],
                           n_classes=spec["n_classes"], policies=spec["policies"],
                           split_threshold=spec["theta"], adjust=spec["adjust"],
                           max_passes=spec["max_passes"], buckets=spec["init_edges"],
                           kv_bytes_per_token=spec["kvpt"], current_safe=spec["current_safe"],
                           pledged=spec["pledged"], accounting=spec["accounting"],
                           truncate=spec["truncate"], **kw)


def _canon_gpu(h):
    s = h["summary"]
    return canonical(edges=h["edges"], bucket=h["bucket"], perm=h["perm"],
                     req_batch=h["req_batch"], req_row=h["req_row"], batches=h["batches"],
                     n_max=s["n_max"], changes=h["changes"], n_passes=s["n_passes"])


def _oracle(spec, lens, cls, tok_off=None, tokens=None):
    ws = cpu.WindowSpec(l_max=spec["l_max"], n_classes=spec["n_classes"],
                        policies=spec["policies"], theta=spec["theta"], adjust=spec["adjust"],
                        max_passes=spec["max_passes"], kvpt=spec["kvpt"],
                        current_safe=spec["current_safe"], pledged=spec["pledged"],
                        accounting=spec["accounting"], truncate=spec["truncate"],
                        init_edges=spec["init_edges"])
    return cpu.window(ws, lens, cls, tok_off, tokens)


@pytest.mark.parametrize("name", fixture_names())
def test_gpu_matches_reference_fixture(name):
    spec, lens, cls, ref = load(name)
    n = len(lens)
    rng = np.random.default_rng(5)
    eff = np.minimum(np.maximum(lens, 0), spec["l_max"] - 1)
    tok_off, tokens = W.token_store(eff, rng)
    sched = _sched(spec, n)
    res = sched.schedule(lens, cls, tok_off, tokens)
    h = res.to_host()
    errs = diff(_canon_gpu(h), ref, bit_exact_waste=True)
    assert not errs, f"{name}: " + "; ".join(errs)
    # the packed tensors equal the oracle's
    o = _oracle(spec, lens, cls, tok_off, tokens)
    m = int(h["summary"]["packed_elems"])
    assert m == int(o.summary["packed_elems"])
    if m:
        assert np.array_equal(h["out_tokens"][:m], o.out_tokens[:m])
        assert np.array_equal(h["out_mask"][:m], o.out_mask[:m])
    assert np.array_equal(h["hist"].reshape(-1), o.hist.reshape(-1))
    assert h["summary"]["n_rejected"] == o.summary["n_rejected"]
    assert h["summary"]["n_pending"] == o.summary["n_pending"]
    sched.close()
