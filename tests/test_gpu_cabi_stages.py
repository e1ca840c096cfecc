"""The unfused C-ABI stage by stage (include/bucketserve.h), called through ctypes with
torch device buffers exactly as a bucketsim binding would:
bs_histogram -> bs_boundaries -> bs_assign / bs_order -> bs_size -> bs_dispatch ->
bs_pack (whole, and chunked over batch ranges into a reusable buffer), checked
against the CPU oracle and the live-reference fixtures."""

import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import cpu  # noqa: E402
from golden_util import load  # noqa: E402
from paper_2507_17120_b200 import _native as N  # noqa: E402
from paper_2507_17120_b200 import workloads as W  # noqa: E402

DEV = torch.device("cuda", 0)


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _run_stages(spec, lens, cls, tok_off, tokens, chunk=None):
    lib = N.load()
    n, L, Cn = len(lens), spec["l_max"], spec["n_classes"]
    ctx = N.Context(0, max(n, 1), L, Cn)
    prm = N.make_params(l_max=L, n_classes=Cn, policies=spec["policies"],
                        split_threshold=spec["theta"], adjust=spec["adjust"],
                        max_passes=spec["max_passes"], n_max=0, kv_bytes_per_token=spec["kvpt"],
                        current_safe=spec["current_safe"], pledged=spec["pledged"],
                        accounting=spec["accounting"], truncate=spec["truncate"], pad_id=0,
                        dispatch=True)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    i32 = dict(dtype=torch.int32, device=DEV)
    d_len = torch.as_tensor(lens).to(DEV)
    d_cls = torch.as_tensor(cls).to(DEV)
    d_off = torch.as_tensor(tok_off).to(DEV)
    d_tok = torch.as_tensor(tokens).to(DEV)
    hist = torch.zeros(Cn * L, **i32)
    summ = torch.zeros(256, dtype=torch.uint8, device=DEV)
    N.check(lib.bs_histogram(ctx.ptr, _p(d_len), _p(d_cls), n, C.byref(prm), _p(hist), _p(summ), st), ctx.ptr)
    edges = torch.zeros(L + 1, **i32)
    cap = 4 * L + 64
    changes = torch.zeros(4 * cap, **i32)
    init = None
    k_init = 0
    if spec["init_edges"] is not None:
        init = torch.as_tensor(np.asarray(spec["init_edges"], np.int32)).to(DEV)
        k_init = len(spec["init_edges"]) - 1
    N.check(lib.bs_boundaries(ctx.ptr, _p(hist), _p(hist), C.byref(prm), _p(init), k_init, _p(edges),
                              _p(changes), cap, _p(summ), st), ctx.ptr)
    bucket_a = torch.zeros(max(n, 1), **i32)
    N.check(lib.bs_assign(ctx.ptr, _p(d_len), n, C.byref(prm), _p(bucket_a), st), ctx.ptr)
    perm = torch.zeros(max(n, 1), **i32)
    seg_off = torch.zeros(L * Cn + 1, **i32)
    bucket_b = torch.zeros(max(n, 1), **i32)
    N.check(lib.bs_order(ctx.ptr, _p(d_len), _p(d_cls), n, C.byref(prm), _p(perm), _p(seg_off),
                         _p(bucket_b), _p(summ), st), ctx.ptr)
    bcap = max(n, 1)
    batches = torch.zeros(64 * bcap, dtype=torch.uint8, device=DEV)
    rb = torch.zeros(max(n, 1), **i32)
    rr = torch.zeros(max(n, 1), **i32)
    N.check(lib.bs_size(ctx.ptr, _p(d_len), _p(perm), _p(seg_off), n, C.byref(prm), _p(batches), bcap,
                        _p(rb), _p(rr), _p(summ), st), ctx.ptr)
    # the plan before K7 rewrites unreached requests
    plan_rb, plan_rr = rb.clone(), rr.clone()
    emit = torch.zeros(bcap, **i32)
    bemit = torch.zeros(bcap, **i32)
    N.check(lib.bs_dispatch(ctx.ptr, _p(perm), _p(seg_off), n, C.byref(prm), _p(batches), bcap, _p(rb),
                            _p(rr), _p(emit), _p(bemit), _p(summ), st), ctx.ptr)
    torch.cuda.synchronize()
    s = summ.cpu().numpy().view(N.SUMMARY_DTYPE)[0]
    nb = int(s["n_batches"])
    b = batches[:64 * nb].cpu().numpy().view(N.BATCH_DTYPE)
    total = int(s["packed_elems"])
    out = {"summary": s, "edges": edges[:int(s["k_buckets"]) + 1].cpu().numpy(),
           "bucket_a": bucket_a[:n].cpu().numpy(), "bucket_b": bucket_b[:n].cpu().numpy(),
           "perm": perm[:n].cpu().numpy(), "seg_off": seg_off.cpu().numpy(), "batches": b,
           "plan_rb": plan_rb[:n].cpu().numpy(), "plan_rr": plan_rr[:n].cpu().numpy(),
           "rb": rb[:n].cpu().numpy(), "rr": rr[:n].cpu().numpy(),
           "emit": emit[:int(s["n_dispatched"])].cpu().numpy(), "bemit": bemit[:nb].cpu().numpy()}
    # K6: whole window, then chunked over batch ranges into one reusable buffer
    cap_el = max(64, total)
    tok_all = torch.full((cap_el,), -7, **i32)
    msk_all = torch.zeros(cap_el, dtype=torch.uint8, device=DEV)
    if nb:
        N.check(lib.bs_pack(ctx.ptr, _p(d_len), _p(perm), _p(d_off), _p(d_tok), C.byref(prm), _p(batches),
                            0, -1, _p(tok_all), _p(msk_all), cap_el, _p(summ), st), ctx.ptr)
    torch.cuda.synchronize()
    out["tokens"], out["mask"] = tok_all[:total].cpu().numpy(), msk_all[:total].cpu().numpy()
    if nb:  # a mask buffer that is only 4-byte aligned: the register-stream fallback
        tok_u = torch.full((cap_el + 8,), -7, **i32)
        msk_u = torch.zeros(cap_el + 16, dtype=torch.uint8, device=DEV)
        N.check(lib.bs_pack(ctx.ptr, _p(d_len), _p(perm), _p(d_off), _p(d_tok), C.byref(prm),
                            _p(batches), 0, -1, C.c_void_p(tok_u.data_ptr() + 16),
                            C.c_void_p(msk_u.data_ptr() + 4), cap_el, _p(summ), st), ctx.ptr)
        torch.cuda.synchronize()
        out["tokens_u"] = tok_u[4:4 + total].cpu().numpy()
        out["mask_u"] = msk_u[4:4 + total].cpu().numpy()
    if chunk and nb:
        pieces_t, pieces_m = [], []
        buf_t = torch.empty(cap_el, **i32)
        buf_m = torch.empty(cap_el, dtype=torch.uint8, device=DEV)
        for b0 in range(0, nb, chunk):
            b1 = min(nb, b0 + chunk)
            ext = int(b[b1 - 1]["out_offset"] + b[b1 - 1]["n"] * b[b1 - 1]["pitch"] - b[b0]["out_offset"])
            N.check(lib.bs_pack(ctx.ptr, _p(d_len), _p(perm), _p(d_off), _p(d_tok), C.byref(prm),
                                _p(batches), b0, b1, _p(buf_t), _p(buf_m), cap_el, _p(summ), st), ctx.ptr)
            torch.cuda.synchronize()
            pieces_t.append(buf_t[:ext].cpu().numpy())
            pieces_m.append(buf_m[:ext].cpu().numpy())
        out["chunked_tokens"] = np.concatenate(pieces_t)
        out["chunked_mask"] = np.concatenate(pieces_m)
    ctx.close()
    return out


def _ws(spec):
    return cpu.WindowSpec(l_max=spec["l_max"], n_classes=spec["n_classes"], policies=spec["policies"],
                          theta=spec["theta"], adjust=spec["adjust"], max_passes=spec["max_passes"],
                          kvpt=spec["kvpt"], current_safe=spec["current_safe"],
                          pledged=spec["pledged"], accounting=spec["accounting"],
                          truncate=spec["truncate"], init_edges=spec["init_edges"])


@pytest.mark.parametrize("name", ["c2_n30000", "reject_heavy_acc1", "pledged_acc0", "one_pass_split",
                                  "four_class_exact", "tiny_L7_ljf_exact", "dispatch_online_rejects"])
def test_stages_match_oracle(name):
    spec, lens, cls, ref = load(name)
    eff = np.minimum(np.maximum(lens, 0), spec["l_max"] - 1)
    tok_off, tokens = W.token_store(eff)
    g = _run_stages(spec, lens, cls, tok_off, tokens, chunk=7)
    o = cpu.window(_ws(spec), lens, cls, tok_off, tokens)
    d = cpu.dispatch(_ws(spec), lens, o)
    assert np.array_equal(g["edges"], o.edges)
    assert np.array_equal(g["bucket_a"], o.bucket) and np.array_equal(g["bucket_b"], o.bucket)
    assert np.array_equal(g["perm"], o.perm)
    assert np.array_equal(g["seg_off"][:len(o.seg_off)], o.seg_off)
    assert np.array_equal(g["plan_rb"], o.req_batch) and np.array_equal(g["plan_rr"], o.req_row)
    for f in ("segment", "start", "end", "n", "max_input_len", "pitch", "token_sum", "footprint",
              "out_offset", "row_base"):
        assert np.array_equal(g["batches"][f], o.batches[f]), f
    assert np.array_equal(g["rb"], d.req_batch) and np.array_equal(g["rr"], d.req_row)
    assert np.array_equal(g["emit"], d.emit_order) and np.array_equal(g["bemit"], d.batch_emit)
    m = int(o.summary["packed_elems"])
    assert np.array_equal(g["tokens"], o.out_tokens[:m]) and np.array_equal(g["mask"], o.out_mask[:m])
    if "chunked_tokens" in g:
        assert np.array_equal(g["chunked_tokens"], g["tokens"])
        assert np.array_equal(g["chunked_mask"], g["mask"])
    if "tokens_u" in g:
        assert np.array_equal(g["tokens_u"], g["tokens"]) and np.array_equal(g["mask_u"], g["mask"])
    assert int(g["summary"]["n_max"]) == int(ref["n_max"])


def test_dispatch_requires_dispatch_sizing():
    lib = N.load()
    ctx = N.Context(0, 16, 64, 2)
    prm = N.make_params(l_max=64, n_classes=2, policies=[0, 1], split_threshold=0.5, adjust=True,
                        max_passes=0, n_max=0, kv_bytes_per_token=2, current_safe=1000, pledged=0,
                        accounting=0, truncate=True, pad_id=0, dispatch=False)
    buf = torch.zeros(1024, dtype=torch.int32, device=DEV)
    rc = lib.bs_dispatch(ctx.ptr, _p(buf), _p(buf), 4, C.byref(prm), _p(buf), 4, _p(buf), _p(buf),
                         _p(buf), _p(buf), _p(buf), None)
    assert rc == N.BS_ERR_INVALID_ARG
    assert b"dispatch" in lib.bs_last_error(ctx.ptr)
    ctx.close()
