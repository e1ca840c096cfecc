"""Captured window graphs: a double-buffered loop alternating two input sets replays one
graph per set (WindowScheduler keeps up to four, least recently used dropped), and every
replay equals an eager run on the same inputs — outcomes, batches and packed bytes."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2507_17120_b200 import workloads as W  # noqa: E402
from paper_2507_17120_b200.window import WindowScheduler  # noqa: E402


def _window(cfg_name, n, seed):
    cfg, lens, cls = W.make_window(cfg_name, n=n, seed=seed)
    tok_off, tokens = W.token_store(lens)
    dev = torch.device("cuda", 0)
    return cfg, [torch.as_tensor(a).to(dev) for a in (lens, cls, tok_off, tokens)]


def _snapshot(res):
    h = res.to_host()
    m = int(h["summary"]["packed_elems"])
    return (h["req_batch"].copy(), h["req_row"].copy(), h["batches"].copy(),
            h["out_tokens"][:m].copy(), h["out_mask"][:m].copy())


def _equal(a, b):
    for x, y in zip(a, b):
        if x.dtype.names:
            for f in x.dtype.names:
                u, v = x[f], y[f]
                if f == "waste":
                    u, v = u.view(np.uint64), v.view(np.uint64)
                assert np.array_equal(u, v), f
        else:
            assert np.array_equal(x, y)


@pytest.mark.parametrize("cfg_name,n", [("c2", 30000), ("c1", 1000)])
def test_alternating_inputs_replay_their_own_graphs(cfg_name, n):
    cfg, set_a = _window(cfg_name, n, 5)
    _, set_b = _window(cfg_name, n, 6)
    s = WindowScheduler(max_requests=n, max_seq_len=cfg.l_max, n_classes=cfg.n_classes,
                        policies=cfg.policies, split_threshold=cfg.theta, adjust=cfg.adjust,
                        buckets=cfg.init_edges, kv_bytes_per_token=cfg.kvpt,
                        current_safe=cfg.current_safe, pack_capacity=n * cfg.l_max,
                        device=torch.device("cuda", 0))
    want = {}
    for name, ins in (("a", set_a), ("b", set_b)):
        want[name] = _snapshot(s.schedule(*ins))
    for step in range(6):
        name, ins = ("a", set_a) if step % 2 == 0 else ("b", set_b)
        _equal(_snapshot(s.schedule(*ins, graph=True)), want[name])
    assert len(s._graphs) == 2
    s.close()


def test_graph_cache_is_bounded():
    cfg, base = _window("c2", 5000, 9)
    s = WindowScheduler(max_requests=5000, max_seq_len=cfg.l_max, n_classes=cfg.n_classes,
                        policies=cfg.policies, kv_bytes_per_token=cfg.kvpt,
                        current_safe=cfg.current_safe, pack_capacity=5000 * cfg.l_max,
                        device=torch.device("cuda", 0))
    sets = [[t.clone() for t in base] for _ in range(6)]  # six distinct input buffers
    want = _snapshot(s.schedule(*base))
    for ins in sets:
        _equal(_snapshot(s.schedule(*ins, graph=True)), want)
    assert len(s._graphs) == WindowScheduler._GRAPHS
    s.close()
