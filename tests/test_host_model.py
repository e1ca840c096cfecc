"""Host-side scalars of the path (memory model, n_max) — restated from the
reference's own known-answer tests (test_memory_model.py, test_batch_controller.py)."""

import math

import numpy as np
import pytest

from oracle import cpu
from paper_2507_17120_b200 import (ConfigError, GpuConfig, ModelConfig, kv_footprint_exact,
                                   kv_footprint_padded, max_safe_batch, safe_memory,
                                   token_budget, waste_ratio)
from paper_2507_17120_b200 import workloads as W

GIB = 2 ** 30


def test_kv_bytes_and_footprint_reference_values():
    m = ModelConfig(40, 40, 128, 2, 4096)            # test_memory_model.py:15-19
    assert kv_footprint_padded(m, 1024, 8) == 6_710_886_400
    assert kv_footprint_padded(m, 1024, 0) == 0
    with pytest.raises(ValueError):
        kv_footprint_padded(ModelConfig(8, 8, 64, 2, 2048), 4096, 1)
    assert kv_footprint_exact(ModelConfig(1, 1, 1, 2, 4096), [100, 200]) == 1200


def test_safe_memory_and_token_budget_reference_values():
    gpu = GpuConfig(40 * GIB, 30 * GIB, 0.10)           # test_memory_model.py:141-160
    assert safe_memory(gpu) == 9_663_676_416
    assert token_budget(ModelConfig(32, 32, 128, 2, 8192), gpu) == 18_432
    assert safe_memory(GpuConfig(8 * GIB, 8 * GIB)) == 0
    # scenario preset: 40 GiB / 26 GiB, 13B-like (test_config.py:135-139)
    assert safe_memory(GpuConfig(40 * GIB, 26 * GIB)) == 13_529_146_982


def test_waste_ratio_reference_values():
    assert waste_ratio([1024, 256, 256, 256]) == pytest.approx(0.5625)
    assert waste_ratio([512, 512, 512]) == 0.0
    with pytest.raises(ValueError):
        waste_ratio([])
    with pytest.raises(ValueError):
        waste_ratio([10, 0, 20])


def test_max_safe_batch_brute_force():
    rng = np.random.default_rng(7)
    for _ in range(500):
        lengths = rng.integers(1, 5000, size=int(rng.integers(0, 64))).tolist()
        budget = int(rng.integers(0, 60_000))
        best = max([k for k in range(len(lengths) + 1) if sum(lengths[:k]) <= budget])
        assert max_safe_batch(lengths, budget) == best


def test_config_validation():
    with pytest.raises(ConfigError):
        ModelConfig(0, 8, 64, 2, 2048)
    with pytest.raises(ConfigError):
        ModelConfig(8, 8, 64, 3, 2048)
    with pytest.raises(ConfigError):
        GpuConfig(total_mem=10, model_mem=20)


def _py_n_max(total, sum_len, safe, kvpt):
    """BatchController.current_n_max, literally (batch_controller.py:100-104)."""
    if total == 0:
        return 1
    mean_len = sum_len / total
    return max(1, int((safe // kvpt) // mean_len))


def test_n_max_matches_python_float_semantics():
    """The device/oracle n_max reproduces CPython int // float on adversarial values."""
    rng = np.random.default_rng(3)
    for _ in range(20000):
        total = int(rng.integers(0, 1 << 26))
        sum_len = int(rng.integers(0, total * 131071 + 1)) if total else 0
        if total and sum_len == 0:
            continue
        kvpt = int(rng.choice([2, 4096, 131072, 524288, 819200]))
        safe = int(rng.integers(0, 200 * GIB))
        assert cpu.n_max(total, sum_len, safe, kvpt) == _py_n_max(total, sum_len, safe, kvpt)


def test_n_max_on_integer_boundaries():
    """Means chosen so token_budget / mean sits on or next to an integer (the cases where
    float rounding of the mean decides the floor); the oracle vs the literal Python."""
    rng = np.random.default_rng(4)
    for kvpt, safe in ((524288, 160_417_028_505), (131072, 147_600_000_000), (819200, 13_529_146_982)):
        budget = safe // kvpt
        for _ in range(3000):
            n = int(rng.choice([1, 3, 7, 999_983, int(rng.integers(1, 1 << 26))]))
            k = int(rng.integers(1, 5000))
            s0 = budget * n // k
            for s in (s0 - 1, s0, s0 + 1, -(-budget * n // k)):
                if s >= n:
                    assert cpu.n_max(n, s, safe, kvpt) == _py_n_max(n, s, safe, kvpt)


def test_baseline_config_constants():
    assert W.CONFIGS["c2"].current_safe == 160_417_028_505
    assert W.CONFIGS["c2"].kvpt == 524_288
    assert W.CONFIGS["c4"].kvpt == 131_072
    assert W.CONFIGS["c4"].current_safe == 147_600_000_000
    assert W.CONFIGS["c2"].current_safe // W.CONFIGS["c2"].kvpt == 305_971
    assert W.CONFIGS["c1"].current_safe == math.floor(0.9 * 14 * GIB)


def test_token_store_host_and_device_agree():
    torch = pytest.importorskip("torch")
    _, lens, _ = W.make_window("c2", n=2000, seed=5)
    o1, t1 = W.token_store(lens, seed=3)
    o2, t2 = W.token_store_device(torch.as_tensor(lens), seed=3)
    assert np.array_equal(o1, o2.numpy()) and np.array_equal(t1, t2.numpy())
    assert (o1[:-1] % 4 == 0).all()
