"""bench.py's multi-rank path end to end on whatever GPUs the box has: `--gpus 2` spawns
two ranks itself (torch.distributed.run on 127.0.0.1); on a one-GPU box `--share-gpus`
runs both on it (gloo process group).  Checks the JSON contract of the line rank 0
prints: n_gpus, weak scaling over request shards, the C1 exchange timing, max-over-rank
timing, and the C5 strong-scaling split of one trace."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--no-e2e", "--no-cpu-baseline", *args]
    if torch.cuda.device_count() < 2:
        cmd.append("--share-gpus")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("collective", ["nccl", "peer"])
def test_two_ranks_weak_scaling(collective):
    if torch.cuda.device_count() < 2 and collective == "nccl":
        collective = "torch"  # NCCL needs one GPU per rank; the shared-GPU run uses gloo
    d = _bench("--requests", "200000", "--collective", collective)
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["config"]["requests_per_gpu"] == 200000
    assert d["c1"] is not None and d["c1"]["ms_per_window"] > 0
    assert d["gpu_launches"] > 0


def test_c5_trace_split_over_two_ranks():
    d = _bench("--config", "c5", "--requests", "500000")
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["requests_per_gpu"] == 500000
    assert d["value"] > 0
