"""bench.py --impl reference on the host (no GPU): one JSON line with the contract's
keys, the same config as the B200 arm, and — when the unmodified reference package is
importable (/root/reference or its baseline/_ref install) — the Python reference timed
beside the oracle port on one core."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _run(*extra):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
           "--requests", "20000", "--steps", "2", "--warmup", "3", *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    from oracle import ref_compose
    d = _run()
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["same_config"] is True and d["config"]["requests_per_step"] == 20000
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    rp = d["reference_python"]
    if not ref_compose.available():
        pytest.skip("reference package not importable here")
    assert rp["value"] > 0 and rp["cores"] == 1 and rp["requests"] == 20000
    assert rp["nproc"] >= 1 and rp["batches"] > 0


def test_reference_arm_without_python_leg():
    d = _run("--no-reference-python")
    assert "reference_python" not in d
