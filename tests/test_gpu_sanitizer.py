"""compute-sanitizer over small windows through every kernel of the path: memcheck
(out-of-bounds / misaligned accesses in every pack path's address arithmetic),
racecheck (shared-memory hazards in the scans, sorts and the dispatch kernel) and
synccheck (barriers / warp-synchronous primitives under divergence)."""
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool,args", [("memcheck", []), ("memcheck", ["--paths"]),
                                       ("racecheck", ["--small"]), ("synccheck", ["--small"]),
                                       ("racecheck", ["--k0"]), ("memcheck", ["--k0"])])
def test_sanitizer_clean(tool, args):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "9"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_window.py")] + args
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert re.search(r"SUMMARY: 0 (errors|hazards)", r.stdout + r.stderr), r.stdout[-3000:]
