"""The C-ABI from plain C (tests/c_abi_example.c): compiled with gcc against
include/bucketserve.h and the in-tree libbucketserve.so, run on the B200.  The
compile step also runs without a GPU (the link against the library is checked)."""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2507_17120_b200", "_lib")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _build(tmp_path):
    cc = shutil.which("gcc")
    if cc is None or not os.path.exists(os.path.join(LIBDIR, "libbucketserve.so")):
        pytest.skip("gcc or the built library is missing")
    exe = str(tmp_path / "c_abi_example")
    cmd = [cc, "-O2", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA, "include"), os.path.join(ROOT, "tests", "c_abi_example.c"),
           "-L", LIBDIR, "-lbucketserve", "-L", os.path.join(CUDA, "lib64"), "-lcudart",
           f"-Wl,-rpath,{LIBDIR}", f"-Wl,-rpath,{os.path.join(CUDA, 'lib64')}", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_example_compiles_and_links(tmp_path):
    exe = _build(tmp_path)
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_c_example_runs_on_b200(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr + r.stdout
    assert r.stdout.startswith("ok:")
