"""In-tree build of the sm_100a C-ABI library (libbucketserve.so).

    python -m paper_2507_17120_b200.build [--force] [--verbose]

nvcc cross-compiles for B200 without a GPU (-gencode arch=compute_100a,code=sm_100a).
The .so is written next to this file under _lib/, so it travels to the GPU box
with the repo snapshot (it is git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import argparse
import glob
import hashlib
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OUT_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(OUT_DIR, "libbucketserve.so")
STAMP = os.path.join(OUT_DIR, "libbucketserve.stamp")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
              "-Xptxas", "-v", "-cudart", "static"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _digest() -> str:
    h = hashlib.sha256()
    for f in sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [
            os.path.join(INCLUDE, "bucketserve.h"), __file__]:
        with open(f, "rb") as fh:
            h.update(f.encode())
            h.update(fh.read())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> str:
    dig = _digest()
    if not force and os.path.exists(LIB) and os.path.exists(STAMP):
        with open(STAMP) as fh:
            if fh.read().strip() == dig:
                return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    host_cc = shutil.which("g++", path="/usr/bin") or "g++"
    base = [nvcc(), *ARCH, *NVCC_FLAGS, "-ccbin", host_cc, "-I", INCLUDE, "-I", CSRC]
    obj_dir = os.path.join(OUT_DIR, "obj")
    os.makedirs(obj_dir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
        r = subprocess.run(base + ["-c", "-o", obj, src], capture_output=True, text=True)
        return src, obj, r

    # one nvcc per translation unit, in parallel, then one link
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(sources()), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, sources()))
    log = []
    for src, obj, r in results:
        log.append(r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {os.path.basename(src)}")
    res = subprocess.run(base + ["-shared", "-o", LIB + ".tmp"] + [o for _, o, _ in results] + ["-ldl"],
                         capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking libbucketserve.so")
    res.stderr = "".join(log) + res.stderr
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(LIB + ".tmp", LIB)
    with open(os.path.join(OUT_DIR, "ptxas.log"), "w") as fh:
        fh.write(res.stderr)
    with open(STAMP, "w") as fh:
        fh.write(dig)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))
