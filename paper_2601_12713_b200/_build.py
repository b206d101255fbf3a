"""Builds libb2l.so in-tree (nvcc, sm_100a only) -- the .so travels to the GPU box
with the repo snapshot (git-ignored, not gpurun-ignored)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libb2l.so")
SOURCES = ["b2l_api.cu", "b2l_hash.cu", "b2l_hash_k2.cu", "b2l_analyze.cu", "b2l_audit.cu", "b2l_ingest.cpp",
           "b2l_capture.cu", "b2l_multi.cu"]
OMPT_LIB = os.path.join(PKG, "libb2l_ompt.so")  # OMPT tool glue over libb2l's capture ABI
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _sources():
    return [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]


def _headers():
    hs = [os.path.join(ROOT, "include", "b2l.h")]
    hs += [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return hs


def up_to_date() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(OMPT_LIB):
        return False
    t = os.path.getmtime(LIB)
    deps = _sources() + _headers() + [__file__, os.path.join(CSRC, "b2l_ompt.cpp")]
    return all(os.path.getmtime(p) <= t for p in deps) and os.path.getmtime(OMPT_LIB) >= t


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "--extended-lambda", "--shared", "-Xcompiler", "-fPIC",
           "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           "-o", LIB + ".tmp", *_sources(), "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libb2l.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(LIB + ".tmp", LIB)
    build_ompt()
    return LIB


def build_ompt() -> str:
    """libb2l_ompt.so: ompt_start_tool + the two EMI callbacks, linked against libb2l.so."""
    src = os.path.join(CSRC, "b2l_ompt.cpp")
    cuda = os.path.dirname(os.path.dirname(NVCC))
    cmd = ["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(cuda, "include"), "-o", OMPT_LIB + ".tmp", src, "-L", PKG, "-lb2l",
           "-L", os.path.join(cuda, "lib64"), "-lcudart", "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("g++ failed building libb2l_ompt.so")
    os.replace(OMPT_LIB + ".tmp", OMPT_LIB)
    return OMPT_LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
