"""In-tree build of the sm_100a CUDA library (and, for tests, the C++ adapter).

The .so files land next to their sources so that gpurun's snapshot carries
them to the GPU box (they are git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd, cwd=None):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=cwd)


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_cuda(force=False, verbose_ptxas=False):
    """libcotten.so: every kernel + the C-ABI (include/cotten.h)."""
    out = os.path.join(PKG, "libcotten.so")
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(ROOT, "include", "cotten.h"))
    if not force and not _stale(out, deps):
        return out
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
           "-o", out, os.path.join(CSRC, "cotten_capi.cu")]
    if verbose_ptxas:
        cmd += ["-Xptxas", "-v"]
    _run(cmd)
    return out


def build_oracle():
    """oracle/: the C restatement and (when /root/reference exists) oracle/_ref."""
    _run(["make", "-s", "-C", os.path.join(ROOT, "oracle")])


def build_cpp_tests():
    """tests/cpp: the C++ adapter and the drop-in check binaries (needs the
    reference headers, so only where /root/reference exists)."""
    _run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")])


def build_all(force=False):
    build_cuda(force=force)
    build_oracle()
    build_cpp_tests()


if __name__ == "__main__":
    build_all(force=True)
