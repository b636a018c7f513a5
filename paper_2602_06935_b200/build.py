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
    deps += [os.path.join(ROOT, "include", h) for h in ("cotten.h", "cotten_encoder.h")]
    if not force and not _stale(out, deps):
        return out
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]
    if verbose_ptxas:
        flags += ["-Xptxas", "-v"]
    # one object per translation unit (rebuilt when its sources changed)
    objs = []
    for tu, tu_deps in (("cotten_capi.cu", [d for d in deps if not d.endswith("encoder.cu")
                                            and not d.endswith("cotten_encoder.h")]),
                        ("encoder.cu", [os.path.join(CSRC, "encoder.cu")] +
                         [os.path.join(ROOT, "include", h) for h in ("cotten.h", "cotten_encoder.h")])):
        obj = os.path.join(PKG, "build", tu.replace(".cu", ".o"))
        os.makedirs(os.path.dirname(obj), exist_ok=True)
        if force or _stale(obj, tu_deps):
            _run([NVCC, *flags, "-c", "-o", obj, os.path.join(CSRC, tu)])
        objs.append(obj)
    _run([NVCC, *ARCH, "-shared", "-o", out, *objs, "-lcublas"])
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
