"""Build the C-ABI shared library libdls_b200.so in-tree (sm_100a only).

    python -m paper_1709_02599_b200.build [--verbose]

nvcc cross-compiles without a GPU; the CUDA runtime is linked statically so the
library loads (and its host-side calls run) on machines without a driver.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libdls_b200.so")
# the same sources with the kernels' internal invariants compiled in (DLS_CHECK):
# tests load it through DLS_LIB to look for bad indices / pool races
LIB_CHECKED = os.path.join(HERE, "libdls_b200_checked.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cpp")) + glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = sources() + glob.glob(os.path.join(HERE, "csrc", "*.h")) + [os.path.join(ROOT, "include", "dls_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    target = out or LIB
    if not force and (out is None or out == LIB_CHECKED) and not _stale(target):
        return target
    tmp = target + ".tmp%d" % os.getpid()
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "--cudart", "static", "-diag-suppress", "177", "-I", os.path.join(ROOT, "include"),
           *["-D" + d for d in defines], "-o", tmp, *sources()]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    if verbose:
        sys.stderr.write(r.stdout + r.stderr)
    os.replace(tmp, target)
    return target


def build_checked(force: bool = False) -> str:
    return build(force=force, out=LIB_CHECKED, defines=("DLS_CHECKS",))


if __name__ == "__main__":
    if "--checked" in sys.argv:
        print(build_checked(force=True))
    else:
        print(build(force=True, verbose="--verbose" in sys.argv))
