"""Build the sm_100a library in-tree (nvcc cross-compiles; no GPU needed).

    python -m paper_2504_19449_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.environ.get("RSP_LIB") or os.path.join(PKG, "librsparse_b200.so")  # RSP_LIB: debug override (A/B of builds)
SOURCES = ["rsp_kernels.cu", "rsp_batch.cu", "rsp_offline.cu", "rsp_api.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "--diag-error", "20011,20014", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
         "-Xptxas", "-v", f"-I{os.path.join(ROOT, 'include')}"]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    headers = [f for f in os.listdir(CSRC) if f.endswith((".cuh", ".h", ".hpp"))]
    deps = [os.path.join(CSRC, f) for f in SOURCES + sorted(headers)]
    deps.append(os.path.join(ROOT, "include", "rsparse_b200.h"))
    if force or _stale(LIB, deps):
        extra = os.environ.get("RSP_NVCC_EXTRA", "").split()  # experiments, e.g. -DRSP_LDG=1
        cmd = [NVCC, *ARCH, *FLAGS, *extra, *[os.path.join(CSRC, f) for f in SOURCES], "-o", LIB]
        out = subprocess.run(cmd, capture_output=True, text=True)
        if out.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + out.stdout + out.stderr)
        with open(os.path.join(PKG, "ptxas_info.txt"), "w") as f:
            f.write(out.stderr)
        if verbose:
            print(out.stderr, file=sys.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
