"""Build libsesgd.so in-tree for sm_100a (nvcc; no JIT cache, the .so travels with the repo)."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsesgd.so")
LIB_CHECKED = os.path.join(PKG, "libsesgd_checked.so")  # -DSESGD_CHECKED: device bounds checks

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-fvisibility=hidden",
    "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "--expt-relaxed-constexpr", "-Xptxas", "-v", "-Wno-deprecated-gpu-targets",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))) \
        + [os.path.join(ROOT, "include", "sesgd.h")]


def up_to_date(lib: str = LIB) -> bool:
    return os.path.exists(lib) and all(os.path.getmtime(lib) >= os.path.getmtime(d) for d in deps())


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    lib = LIB_CHECKED if checked else LIB
    if not force and up_to_date(lib):
        return lib
    extra = ["-DSESGD_CHECKED"] if checked else []
    cmd = ["nvcc", *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-o", lib, *sources()]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(PKG, "build_checked.log" if checked else "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed (see {log}):\n{res.stderr[-4000:]}")
    if verbose:
        print(res.stderr)
    return lib


if __name__ == "__main__":
    build(force=True, verbose=True)
