"""Build libme.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels
with the repo snapshot to the GPU box)."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libme.so"
LIB_CHECKED = PKG / "libme_checked.so"  # device-side bounds assertions (-DME_CHECKS), for tests
SOURCES = ["me_space.cpp", "me_kernels.cu", "me_fused.cu", "me_digest.cu", "me_rank.cu", "me_abi.cu"]
HEADERS = ["me_space.hpp", "me_kernels.cuh", "me_dev.cuh"]


def nccl_root() -> Path:
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        p = Path(list(spec.submodule_search_locations)[0])
        if (p / "include" / "nccl.h").exists():
            return p
    raise RuntimeError("NCCL headers (nvidia.nccl) not found")


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (Path(c).exists() or c == "nvcc"):
            return c
    return "nvcc"


def stale(lib: Path = LIB) -> bool:
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "me.h", Path(__file__)]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> Path:
    lib = LIB_CHECKED if checked else LIB
    if not force and not stale(lib):
        return lib
    nr = nccl_root()
    cmd = [nvcc(), "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", "-lineinfo",
           "-gencode", "arch=compute_100a,code=sm_100a",
           "-Xptxas", "-v" if verbose else "-O3",
           "-I", str(ROOT / "include"), "-I", str(nr / "include"),
           *[str(CSRC / s) for s in SOURCES],
           "-L", str(nr / "lib"), "-l:libnccl.so.2", f"-Xlinker=-rpath={nr / 'lib'}",
           *(["-DME_CHECKS"] if checked else []),
           "-o", str(lib) + ".tmp"]
    subprocess.check_call(cmd)
    os.replace(str(lib) + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
