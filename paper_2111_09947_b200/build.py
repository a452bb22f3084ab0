"""Build the CUDA library in-tree (sm_100a) — called by __graft_entry__.build()."""

from __future__ import annotations

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB_PATH = os.path.join(OUT_DIR, "libmaskmul_b200.so")
# host-only Matrix Market reader (include/maskmul_mmio.h): loads without a GPU
MMIO_LIB_PATH = os.path.join(OUT_DIR, "libmaskmul_mmio.so")
MMIO_SOURCE = "mmio_host.cpp"
SOURCES = ["maskmul_abi.cu"]


def headers() -> list[str]:
    """Every csrc/*.cuh (globbed, so a new header can never be missed by _stale)."""
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cuh"))


NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17", "--expt-relaxed-constexpr",
    "-shared", "-Xcompiler", "-fPIC",
]


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; cannot build the CUDA library")
    return cand


def _stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    deps = [os.path.join(CSRC, f) for f in SOURCES + headers()]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "maskmul_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build_mmio(force: bool = False, verbose: bool = False) -> str:
    src = os.path.join(CSRC, MMIO_SOURCE)
    hdr = os.path.join(os.path.dirname(HERE), "include", "maskmul_mmio.h")
    if (not force and os.path.exists(MMIO_LIB_PATH)
            and os.path.getmtime(MMIO_LIB_PATH) >= max(os.path.getmtime(src), os.path.getmtime(hdr))):
        return MMIO_LIB_PATH
    os.makedirs(OUT_DIR, exist_ok=True)
    tmp = MMIO_LIB_PATH + ".tmp"
    cmd = [shutil.which("g++") or "g++", "-O3", "-std=c++17", "-fPIC", "-shared", "-pthread",
           "-Wall", "-Wextra", "-o", tmp, src]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, MMIO_LIB_PATH)
    return MMIO_LIB_PATH


def build(force: bool = False, verbose: bool = False) -> str:
    build_mmio(force=force, verbose=verbose)
    if not force and not _stale():
        return LIB_PATH
    os.makedirs(OUT_DIR, exist_ok=True)
    tmp = LIB_PATH + ".tmp"
    cmd = [_nvcc(), *NVCC_FLAGS, "-o", tmp] + [os.path.join(CSRC, f) for f in SOURCES]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force=True, verbose=True))
