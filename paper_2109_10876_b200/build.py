"""Build recipe for libtmd_gpu.so (sm_100a only, in-tree).

`python -m paper_2109_10876_b200.build` or `__graft_entry__.build()` compiles
the CUDA engine with nvcc straight into the package directory, so the shared
object travels with the repo snapshot to the GPU box. No torch extension
machinery: the library is plain CUDA C++ behind a C ABI (include/tmd_gpu.h).
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libtmd_gpu.so"

SOURCES = [CSRC / "tmd_engine.cu", CSRC / "tmd_host.cpp"]
HEADERS = [ROOT / "include" / "tmd_gpu.h", *sorted(CSRC.glob("*.cuh")), *sorted(CSRC.glob("*.h"))]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2",
    "-Xptxas", "-v",
    "-shared",
]


def nccl_dir():
    """The NCCL that torch loads (pip nvidia-nccl): same library, one copy per
    process. None: build without the native multi-GPU loop."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations or []) if spec else []:
        d = Path(base) / "nccl"
        if (d / "include" / "nccl.h").exists() and (d / "lib" / "libnccl.so.2").exists():
            return d
    return None


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in SOURCES + HEADERS + [Path(__file__)])


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not stale():
        return LIB
    extra = ["-DTMD_NO_NCCL"]
    nd = nccl_dir()
    if nd is not None:
        lib = nd / "lib"
        extra = [f"-I{nd / 'include'}", f"-L{lib}", "-l:libnccl.so.2",
                 "-Xlinker", f"-rpath,{lib}"]
    if os.environ.get("TMD_RDC") == "1":  # (experiment: relocatable device code)
        extra = ["-rdc=true", *extra, "-lcudadevrt"]
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-o", str(LIB), *map(str, SOURCES)]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True)
    log = res.stdout + res.stderr
    (PKG / "build.log").write_text(" ".join(cmd) + "\n" + log)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{log[-4000:]}")
    if verbose:
        print(log)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
