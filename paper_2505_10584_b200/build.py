"""Build libaqb.so (all hand-written sm_100a kernels + the C-ABI) in-tree.

``python -m paper_2505_10584_b200.build`` or ``__graft_entry__.build()``.
nvcc cross-compiles for sm_100a without a GPU; the .so lands next to this
file (git-ignored, but it travels to the GPU box with the gpurun snapshot).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB = os.path.join(HERE, "libaqb.so")
SOURCES = ["host.cu", "elementwise.cu", "gemm.cu", "attention.cu", "peer.cu", "fp32.cu", "tiles.cu"]
HEADERS = ["ptx.cuh", "host.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-cudart", "static",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; cannot build libaqb.so")


def _defines_file() -> str:
    return os.path.join(HERE, "_obj", "defines.txt")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    try:  # a library built with other AQB_BUILD_DEFINES (e.g. a trace build) is stale
        with open(_defines_file()) as fh:
            if fh.read() != os.environ.get("AQB_BUILD_DEFINES", ""):
                return True
    except OSError:
        pass
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(INCLUDE, "aqb.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def header_hash() -> str:
    """sha256 of include/aqb.h — compiled in as aqb_build_id() and checked at load time."""
    import hashlib

    with open(os.path.join(INCLUDE, "aqb.h"), "rb") as fh:
        return hashlib.sha256(fh.read()).hexdigest()


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile each translation unit in parallel (``nvcc -c``), then link the shared library."""
    from concurrent.futures import ThreadPoolExecutor

    if not force and not _stale():
        return LIB
    objdir = os.path.join(HERE, "_obj")
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f not in ("-shared", "-cudart", "static")]
    define = f'-DAQB_HEADER_HASH="{header_hash()}"'
    extra = os.environ.get("AQB_BUILD_DEFINES", "").split()  # e.g. -DAQB_GEMM_TRACE (measurement builds)

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [nvcc(), *compile_flags, define, *extra, "-I", INCLUDE, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src} ({res.returncode}):\n{res.stderr[-8000:]}")
        return obj

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB + ".tmp"
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", *objs, "-o", tmp]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed ({res.returncode}):\n{res.stderr[-8000:]}")
    os.replace(tmp, LIB)
    with open(_defines_file(), "w") as fh:
        fh.write(os.environ.get("AQB_BUILD_DEFINES", ""))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
