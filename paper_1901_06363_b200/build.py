"""In-tree build of the native library (libgeodock_b200.so).

nvcc compiles the sm_100a kernels with ``-fmad=false`` (the fp64 recipe
must not be contracted into DFMA); g++ compiles the host runtime with
``-ffp-contract=off``.  The result lands next to this file so it travels
to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libgeodock_b200.so"
BUILD = PKG / "_build"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
HOST_SRCS = ["capi.cpp", "prep.cpp", "orient.cpp", "synth.cpp", "analysis.cpp", "planner.cpp"]
# flex_cp.cu / rigid_cp.cu compile flex.cu / rigid.cu again for the compact
# voxel-record format (kernels.h).
CUDA_SRCS = ["rigid.cu", "flex.cu", "rigid_cp.cu", "flex_cp.cu", "pocket_index.cu", "prep.cu"]
HEADERS = ["kernels.h", "device_common.cuh", "prep.hpp", "orient.hpp"]


def _run(cmd: list[str]) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd)}")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


# -D flags shared by device and host objects (layout knobs such as
# GD_VOX_INLINE must agree on both sides); GD_NVCC_EXTRA is device-only.
DEFS = os.environ.get("GD_DEFS", "").split()


def build(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    inc = ["-I", str(ROOT / "include"), "-I", str(CSRC)]
    hdrs = [CSRC / h for h in HEADERS] + [ROOT / "include" / "geodock_b200.h"]
    objs, jobs = [], []
    for src in CUDA_SRCS:
        obj = BUILD / (src + ".o")
        deps = [CSRC / src] + hdrs + ([CSRC / src.replace("_cp", "")] if "_cp" in src else [])
        if force or _stale(obj, deps):
            jobs.append([NVCC, *ARCH, "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
                         *os.environ.get("GD_NVCC_EXTRA", "").split(), *DEFS,
                         "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3", *inc,
                         "-c", str(CSRC / src), "-o", str(obj)])
        objs.append(obj)
    for src in HOST_SRCS:
        obj = BUILD / (src + ".o")
        if force or _stale(obj, [CSRC / src] + hdrs):
            jobs.append(["g++", "-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-Wall", *DEFS,
                         "-I/usr/local/cuda/include", *inc, "-c", str(CSRC / src), "-o", str(obj)])
        objs.append(obj)
    # The translation units are independent: compile them side by side (the
    # two flex TUs dominate, ~100 s each).
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as pool:
        list(pool.map(_run, jobs))
    if force or _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB),
              *map(str, objs), "-lpthread"])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
