"""Build recipes for the in-tree native libraries (no JIT cache; the built
.so files travel to the GPU box with the repo snapshot).

    lib/libspamm_gpu.so   sm_100a kernels + the C ABI (include/spamm_gpu.h,
                          include/spamm_synth.h); cudart linked statically so
                          the library loads (and reports "no device") on a
                          machine without a GPU.
    lib/libspamm_ec.so    C++ drop-in of the reference API (include/spamm/*.hpp)
                          over the C ABI.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "lib"
OBJ = ROOT / "build" / "obj"
INCLUDE = ROOT / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
    "-Xcompiler", "-Wno-deprecated-declarations", "-Xcompiler", "-ffp-contract=off",
    f"-I{INCLUDE}", f"-I{CSRC}",
]
CU_SOURCES = ["norms.cu", "matrix.cu", "cse.cu", "spamm.cu", "synth.cu", "truncate.cu", "algebra.cu", "purify.cu", "bstream.cu", "comm.cu"]
HEADERS = list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h")) + [Path(__file__)]

CXX = os.environ.get("CXX", "g++")
DROPIN_SOURCES = ["dropin/quadtree.cpp", "dropin/multiply.cpp", "dropin/error_control.cpp",
                  "dropin/matrix_market.cpp", "dropin/experiment.cpp",
                  "dropin/purification.cpp", "dropin/runtime.cpp", "dropin/distributed.cpp"]


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def _run(cmd):
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("build failed: " + " ".join(map(str, cmd)))
    return res


def build_gpu(verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    LIB.mkdir(parents=True, exist_ok=True)
    jobs = []
    objs = []
    for src in CU_SOURCES:
        s = CSRC / src
        o = OBJ / (s.stem + ".o")
        objs.append(o)
        if _stale(o, [s] + HEADERS):
            jobs.append([NVCC] + NVCC_FLAGS + ["-c", str(s), "-o", str(o)])
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for r in ex.map(_run, jobs):
            if verbose:
                print(r.stdout + r.stderr)
    out = LIB / "libspamm_gpu.so"
    if _stale(out, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", str(out)] + [str(o) for o in objs])
    return out


def build_dropin() -> Path:
    LIB.mkdir(parents=True, exist_ok=True)
    srcs = [CSRC / s for s in DROPIN_SOURCES]
    out = LIB / "libspamm_ec.so"
    hdrs = list((INCLUDE / "spamm").glob("*.hpp")) + list((CSRC / "dropin").glob("*.hpp")) + HEADERS
    gpu = LIB / "libspamm_gpu.so"
    if _stale(out, srcs + hdrs + [gpu]):
        _run([CXX, "-std=c++20", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
              f"-I{INCLUDE}", "-o", str(out)] + [str(s) for s in srcs] +
             [f"-L{LIB}", "-lspamm_gpu", "-Wl,-rpath,$ORIGIN"])
    return out


def build_all(verbose: bool = False):
    build_gpu(verbose)
    if all((CSRC / s).exists() for s in DROPIN_SOURCES):
        build_dropin()


if __name__ == "__main__":
    build_all(verbose="-v" in sys.argv)
    print("built", sorted(p.name for p in LIB.glob("*.so")))
