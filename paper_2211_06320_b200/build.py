"""Build libfpe.so in-tree: nvcc for sm_100a (sm_100a only, no other targets).

    python -m paper_2211_06320_b200.build          # incremental
    python -m paper_2211_06320_b200.build --force
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
SO = os.path.join(HERE, "libfpe.so")
# experiments only: extra nvcc flags (e.g. -DFPE_EXP_NO_ZPOW) into a separately named library
EXTRA = os.environ.get("FPE_EXTRA_FLAGS", "").split()
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUFLAGS = EXTRA + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
           "--expt-relaxed-constexpr", "-I", os.path.join(HERE, "..", "include")]
SOURCES = ["api.cu", "kernels.cu", "sort.cu", "eval_tiled.cu", "precondition.cpp", "precondition_gpu.cu", "eval_mma.cu"]
HEADERS = ["fpe_internal.h", "fpe_hd.cuh", "fpe_polar.cuh", "fpe_math.cuh", "kernels.cuh", "log_table.h", "device_common.cuh", "sort.cuh", "eval_tiled.cuh", "tma.cuh", "mma_piece.cuh"]


def _newer(src: list[str], dst: str) -> bool:
    if not os.path.exists(dst):
        return True
    t = os.path.getmtime(dst)
    return any(os.path.getmtime(s) > t for s in src)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    deps = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(HERE, "..", "include", "fpe.h")]
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _newer([s] + deps, o):
            cmd = [NVCC] + ARCH + CUFLAGS + ["-c", s, "-o", o]
            if src.endswith(".cpp"):
                cmd = [NVCC, "-x", "cu"] + ARCH + CUFLAGS + ["-c", s, "-o", o]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            with open(o + ".ptxas.log", "w") as f:
                f.write(r.stdout + r.stderr)
            if verbose:
                sys.stderr.write(r.stderr)
    if force or _newer(objs, SO):
        cmd = [NVCC] + ARCH + ["-shared", "-o", SO] + objs + ["-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO)
