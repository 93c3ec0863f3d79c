"""Build libpdilqr.so in-tree with nvcc for sm_100a (B200).  No JIT cache: the .so lives next to
this file so it travels with the repository snapshot to the GPU box."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpdilqr.so")
SOURCES = [os.path.join(CSRC, "pdilqr.cu")]
HEADERS = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))] + \
          [os.path.join(ROOT, "include", "pdilqr.h")]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-shared",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-warn-spills",
]
# PDILQR_FAST_BUILD=1: nvcc --split-compile (all host cores, ~3x faster build) for development
# iterations only -- measured 9% slower SRBD kernels on B200, so the default build does not use it.
if os.environ.get("PDILQR_FAST_BUILD") == "1":
    NVCC_FLAGS.append("--split-compile=0")


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


PARTS = (1, 2, 3, 4, 5)  # see the partition comment at the top of csrc/pdilqr.cu


def build(force: bool = False, verbose: bool = False, extra: list[str] | None = None) -> str:
    """Compile the five parts of pdilqr.cu as separate translation units in parallel (host ABI,
    f32 / f64 kernels for n, m <= 16, f32 / f64 large-n kernels) and link them into one .so.
    Same code and flags as a single-TU build (PDILQR_PART=0), a fraction of the wall time."""
    if not force and not needs_build():
        return LIB
    import concurrent.futures as cf
    import tempfile
    tmp = tempfile.mkdtemp(prefix="pdilqr_build_")
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    flags = [f for f in NVCC_FLAGS if f != "-shared"] + list(extra or [])
    objs = [os.path.join(tmp, f"part{k}.o") for k in PARTS]

    def compile_part(k, obj):
        # one wrapper file per part: nvcc names anonymous namespaces after the main file, so the
        # parts must not share a file name
        src = os.path.join(tmp, f"pdilqr_part{k}.cu")
        with open(src, "w") as f:
            f.write(f'#define PDILQR_PART {k}\n#include "pdilqr.cu"\n')
        cmd = [nvcc(), *flags, *inc, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)

    with cf.ThreadPoolExecutor(len(PARTS)) as ex:
        for f in [ex.submit(compile_part, k, o) for k, o in zip(PARTS, objs)]:
            f.result()
    link = [nvcc(), "-shared", "-Xcompiler", "-fPIC", "-gencode", "arch=compute_100a,code=sm_100a",
            *objs, "-o", LIB + ".tmp"]
    if verbose:
        print(" ".join(link), file=sys.stderr)
    subprocess.check_call(link)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, extra=["-Xptxas", "-v"] if "-v" in sys.argv else None)
    print(LIB)
