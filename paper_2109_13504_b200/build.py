"""Build libmgp.so in-tree for sm_100a (the .so travels with the repo snapshot).

    python -m paper_2109_13504_b200.build [--force]
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libmgp.so")
SOURCES = [os.path.join(CSRC, "mgp_abi.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("mgp_kernels.cuh", "mgp_device.cuh", "mgp_prefix.cuh")] + [
    os.path.join(ROOT, "include", "megopolis_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=false",  # float64 reductions must round exactly like numpy (no FMA contraction)
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-warn-spills",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(p) > t for p in DEPS)


# measurement probe (bench.py's L2 / HBM read peaks; not on the product path)
PROBE_SRC = os.path.join(CSRC, "mgp_probe.cu")
PROBE_OUT = os.path.join(HERE, "libmgp_probe.so")


def _nvcc(src, out, verbose):
    cmd = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", out + ".tmp", src]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)


def build_probe(force: bool = False, verbose: bool = False) -> str:
    if force or not os.path.exists(PROBE_OUT) or os.path.getmtime(PROBE_SRC) > os.path.getmtime(PROBE_OUT):
        _nvcc(PROBE_SRC, PROBE_OUT, verbose)
    return PROBE_OUT


def build(force: bool = False, verbose: bool = False) -> str:
    build_probe(force, verbose)
    if not force and not needs_build():
        return OUT
    _nvcc(SOURCES[0], OUT, verbose)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
