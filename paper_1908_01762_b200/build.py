"""Compile libsisph.so (the sm_100a hot path + C ABI) in-tree with nvcc.

    python -m paper_1908_01762_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsisph.so")
SOURCES = ["sisph_engine.cu"]
DEPS = SOURCES + ["sisph_kernels.cuh", "sisph_device.cuh", "sisph_comm.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-v",
    "-shared",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    srcs = [os.path.join(CSRC, s) for s in DEPS] + [os.path.join(ROOT, "include", "sisph.h"), __file__]
    return any(os.path.getmtime(s) > t for s in srcs)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """out / defines: an A/B variant library (e.g. libsisph_v1.so built with -DSISPH_X),
    loaded by the binding when SISPH_LIB names it; the default build is libsisph.so."""
    lib_out = out or LIB
    if out is None and not force and not _stale():
        return LIB
    cmd = [NVCC, *FLAGS, *defines, "-I", os.path.join(ROOT, "include"), "-o", lib_out + ".tmp",
           *[os.path.join(CSRC, s) for s in SOURCES]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libsisph.so")
    if out is None:
        with open(os.path.join(HERE, "ptxas_info.txt"), "w") as f:
            f.write(r.stderr)
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(lib_out + ".tmp", lib_out)
    return lib_out


TOOLS = os.path.join(HERE, "libsisph_tools.so")


def build_tools(force: bool = False) -> str:
    """libsisph_tools.so: bench.py's measurement helpers (the FP32 ALU roof), not the hot path."""
    src = os.path.join(CSRC, "sisph_tools.cu")
    if not force and os.path.exists(TOOLS) and os.path.getmtime(TOOLS) >= max(os.path.getmtime(src),
                                                                               os.path.getmtime(__file__)):
        return TOOLS
    flags = [f for f in FLAGS if f not in ("-Xptxas", "-v")]
    cmd = [NVCC, *flags, "-o", TOOLS + ".tmp", src]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libsisph_tools.so")
    os.replace(TOOLS + ".tmp", TOOLS)
    return TOOLS


if __name__ == "__main__":
    # python -m paper_1908_01762_b200.build [--force] [--out PATH] [-DNAME ...]
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else None
    defs = [a for a in args if a.startswith("-D")]
    print(build(force="--force" in args, verbose=True, out=out, defines=defs))
