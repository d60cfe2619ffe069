"""Builds libtpgen.so in-tree for sm_100a (nvcc; no JIT, no torch extension)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtpgen.so")
SOURCES = ["engine.cu", "planner.cpp", "abi.cpp", "tpcover.cpp", "normalize.cpp"]
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".h", ".cuh")))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "--expt-relaxed-constexpr",
    "-shared",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "tpgen.h"))
    deps.append(__file__)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, variant: str = "", defines=()) -> str:
    """Builds libtpgen.so (or, for A/B experiments, libtpgen_<variant>.so with extra -D defines;
    loaded when TPGEN_LIB_VARIANT=<variant>)."""
    lib = LIB if not variant else os.path.join(HERE, f"libtpgen_{variant}.so")
    if not force and not variant and not _stale():
        return LIB
    tmp = lib + f".tmp{os.getpid()}"
    dbg = ["-DTPGEN_KERNEL_DEBUG"] if os.environ.get("TPGEN_KERNEL_DEBUG") else []
    dbg += [f"-D{d}" for d in defines]
    cmd = [NVCC] + FLAGS + dbg + (["-Xptxas", "-v"] if verbose else []) + \
        [os.path.join(CSRC, f) for f in SOURCES] + ["-o", tmp]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc build of libtpgen.so failed")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), "")
    defs = [a[2:] for a in sys.argv if a.startswith("-D")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, variant=var, defines=defs))
