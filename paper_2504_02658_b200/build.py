"""Builds the sm_100a CUDA library in-tree: paper_2504_02658_b200/lib/libmilo_b200.so.

nvcc cross-compiles for sm_100a on a GPU-less host; the .so travels to the GPU
box with the repo snapshot.  No JIT cache, no torch extension machinery.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIB_DIR, "libmilo_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
         "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith((".cu", ".cuh")))


def needs_rebuild() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + [os.path.join(ROOT, "include", "milo_b200.h")]
    return any(os.path.getmtime(s) > t for s in deps)


def build(force: bool = False, verbose: bool = False, variant: str = "", defines=()) -> str:
    """Builds lib/libmilo_b200.so, or lib/variants/libmilo_b200_<variant>.so with
    extra -D defines (experiments; selected by MILO_B200_LIB_VARIANT)."""
    out = os.path.join(LIB_DIR, "variants", f"libmilo_b200_{variant}.so") if variant else LIB
    if not variant and not force and not needs_rebuild():
        return LIB
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = [NVCC, *ARCH, *FLAGS, *(f"-D{d}" for d in defines), "-I", os.path.join(ROOT, "include"), "-o", out + ".tmp",
           os.path.join(CSRC, "milo_b200.cu")]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = res.stdout + res.stderr
    with open(out + ".ptxas.log" if variant else os.path.join(LIB_DIR, "ptxas.log"), "w") as f:
        f.write(log)
    if res.returncode != 0:
        sys.stderr.write(log)
        raise RuntimeError("nvcc failed")
    if verbose:
        sys.stdout.write(log)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    if "--variant" in sys.argv:  # --variant NAME DEF1 DEF2 ...
        i = sys.argv.index("--variant")
        print(build(variant=sys.argv[i + 1], defines=sys.argv[i + 2:]))
        sys.exit(0)
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
