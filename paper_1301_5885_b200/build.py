"""Build libbipb.so in-tree (nvcc, sm_100a).  No torch involvement: the library is a
plain C-ABI shared object (include/bipb.h)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = [os.path.join(HERE, "csrc", f) for f in ("bipb.cu",)]
DEPS = SRC + sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [os.path.join(ROOT, "include", "bipb.h")]
LIB = os.path.join(HERE, "libbipb.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",            # every FMA is explicit in the source (bitwise-reproducible pairs)
    "-Xcompiler", "-fPIC", "-shared",
    "-I", os.path.join(ROOT, "include"),
]


def build(force: bool = False, extra: list[str] | None = None, out: str | None = None, verbose: bool = False) -> str:
    out = out or LIB
    if not force and extra is None and os.path.exists(out):
        t = os.path.getmtime(out)
        if all(os.path.getmtime(d) <= t for d in DEPS):
            return out
    cmd = [NVCC, *FLAGS, *(extra or []), "-o", out, *SRC, "-ldl"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
