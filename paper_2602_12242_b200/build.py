"""Build libmagnex_b200.so in-tree with nvcc for sm_100a (no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmagnex_b200.so")
SOURCES = ["api.cu", "stencil.cu", "demag.cu", "demag_fast.cu", "newell.cu", "yz_pipe.cu", "x_warp.cu", "longy.cu", "fno.cu", "cufft_compare.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-ffp-contract=off", "-Xptxas", "-v"]


def build(verbose: bool = False) -> str:
    newest_dep = max([os.path.getmtime(os.path.join(CSRC, h)) for h in os.listdir(CSRC)
                      if h.endswith((".cuh", ".h", ".inc"))] +
                     [os.path.getmtime(os.path.join(HERE, "..", "include", "magnex_b200.h"))])
    objs, todo = [], []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(CSRC, s.replace(".cu", ".o"))
        if not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(src), newest_dep):
            todo.append((s, src, obj))
        objs.append(obj)

    def compile_one(item):
        s, src, obj = item
        return s, subprocess.run([NVCC, *FLAGS, "-c", src, "-o", obj], capture_output=True, text=True)

    # the translation units are independent: compile them concurrently
    with ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 1))) as ex:
        for s, r in ex.map(compile_one, todo):
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {s}")
            if verbose:
                sys.stderr.write(r.stderr)
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs, "-o", LIB,
           "-lcufft", "-Xcompiler", "-fPIC"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
