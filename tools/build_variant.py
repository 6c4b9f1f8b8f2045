"""Build a variant of libmagnex_b200.so with extra -D flags on some sources
(performance experiments; load it with MXB_LIB=variants/<name>/libmagnex_b200.so).

  python tools/build_variant.py <name> <source.cu>[,<source.cu>...] -DFOO=1 ...
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_12242_b200 import build as B  # noqa: E402

name, srcs, defs = sys.argv[1], sys.argv[2].split(","), sys.argv[3:]
B.build()
out = os.path.join(ROOT, "variants", name)
os.makedirs(out, exist_ok=True)
objs = []
for s in B.SOURCES:
    if s in srcs:
        o = os.path.join(out, s.replace(".cu", ".o"))
        cmd = [B.NVCC, *B.FLAGS, *defs, "-c", os.path.join(B.CSRC, s), "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.exit(r.stderr)
        objs.append(o)
    else:
        objs.append(os.path.join(B.CSRC, s.replace(".cu", ".o")))
lib = os.path.join(out, "libmagnex_b200.so")
subprocess.run([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs, "-o", lib,
                "-lcufft", "-Xcompiler", "-fPIC"], check=True)
print(lib)
