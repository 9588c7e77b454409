#!/usr/bin/env python
"""Dev tool: build libnmg.so variants with extra nvcc defines for A/B timing on the GPU box.
Usage: python tools/build_variant.py NAME -DFOO=1 [...]   -> paper_2603_01064_b200/variants/libnmg_NAME.so
Run with NMG_LIB=<that path>."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_01064_b200 import build as B  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    out = os.path.join(ROOT, "paper_2603_01064_b200", "variants")
    obj = os.path.join(out, "obj_" + name)
    os.makedirs(obj, exist_ok=True)
    objs, procs = [], []
    for src in B.sources():
        o = os.path.join(obj, os.path.basename(src) + ".o")
        objs.append(o)
        procs.append(subprocess.Popen([B.NVCC, *B.NVCC_FLAGS, *defs, "-c", src, "-o", o]))
    for p in procs:
        assert p.wait() == 0
    lib = os.path.join(out, f"libnmg_{name}.so")
    subprocess.run([B.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", lib, "-lcudart"],
                   check=True)
    print(lib)


if __name__ == "__main__":
    main()
