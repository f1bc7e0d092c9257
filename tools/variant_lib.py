"""Build an experiment variant of libmoep_b200.so with extra -D flags into
tools/_variants/<name>/ (the product library is untouched). Load it in a
fresh process with MOEP_LIB=<path> (paper_2511_10676_b200/_lib.py).

    python tools/variant_lib.py NAME [-DFLAG ...]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_10676_b200 import build as b  # noqa: E402


def build(name, flags):
    out = os.path.join(ROOT, "tools", "_variants", name)
    os.makedirs(out, exist_ok=True)
    procs, objs = [], []
    for src in b.sources():
        obj = os.path.join(out, os.path.basename(src).replace(".cu", ".o"))
        cmd = [b.nvcc(), *b.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *flags,
               "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        procs.append(subprocess.Popen(cmd))
        objs.append(obj)
    for p in procs:
        if p.wait() != 0:
            raise SystemExit("nvcc failed")
    lib = os.path.join(out, "libmoep_b200.so")
    subprocess.run([b.nvcc(), *b.ARCH, "-shared", "-o", lib, *objs], check=True)
    return lib


if __name__ == "__main__":
    print(build(sys.argv[1], sys.argv[2:]))
