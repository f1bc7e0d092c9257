"""Where the K1 pair kernel's roles wait (cycles in each mbarrier wait, one
representative thread per role), from a profiling build of the library
(-DMOEP_K1_PROF; the product library has no counters). Builds it into
tools/_k1prof/ if needed (nvcc), then runs one DSV2L 1 M-token K1 launch."""
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tools", "_k1prof")
LIB = os.path.join(OUT, "libmoep_b200_prof.so")


NOACT = "--noact" in sys.argv
if NOACT:
    LIB = os.path.join(OUT, "libmoep_b200_prof_noact.so")


def build():
    sys.path.insert(0, ROOT)
    from paper_2511_10676_b200 import build as b
    os.makedirs(OUT, exist_ok=True)
    objs = []
    for src in b.sources():
        obj = os.path.join(OUT, os.path.basename(src).replace(".cu", "_noact.o" if NOACT else ".o"))
        subprocess.run([b.nvcc(), *b.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-DMOEP_K1_PROF",
                        *(["-DMOEP_K1_PROF_NOACT"] if NOACT else []),
                        "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj], check=True)
        objs.append(obj)
    subprocess.run([b.nvcc(), *b.ARCH, "-shared", "-o", LIB, *objs], check=True)


if __name__ == "__main__":
    if "--build" in sys.argv or not os.path.exists(LIB):
        build()
        if "--build" in sys.argv:
            sys.exit(0)
    os.environ["MOEP_LIB"] = LIB
    sys.path.insert(0, ROOT)
    import torch
    import bench
    from paper_2511_10676_b200 import _lib
    L = _lib.lib()
    prof = L.moep_k1_prof  # role counters exist in the v2 pair kernel only
    prof.argtypes = [C.c_void_p, C.c_int]
    layers = bench.make_layers(torch.device("cuda"), 1, bench.TOKENS, 0)
    _, dp, x, t = layers[0]
    dp.k1_kernel = _lib.MOEP_K1_PAIR_V2
    part = torch.empty((148, 136), dtype=torch.int32, device="cuda")
    run = lambda: dp._k1(x, m_sel=0, bounds=(1, 6, 10), truth=t, k=6, m_values=[6, 10, 64], partials=part)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    prof(None, 1)
    run()
    torch.cuda.synchronize()
    import numpy as np
    buf = np.zeros((160, 16), dtype=np.uint64)
    prof(buf.ctypes.data, 0)
    names = {0: "TMA x/W1: wait empty (ring full)", 1: "TMA W2: wait w2_empty", 2: "MMA: wait z_empty",
             3: "MMA: wait w2_full", 4: "MMA: wait a2_full (block)", 5: "MMA: wait acc_empty",
             6: "MMA: wait full (operands)", 7: "EPI WG0: wait acc_full", 8: "EPI WG0: wait a2_emptyB",
             9: "EPI WG1: wait a2_emptyA", 10: "EPI WG0: wait z_full", 11: "EPI WG1: wait acc_full",
             12: "EPI WG0: drain (ld + arrive) duration", 13: "EPI WG1: drain duration",
             14: "EPI WG0: bias/act/hi-lo convert duration", 15: "total kernel cycles (thread 0)"}
    lead = buf[0:148:2]          # leader CTAs (MMA issuer lives there)
    tot = lead[:, 15].astype(float).mean()
    for s_, n in names.items():
        v = lead[:, s_].astype(float).mean()
        print(f"{n:44s} {v / tot * 100:6.2f} %  ({v:.0f} cycles, {v / 448:.0f} per chunk)")  # v3: 11 chunks / tile
