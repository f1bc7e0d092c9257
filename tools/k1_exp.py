"""K1 timing experiments on variant builds (timing only; variants compute
wrong results). Each variant recompiles csrc/k1v2_predict.cu with extra -D
flags and links it with the product objects into tools/_k1prof/, then times
16 back-to-back launches of one DSV2L 1 M-token layer (same method as
tools/k1_cycle.py) in a subprocess with MOEP_LIB pointing at the variant.

    python tools/k1_exp.py base NOW1 NOX NOACT
flags: NOW1 (W1 loaded once per item), NOX (x loaded once per item),
NOACT (identity activation), PROF (role counters)."""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tools", "_k1prof")
FLAGS = {"DEC512": ["-DMOEP_DEC_ROWS_MAX=512"], "DEC1024": ["-DMOEP_DEC_ROWS_MAX=1024"],
         "W1NORMAL": ["-DK1V4_W1_NORMAL"], "XNORMAL": ["-DK1V4_X_NORMAL"], "TRACE": ["-DMOEP_K1_PROF"], "NOW1": ["-DMOEP_K1_EXP_NOW1"], "NOX": ["-DMOEP_K1_EXP_NOX"], "NOACT": ["-DMOEP_K1_PROF_NOACT"],
         "base": []}

TIMER = r'''
import os, sys, json, torch
sys.path.insert(0, %r)
import bench
dev = torch.device("cuda")
layers = bench.make_layers(dev, 1, bench.TOKENS, 0)
_, dp, x, t = layers[0]
part = torch.empty((148, 2 + 2 * 3 + 2 * bench.E), dtype=torch.int32, device=dev)
run = lambda: dp._k1(x, m_sel=0, bounds=(1, 6, 10), truth=t, k=6, m_values=bench.M_LIST, partials=part)
for _ in range(3): run()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(16): run()
b.record(); torch.cuda.synchronize()
print(json.dumps({"ms": a.elapsed_time(b) / 16}))
''' % ROOT


TRACE = r'''
import os, sys, json, ctypes as C, numpy as np, torch
sys.path.insert(0, %r)
import bench
from paper_2511_10676_b200 import _lib
L = _lib.lib()
dev = torch.device("cuda")
layers = bench.make_layers(dev, 1, bench.TOKENS, 0)
_, dp, x, t = layers[0]
part = torch.empty((148, 2 + 2 * 3 + 2 * bench.E), dtype=torch.int32, device=dev)
run = lambda: dp._k1(x, m_sel=0, bounds=(1, 6, 10), truth=t, k=6, m_values=bench.M_LIST, partials=part)
for _ in range(3): run()
torch.cuda.synchronize()
run(); torch.cuda.synchronize()
buf = np.zeros((16, 64), dtype=np.int64)
fn = L.moep_k1_trace if os.environ.get("MOEP_K1_TRACE") == "v2" else L.moep_k1v4_trace  # 1 M tokens: v4 runs
fn.argtypes = [C.c_void_p]
fn(buf.ctypes.data)
print(json.dumps(buf.tolist()))
''' % ROOT

NAMES = ["mma_acc_empty_done", "mma_first_full", "mma_gemm1_issued", "mma_g2h0_issued", "mma_g2h1_issued",
         "wg0_acc_full", "wg0_drained", "wg0_converted", "wg0_a2_written", "wg1_acc_full", "wg1_drained",
         "wg1_converted", "wg1_a2_emptyA", "wg1_a2_written", "wg0_tok_start", "wg0_tok_end"]


def trace():
    lib = os.path.join(OUT, "libmoep_exp_TRACE.so")
    if not os.path.exists(lib):
        build("TRACE")
    env = dict(os.environ, MOEP_LIB=lib)
    out = subprocess.run([sys.executable, "-c", TRACE], env=env, capture_output=True, text=True)
    line = [l for l in out.stdout.splitlines() if l.startswith("[")]
    if not line:
        print(out.stderr[-2000:])
        return
    import numpy as np
    buf = np.array(json.loads(line[-1]), dtype=np.int64)
    t0 = buf[0, 0]
    rel = np.where(buf != 0, buf - t0, -1)
    print("chunk " + " ".join(f"{n[:14]:>14s}" for n in NAMES))
    for c in range(40):
        print(f"{c:5d} " + " ".join(f"{v:14d}" for v in rel[:, c]))
    with open(os.path.join(ROOT, "gpurun_out", "k1_trace.json"), "w") as f:
        json.dump({"names": NAMES, "cycles_rel": rel.tolist()}, f)


def build(tag):
    sys.path.insert(0, ROOT)
    from paper_2511_10676_b200 import build as b
    b.build()
    os.makedirs(OUT, exist_ok=True)
    lib = os.path.join(OUT, f"libmoep_exp_{tag}.so")
    objs = []
    for name in ("k1v2_predict", "k1v4_predict", "k2b_fixup"):
        obj = os.path.join(OUT, f"{name}_{tag}.o")
        subprocess.run([b.nvcc(), *b.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *FLAGS[tag],
                        "-I", os.path.join(ROOT, "include"), "-c", os.path.join(b.CSRC, name + ".cu"), "-o", obj],
                       check=True)
        objs.append(obj)
    others = [o for o in glob.glob(os.path.join(b.HERE, "_build", "*.o"))
              if not o.endswith(("k1v2_predict.o", "k1v4_predict.o", "k2b_fixup.o"))]
    subprocess.run([b.nvcc(), *b.ARCH, "-shared", "-o", lib, *objs, *others], check=True)
    return lib


if __name__ == "__main__":
    tags = sys.argv[1:] or ["base"]
    if tags[0] == "--trace":
        trace()
        sys.exit(0)
    if tags[0] == "--build":
        for t in tags[1:]:
            print(build(t))
        sys.exit(0)
    res = {}
    for t in tags:
        lib = os.path.join(OUT, f"libmoep_exp_{t}.so")
        if not os.path.exists(lib):
            build(t)
        env = dict(os.environ, MOEP_LIB=lib)
        out = subprocess.run([sys.executable, "-c", TIMER], env=env, capture_output=True, text=True)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        res[t] = json.loads(line[-1])["ms"] if line else out.stderr[-500:]
        print(t, res[t], flush=True)
    print(json.dumps(res))
