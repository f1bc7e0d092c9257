"""Clocks / power during a sustained cuBLAS bf16 GEMM vs a sustained K1 run
(is K1 limited by the power cap through energy per FLOP?)."""
import json, os, subprocess, sys, threading, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def sample(stop, out):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                            "--format=csv,noheader,nounits"], capture_output=True, text=True)
        out.append(r.stdout.strip())
        time.sleep(0.2)


def measure(fn, flop, seconds=3.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    stop, samples = threading.Event(), []
    t = threading.Thread(target=sample, args=(stop, samples))
    t.start()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    a.record()
    t0 = time.time()
    while time.time() - t0 < seconds:
        for _ in range(4):
            fn()
        n += 4
        torch.cuda.synchronize()
    b.record()
    torch.cuda.synchronize()
    stop.set(); t.join()
    ms = a.elapsed_time(b) / n
    clk = sorted(float(s.split(",")[0]) for s in samples if s)
    pw = sorted(float(s.split(",")[1]) for s in samples if s)
    return {"ms": ms, "tflops": flop / ms / 1e9, "sm_mhz_median": clk[len(clk) // 2], "power_w_median": pw[len(pw) // 2]}


M = N = K = 8192
A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
B = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
res = {"cublas_bf16_8192": measure(lambda: torch.mm(A, B, out=C), 2 * M * N * K)}
del A, B, C
layers = bench.make_layers(torch.device("cuda"), 1, bench.TOKENS, 0)
_, dp, x, t = layers[0]
part = torch.empty((148, 2 + 6 + 128), dtype=torch.int32, device="cuda")
res["k1_dsv2l_1m"] = measure(lambda: dp._k1(x, m_sel=0, bounds=(1, 6, 10), truth=t, k=6, m_values=[6, 10, 64],
                                            partials=part), bench.FLOP_PER_TOKEN * bench.TOKENS)
print(json.dumps(res))
