"""MOEPA1 ingestion throughput: a DSV2L-shaped trace
(d=2048, E=64, k=6: 8,472 B/record) written to local disk, then
read_trace_device (parallel positional reads -> pinned -> H2D -> K10) timed
end to end; plus the device-side part alone (records already pinned)."""
import json, os, sys, tempfile, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_10676_b200 import trace_io, _lib  # noqa: E402
from paper_2511_10676_b200.data import TraceFile  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 250_000
d, e, k = 2048, 64, 6
rng = np.random.default_rng(0)
acts = rng.standard_normal((n, d), dtype=np.float32)
lg = rng.standard_normal((n, e))
sc = np.exp(lg - lg.max(1, keepdims=True)); sc /= sc.sum(1, keepdims=True)
sc = sc.astype(np.float32)
topk = np.sort(np.argsort(-sc.astype(np.float64), axis=1, kind="stable")[:, :k], axis=1)
tf = TraceFile(d, e, k, acts, sc, topk)
path = os.path.join(tempfile.mkdtemp(), "big.moepa")
trace_io.write_trace(path, tf)
size = os.path.getsize(path)
# warm the page cache, then time
trace_io.read_trace_device(path)
torch.cuda.synchronize()
res = {}
for threads in (4, 8, 16):
    t0 = time.perf_counter()
    t = trace_io.read_trace_device(path, threads=threads)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    res[f"file_to_hbm_gbs_{threads}threads"] = size / dt / 1e9
# device-side part: pinned records -> H2D -> K10
rec = torch.from_numpy(trace_io._records(tf).view(np.int32)).pin_memory()
drec = torch.empty_like(rec, device="cuda")
a_out = torch.empty((n, d), dtype=torch.bfloat16, device="cuda")
s_out = torch.empty((n, e), dtype=torch.float32, device="cuda")
k_out = torch.empty((n, k), dtype=torch.int32, device="cuda")
st = torch.zeros(6, dtype=torch.int64, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for _ in range(2):
    ev[0].record(); drec.copy_(rec, non_blocking=True); ev[1].record()
    _lib.lib().moep_trace_ingest(drec.data_ptr(), n, d, e, k, _lib.MOEP_BF16, a_out.data_ptr(), s_out.data_ptr(),
                                 k_out.data_ptr(), 0, st.data_ptr(), torch.cuda.current_stream().cuda_stream)
    ev[2].record(); torch.cuda.synchronize()
res.update({"records": n, "file_bytes": size, "h2d_gbs": size / ev[0].elapsed_time(ev[1]) * 1e3 / 1e9,
            "k10_gbs": size / ev[1].elapsed_time(ev[2]) * 1e3 / 1e9, "k10_ms": ev[1].elapsed_time(ev[2]),
            "status": st.cpu().tolist(), "host_cores": os.cpu_count()})
os.remove(path)
print(json.dumps(res))
