"""K1 logit error and near-tie flag cost at full scale (one 1M-token layer).

For each workload kind (workloads.py) and shape: K1's fp32 logits against
float64 logits of the same bf16 inputs (torch fp64 here: a measurement tool),
as |dz| / (||h||_2 * max_e ||w2_e||_2), the scale of the K1 margin; then the
flagged fraction, the accuracy and the per-layer pipeline time of
DevicePredictor.evaluate(ids_m=m) at several tau_rel.

    python tools/precision_scan.py [--n 1048576] [--kinds random,gate]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_10676_b200 as pb  # noqa: E402
import workloads as W  # noqa: E402


def fp64_logits(model, x, chunk=1 << 16):
    dev = x.device
    w1 = torch.as_tensor(model.w1, device=dev)
    w2 = torch.as_tensor(model.w2, device=dev)
    b1 = torch.as_tensor(model.b1, device=dev)
    b2 = torch.as_tensor(model.b2, device=dev)
    zs, hn = [], []
    for s in range(0, x.shape[0], chunk):
        a = x[s: s + chunk].double() @ w1.T + b1
        h = a * torch.sigmoid(a)
        zs.append(h @ w2.T + b2)
        hn.append(torch.linalg.vector_norm(h, dim=1))
    return torch.cat(zs), torch.cat(hn)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--kinds", default="random,gate")
    ap.add_argument("--shapes", default="dsv2l,qwen3")
    ap.add_argument("--taus", default="2e-6,4e-6,8e-6")
    args = ap.parse_args()
    dev = torch.device("cuda")
    shapes = {"dsv2l": (2048, 2048, 64, 6, [6, 10, 64]), "qwen3": (2048, 2048, 128, 8, [8, 12, 128])}
    for shape in args.shapes.split(","):
        d, h, E, k, ms = shapes[shape]
        for kind in args.kinds.split(","):
            model, x, truth = W.make_layer(kind, d, h, E, k, args.n, seed=3, device=dev)
            dp = pb.DevicePredictor(model, dev)
            lg = torch.empty((args.n, E), dtype=torch.float32, device=dev)
            dp._k1(x, logits=lg)
            z64, hn = fp64_logits(model, x)
            scale = hn * dp.w2_norm
            err = ((lg.double() - z64).abs().amax(1) / scale)
            q = torch.quantile(err[: 1 << 24].float(), torch.tensor([0.5, 0.999, 0.99999], device=dev))
            absmax = float((lg.double() - z64).abs().max())
            rec = {"shape": shape, "kind": kind, "n": args.n, "err_ratio_max": float(err.max()),
                   "err_ratio_p50": float(q[0]), "err_ratio_p999": float(q[1]), "err_ratio_p99999": float(q[2]),
                   "abs_err_max": absmax, "scale_median": float(scale.median()),
                   "z_std": float(z64.std()), "taus": []}
            del z64
            for _ in range(2):
                dp._k1(x, logits=lg)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                dp._k1(x, logits=lg)
            b.record()
            torch.cuda.synchronize()
            rec["k1_ms"] = a.elapsed_time(b) / 5
            rec["lib"] = os.environ.get("MOEP_LIB", "product")
            for tau in [float(t) for t in args.taus.split(",")]:
                dp.tau_rel = tau
                st = dp.new_status()
                for ids_m in (0, k):
                    for _ in range(2):
                        cnt, fc, ids = dp.evaluate(x, truth, k, ms, ids_m=ids_m, status=st)
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    for _ in range(3):
                        cnt, fc, ids = dp.evaluate(x, truth, k, ms, ids_m=ids_m, status=st)
                    b.record()
                    torch.cuda.synchronize()
                    c = pb.EvalCounters.from_array(cnt.cpu().numpy(), k, E, ms)
                    rec["taus"].append({"tau_rel": tau, "ids_m": ids_m, "flagged": int(fc.item()),
                                        "flagged_frac": int(fc.item()) / args.n,
                                        "ms_per_layer": a.elapsed_time(b) / 3,
                                        "exact": c.overprov[k] / c.n, "top1": c.top1 / c.n,
                                        "overprov": c.overprov[ms[1]] / c.n})
            print(json.dumps(rec), flush=True)
            del x, truth, lg, dp


if __name__ == "__main__":
    main()
