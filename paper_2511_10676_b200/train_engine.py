"""Device training state for the expert predictor (one GPU, optional DP hooks).

Parameters live in one flat master buffer [w1 | w2 | b1 | b2 (| bn_scale |
bn_shift)] (the layout the fused optimizer K6 walks), with gradients, moments
and — in fp32 mode — a bf16 shadow of [w1 | w2] that the tensor-core forward
(K1) reads. arch1 also keeps the batch-norm running statistics on the device.

Precision modes:
  "fp64"  exact-parity mode: forward through K2 (fp64 CUDA cores) with the
          pre-activation output; arch1 adds batch-norm batch statistics and the
          reference's Philox dropout stream on the device (bn_train.cu);
          K4 loss in fp64, K5 / bn_backward in fp64, dW1 by an fp64 GEMM, K6 in
          fp64 — the reference's float64 arithmetic step for step
          (trainer.py:131-204, predictor.py:193-327).
  "fp32"  throughput mode (arch2): forward K1 (bf16 tcgen05 GEMMs with the hi/lo
          GEMM2, fp32 pre-activations), K4 on fp32 logits (fp64 math), K5 fp32,
          dW1 = dA^T X on the tcgen05 tensor cores (moep_dw1_bf16, MN-major
          operands straight from K5's dA and the input) with dA split hi+lo,
          fp32 master weights and Adam moments.
One step = forward, loss (+ optional all-reduce of the 3 loss partial sums for
batch-global normalisers), backward, optional gradient all-reduce, optimizer.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import MOEP_F64, check, dtype_code, lib, ptr
from .exceptions import ConfigurationError
from .losses import LossSpec, device_loss

OPT_KIND = {"sgd": 0, "momentum": 1, "adam": 2}


def _stream(dev):
    return torch.cuda.current_stream(dev).cuda_stream


class DeviceTrainer:
    def __init__(self, model, loss: LossSpec, optimizer="adam", lr=1e-3, momentum=0.9, beta1=0.9,
                 beta2=0.999, eps=1e-8, precision="fp32", device="cuda", grad_allreduce=None,
                 loss_allreduce=None):
        # fp64: exact parity mode (the reference's arithmetic); fp32: fp32 master
        # weights, bf16 tensor-core GEMMs with hi/lo split operands; bf16: as fp32
        # but the dW1 GEMM takes dA rounded to bf16 (no lo half: half the GEMM)
        if precision not in ("fp32", "fp64", "bf16"):
            raise ConfigurationError(f"unknown precision {precision!r}")
        if model.arch == "arch1" and precision != "fp64":
            raise ConfigurationError("arch1 (batch-norm) training runs in the fp64 mode")
        self.dev = torch.device(device)
        lib()
        self.arch = model.arch
        self.loss_spec, self.kind = loss, OPT_KIND[optimizer]
        self.lr, self.momentum, self.beta1, self.beta2, self.eps = lr, momentum, beta1, beta2, eps
        self.precision = precision
        self.k1_kernel = _lib.MOEP_K1_AUTO  # forced forward K1 kernel (A-B timing), else auto
        self.dt = torch.float64 if precision == "fp64" else torch.float32
        self.d, self.H, self.E = model.d, model.hidden, model.n_experts
        d, H, E = self.d, self.H, self.E
        self.shapes = [(H, d), (E, H), (H,), (E,)]
        arrays = [model.w1, model.w2, model.b1, model.b2]
        if self.arch == "arch1":
            self.shapes += [(H,), (H,)]
            arrays += [model.bn_scale, model.bn_shift]
        self.sizes = [int(np.prod(s)) for s in self.shapes]
        self.offs = np.concatenate([[0], np.cumsum(self.sizes)]).tolist()
        self.flat = torch.empty(self.offs[-1], dtype=self.dt, device=self.dev)
        for arr, o, s in zip(arrays, self.offs, self.sizes):
            self.flat[o: o + s].copy_(torch.as_tensor(np.ascontiguousarray(arr, dtype=np.float64).ravel()))
        self.grad = torch.zeros_like(self.flat)
        self.m = torch.zeros_like(self.flat)
        self.v = torch.zeros_like(self.flat) if self.kind == 2 else None
        self.n_shadow = H * d + E * H
        self.shadow = self.flat[: self.n_shadow].to(torch.bfloat16) if precision != "fp64" else None
        if self.arch == "arch1":
            f64 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).to(self.dev)
            self.run_mean, self.run_var = f64(model.bn_mean), f64(model.bn_var)
            self.bn_momentum, self.bn_eps = float(model.bn_momentum), float(model.bn_eps)
            self.dropout_rate = float(model.dropout_rate)
            self.dropout_seed = int(model.dropout_seed) & 0xFFFFFFFFFFFFFFFF
            self.dropout_step = int(getattr(model, "_dropout_step", 0))
        self.nonfinite = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self._dw1_ws = None  # K-split partials of the tcgen05 dW1 GEMM
        self.t = 0
        self.grad_allreduce, self.loss_allreduce = grad_allreduce, loss_allreduce
        self.n_sms = lib().moep_num_sms()

    # ------------------------------------------------------------ views
    def view(self, buf, i):
        return buf[self.offs[i]: self.offs[i] + self.sizes[i]].view(self.shapes[i])

    def params_numpy(self):
        return [self.view(self.flat, i).double().cpu().numpy() for i in range(len(self.sizes))]

    # ---------------------------------------------------------- forward
    def _k2_preact(self, x64, z):
        """fp64 pre-activations a = x W1^T + b1 through K2 (its eval logits go to z)."""
        n = x64.shape[0]
        a_pre = torch.empty((n, self.H), dtype=torch.float64, device=self.dev)
        w2t = self.view(self.flat, 1).t().contiguous()
        A = _lib.Fp64Args()
        A.n_tokens, A.d, A.hidden, A.n_experts = n, self.d, self.H, self.E
        A.arch = 1 if self.arch == "arch1" else 2
        A.x_dtype, A.w_dtype = dtype_code(x64), MOEP_F64
        A.x, A.w1, A.w2, A.w2t = ptr(x64), ptr(self.view(self.flat, 0)), ptr(self.view(self.flat, 1)), ptr(w2t)
        A.b1, A.b2 = ptr(self.view(self.flat, 2)), ptr(self.view(self.flat, 3))
        if self.arch == "arch1":
            A.bn_scale, A.bn_shift = ptr(self.view(self.flat, 4)), ptr(self.view(self.flat, 5))
            A.bn_mean, A.bn_var, A.bn_eps = ptr(self.run_mean), ptr(self.run_var), self.bn_eps
        A.logits64, A.a_out = ptr(z), ptr(a_pre)
        check(lib().moep_predict_fp64(A, _stream(self.dev)), "moep_predict_fp64")
        return a_pre

    def forward(self, x, dropout_mask=None, training=True):
        """Train-mode forward: logits [N, E], the cache the backward needs, and
        the activations actually used."""
        n = x.shape[0]
        if self.precision != "fp64":
            xb = x if x.dtype == torch.bfloat16 else x.to(torch.bfloat16)
            z = torch.empty((n, self.E), dtype=torch.float32, device=self.dev)
            a_pre = torch.empty((n, self.H), dtype=torch.float32, device=self.dev)
            flags = torch.empty(n, dtype=torch.uint8, device=self.dev)
            fl = torch.empty(n, dtype=torch.int32, device=self.dev)
            fc = torch.zeros(1, dtype=torch.int32, device=self.dev)
            A = _lib.PredictArgs()
            A.n_tokens, A.d, A.hidden, A.n_experts, A.arch = n, self.d, self.H, self.E, 2
            A.x = ptr(xb)
            A.w1 = ptr(self.shadow[: self.H * self.d])
            A.w2 = ptr(self.shadow[self.H * self.d:])
            A.b1, A.b2 = ptr(self.view(self.flat, 2)), ptr(self.view(self.flat, 3))
            A.logits, A.flags, A.flag_list, A.flag_count, A.a_out = ptr(z), ptr(flags), ptr(fl), ptr(fc), ptr(a_pre)
            need = int(lib().moep_predict_split_floats(n, self.H, self.E))
            scratch = torch.empty(need, dtype=torch.float32, device=self.dev) if need else None
            A.split_scratch, A.split_scratch_floats = ptr(scratch), need
            A.kernel = int(self.k1_kernel)
            check(lib().moep_predict_bf16(A, _stream(self.dev)), "moep_predict_bf16")
            return z, {"a": a_pre}, xb
        x64 = x if x.dtype in (torch.float64, torch.bfloat16) else x.to(torch.float64)
        z = torch.empty((n, self.E), dtype=torch.float64, device=self.dev)
        a_pre = self._k2_preact(x64, z)
        if self.arch == "arch2":
            return z, {"a": a_pre}, x64
        H = self.H
        buf = {k: torch.empty((n, H), dtype=torch.float64, device=self.dev) for k in ("a_hat", "bn_out", "keep", "h")}
        inv_std = torch.empty(H, dtype=torch.float64, device=self.dev)
        mask = None
        if dropout_mask is not None:
            mask = torch.as_tensor(np.asarray(dropout_mask, dtype=np.uint8)).to(self.dev).contiguous()
        check(lib().moep_bn_forward(ptr(a_pre), n, H, ptr(self.view(self.flat, 4)), ptr(self.view(self.flat, 5)),
                                    ptr(self.run_mean), ptr(self.run_var), self.bn_momentum, self.bn_eps,
                                    self.dropout_rate, self.dropout_seed, self.dropout_step, ptr(mask),
                                    ptr(buf["a_hat"]), ptr(buf["bn_out"]), ptr(buf["keep"]), ptr(buf["h"]),
                                    ptr(inv_std), int(training), _stream(self.dev)), "moep_bn_forward")
        if training and self.dropout_rate > 0 and dropout_mask is None:
            self.dropout_step += 1  # the reference draws one mask per train forward (predictor.py:228-230)
        check(lib().moep_rows_dot(ptr(buf["h"]), ptr(self.view(self.flat, 1)), ptr(self.view(self.flat, 3)), n, H,
                                  self.E, ptr(z), _stream(self.dev)), "moep_rows_dot")
        buf["inv_std"] = inv_std
        buf["training"] = training
        return z, buf, x64

    # --------------------------------------------------------- backward
    def backward(self, x_used, cache, dz):
        """Gradients into self.grad: K5 / bn_backward, then the dW1 GEMM."""
        n = x_used.shape[0]
        H, E = self.H, self.E
        if self.arch == "arch1":
            da = torch.empty((n, H), dtype=torch.float64, device=self.dev)
            check(lib().moep_bn_backward(ptr(dz), ptr(self.view(self.flat, 1)), n, H, E, ptr(cache["h"]),
                                         ptr(cache["keep"]), ptr(cache["bn_out"]), ptr(cache["a_hat"]),
                                         ptr(cache["inv_std"]), ptr(self.view(self.flat, 4)), ptr(da),
                                         ptr(self.view(self.grad, 1)), ptr(self.view(self.grad, 2)),
                                         ptr(self.view(self.grad, 4)), ptr(self.view(self.grad, 5)),
                                         int(cache.get("training", True)), _stream(self.dev)), "moep_bn_backward")
            torch.sum(dz, dim=0, out=self.view(self.grad, 3))
        else:
            # row slices: enough CTAs to fill the GPU (the x2 fp32 kernel has half the columns per CTA)
            n_slices = max(1, min(64 if self.precision == "fp64" else 128, n // 128))
            scratch = torch.empty(n_slices * (E * H + H + E), dtype=self.dt, device=self.dev)
            if self.precision == "fp64":
                da = torch.empty((n, H), dtype=self.dt, device=self.dev)
                check(lib().moep_act_backward(ptr(cache["a"]), ptr(dz), ptr(self.view(self.flat, 1)),
                                              dtype_code(dz), n, H, E, n_slices, ptr(da), ptr(self.view(self.grad, 1)),
                                              ptr(self.view(self.grad, 2)), ptr(self.view(self.grad, 3)),
                                              ptr(scratch), _stream(self.dev)), "moep_act_backward")
            else:
                # dA leaves K5 as bf16 hi (| lo) halves: the dW1 GEMM operands directly
                lo = self.precision == "fp32"
                da = torch.empty((n, (2 if lo else 1) * H), dtype=torch.bfloat16, device=self.dev)
                check(lib().moep_act_backward_bf16split(ptr(cache["a"]), ptr(dz), ptr(self.view(self.flat, 1)), n,
                                                        H, E, n_slices, int(lo), ptr(da),
                                                        ptr(self.view(self.grad, 1)),
                                                        ptr(self.view(self.grad, 2)), ptr(self.view(self.grad, 3)),
                                                        ptr(scratch), _stream(self.dev)),
                      "moep_act_backward_bf16split")
        gw1 = self.view(self.grad, 0)
        if self.precision == "fp64":
            # fp64 dW1 = dA^T X on the fp64 tensor cores (moep_dgemm_tn)
            xs = x_used if x_used.dtype == torch.float64 else x_used.to(torch.float64)
            xs = xs.contiguous()
            check(lib().moep_dgemm_tn(ptr(da), H, ptr(xs), self.d, ptr(gw1), self.d, H, self.d, n,
                                      _stream(self.dev)), "moep_dgemm_tn")
        else:
            # tcgen05 dW1 (moep_dw1_bf16): dA leaves K5 as bf16 [n, P*h] (P = 2: hi | lo)
            passes = 2 if self.precision == "fp32" else 1
            need = int(lib().moep_dw1_workspace_floats(H, self.d, n, passes))
            if need and (self._dw1_ws is None or self._dw1_ws.numel() < need):
                self._dw1_ws = torch.empty(need, dtype=torch.float32, device=self.dev)
            ws = self._dw1_ws if need else None
            check(lib().moep_dw1_bf16(ptr(da), ptr(x_used.contiguous()), n, H, self.d, passes, ptr(gw1), ptr(ws),
                                      ws.numel() if ws is not None else 0, _stream(self.dev)), "moep_dw1_bf16")
        return da

    # -------------------------------------------------------------- step
    def optimizer_step(self):
        self.t += 1
        A = _lib.OptimArgs()
        A.kind, A.dtype, A.n = self.kind, dtype_code(self.flat), self.flat.numel()
        A.params, A.grads, A.m, A.v = ptr(self.flat), ptr(self.grad), ptr(self.m), ptr(self.v)
        A.lr, A.beta1, A.beta2, A.eps, A.momentum, A.t = self.lr, self.beta1, self.beta2, self.eps, self.momentum, self.t
        A.shadow_bf16, A.n_shadow, A.nonfinite = ptr(self.shadow), self.n_shadow, ptr(self.nonfinite)
        check(lib().moep_optim_step(A, _stream(self.dev)), "moep_optim_step")

    def step(self, x, scores, mask, rank, n_global=None):
        """One training step; returns the device loss tensor [loss, n_pairs] (no host sync).

        Under data parallelism a rank whose slice of the minibatch is empty
        (a last minibatch smaller than the world) still joins both all-reduces
        with zero partial sums and a zero gradient, so its peers do not wait
        forever and every rank applies the same update."""
        if x.shape[0] == 0:
            return self._empty_step(n_global or 0)
        z, cache, x_used = self.forward(x)
        zs = z if scores.dtype == z.dtype else z.to(scores.dtype)
        out, dz = device_loss(self.loss_spec, zs, scores, mask, rank, n_global=n_global,
                              allreduce=self.loss_allreduce)
        if dz.dtype != self.dt:
            dz = dz.to(self.dt)
        self.backward(x_used, cache, dz.contiguous())
        if self.grad_allreduce is not None:
            self.grad_allreduce(self.grad)
        self.optimizer_step()
        return out

    def _empty_step(self, n_global):
        from .losses import FAMILY_CODE
        code = FAMILY_CODE[self.loss_spec.family]
        partials = torch.zeros((1, 3), dtype=torch.float64, device=self.dev)
        if self.loss_allreduce is not None:
            self.loss_allreduce(partials)
        out = torch.empty(2, dtype=torch.float64, device=self.dev)
        check(lib().moep_loss_finalize(ptr(partials), 1, 0, self.E, code, self.loss_spec.ranking_lambda,
                                       int(self.loss_spec.normalize_ranking), dtype_code(self.flat), None, None,
                                       ptr(out), _stream(self.dev)), "moep_loss_finalize")
        self.grad.zero_()
        if self.grad_allreduce is not None:
            self.grad_allreduce(self.grad)
        self.optimizer_step()
        return out

    def to_model(self, template):
        from .predictor import PredictorModel
        ps = self.params_numpy()
        w1, w2, b1, b2 = ps[:4]
        if self.arch == "arch1":
            return PredictorModel("arch1", w1, b1, w2, b2, bn_scale=ps[4], bn_shift=ps[5],
                                  bn_mean=self.run_mean.cpu().numpy(), bn_var=self.run_var.cpu().numpy(),
                                  dropout_rate=template.dropout_rate, bn_momentum=template.bn_momentum,
                                  bn_eps=template.bn_eps, dropout_seed=template.dropout_seed,
                                  _dropout_step=self.dropout_step)
        return PredictorModel("arch2", w1, b1, w2, b2, dropout_rate=template.dropout_rate,
                              dropout_seed=template.dropout_seed)
