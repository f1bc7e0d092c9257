"""Deployment at the hook point.

The reference trains its predictors on the exporter's `input_layernorm`
output (exporter/src/moeexport/hooks.py:19, 113-114) and only models what a
deployment does with the prediction (pipesim.py:272-305: the prefetch window
is attention + post-norm + select - predict; a miss costs an on-demand load).
`HookPointPredictor` executes it for one MoE layer of a decoder:

  pre_attention(hidden)   K0: the layer's input norm (rmsnorm / layernorm with
                          the model's gamma / beta / eps) -> x_hat, the tensor the
                          attention consumes; the predictor's top-m on x_hat (the
                          exact decode kernel for small batches, K1 + fix-up
                          otherwise); the prefetch of the predicted experts on a
                          side stream (K8 plan + copy engines or the K9 gather).
                          Nothing synchronises with the host except the
                          copy-engine path, which reads the tiny plan.
  post_router(true_ids)   once the router has chosen: the experts it chose that
                          are not resident are loaded on demand ("emergency"
                          loads, copy engines); returns their cache slots.
  check()                 the input contract (predictor.py:188-189): raises
                          ConfigurationError if a hidden state was non-finite.

Everything is enqueued on the caller's current stream (the decoder's), the
loads on the prefetcher's copy stream, ordered by events.
"""

from __future__ import annotations

import torch

from .engine import DevicePredictor, input_norm
from .exceptions import ConfigurationError
from .prefetch import Prefetcher


class HookPointPredictor:
    def __init__(self, model, m: int, norm: str = "rmsnorm", gamma=None, beta=None, eps=None,
                 prefetcher: Prefetcher | None = None, gather_ctas: int = 0, device="cuda"):
        self.pred = model if isinstance(model, DevicePredictor) else DevicePredictor(model, device)
        if not 1 <= m <= self.pred.E:
            raise ValueError(f"m={m} out of range for {self.pred.E} experts")
        self.m, self.norm, self.eps = m, norm, eps
        dev = self.pred.device
        self.gamma = None if gamma is None else torch.as_tensor(gamma, dtype=torch.float64).to(dev)
        self.beta = None if beta is None else torch.as_tensor(beta, dtype=torch.float64).to(dev)
        self.pf = prefetcher
        self.gather_ctas = gather_ctas          # 0: copy engines; > 0: K9 SM gather with that many CTAs
        self.norm_status = torch.zeros(2, dtype=torch.int32, device=dev)
        self.status = self.pred.new_status()
        self.predicted = None
        self.n_prefetched = 0
        self.ready = torch.cuda.Event()

    def pre_attention(self, hidden: torch.Tensor, prefetch: bool = True):
        """x_hat (bf16, for the attention) and the predicted ids [B, m] (int32,
        ascending); with `prefetch`, the load of the predicted experts is put in
        flight (otherwise call start_prefetch() after enqueueing the attention:
        the copy-engine path reads the plan on the host, which must not hold
        back the attention's launch)."""
        x_hat = input_norm(hidden, self.norm, self.gamma, self.beta, self.eps, status=self.norm_status,
                           device=self.pred.device)
        ids = self.pred.topk(x_hat, self.m, validate=False, status=self.status)
        self.predicted = ids
        if self.pf is not None:
            self.ready.record(torch.cuda.current_stream(self.pred.device))
            if prefetch:
                self.start_prefetch()
        return x_hat, ids

    def start_prefetch(self):
        """Load the predicted experts on the copy stream (after the predictor)."""
        self.pf.copy.wait_event(self.ready)
        if self.gather_ctas > 0:
            self.pf.load_sm_gather(self.predicted, self.gather_ctas)
            self.n_prefetched = -1           # known on the device only (pf.need_count)
        else:
            self.n_prefetched = self.pf.load_copy_engine(self.predicted)

    def post_router(self, true_ids: torch.Tensor):
        """Emergency loads of the router's experts that were not prefetched;
        returns (slot per true expert [B, k] int32, number of experts loaded now).
        The decoder's stream waits for every load it needs."""
        if self.pf is None:
            raise ConfigurationError("post_router needs a Prefetcher")
        main = torch.cuda.current_stream(self.pred.device)
        self.pf.copy.wait_stream(main)
        n = self.pf.load_copy_engine(true_ids)
        main.wait_stream(self.pf.copy)
        slots = self.pf.cache.slot_of[true_ids.to(device=self.pred.device, dtype=torch.long)]
        return slots, n

    def graph(self, batch: int) -> "GraphedHook":
        """pre_attention for a fixed decode batch captured into a CUDA graph.

        A decode step's pre-attention work is ~15 us of kernels (K0, the exact
        decode predictor) behind ~100 us of host launch overhead; replaying the
        graph issues it in one launch. The graph reads a static input buffer
        and writes static x_hat / ids buffers (valid until the next replay);
        the prefetch is started after the replay (start_prefetch), because the
        copy-engine path reads the plan on the host."""
        dev = self.pred.device
        static_in = torch.zeros((batch, self.pred.d), dtype=torch.bfloat16, device=dev)
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):  # warm-up outside the capture (allocator, attributes)
            for _ in range(2):
                self.pre_attention(static_in, prefetch=False)
        torch.cuda.current_stream(dev).wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            x_hat, ids = self.pre_attention(static_in, prefetch=False)
        return GraphedHook(self, g, static_in, x_hat, ids)

    def check(self):
        if int(self.norm_status[0].item()):
            raise ConfigurationError("input must be finite")


class GraphedHook:
    """A captured pre_attention (HookPointPredictor.graph)."""

    def __init__(self, hook: HookPointPredictor, g, static_in, x_hat, ids):
        self.hook, self.g, self.static_in, self.x_hat, self.ids = hook, g, static_in, x_hat, ids

    def pre_attention(self, hidden: torch.Tensor, prefetch: bool = True):
        """Same contract as HookPointPredictor.pre_attention for this batch size;
        returns the static (x_hat, ids) buffers of the graph."""
        if tuple(hidden.shape) != tuple(self.static_in.shape):
            raise ConfigurationError(f"graph captured for {tuple(self.static_in.shape)}, got {tuple(hidden.shape)}")
        self.static_in.copy_(hidden)
        self.g.replay()
        h = self.hook
        h.predicted = self.ids
        if h.pf is not None:
            h.ready.record(torch.cuda.current_stream(h.pred.device))
            if prefetch:
                h.start_prefetch()
        return self.x_hat, self.ids
