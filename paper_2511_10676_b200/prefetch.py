"""Predicted-expert prefetch: pinned host expert store -> device expert cache.

The reference only models this path analytically (pipesim.py:185-325:
per-expert bytes, parallel load lanes, prefetch window = attention + post-norm
+ select - predict; stall = max(0, prefetch_end - t_select)). Here the bytes
actually move:

  ExpertStore   every expert blob of a layer in page-locked host memory
                (device-mapped, so the GPU can also read it directly)
  ExpertCache   device slots + an expert -> slot table
  Prefetcher    K8 plans the load on the device (union of the predicted
                m-sets of the batch minus resident experts), then either
                  * copy engines: one cudaMemcpyAsync per missing expert on a
                    side stream (the host reads the tiny plan first), or
                  * K9: an SM-driven gather from mapped host memory, enqueued
                    with no host round trip at all;
                an event marks completion for the consumer (expert compute).
Sizes follow the real models: DeepSeek-V2-Lite expert = 3 * 2048 * 1408 * 2 B
= 17,301,504 B; Qwen3-30B-A3B expert = 3 * 2048 * 768 * 2 B = 9,437,184 B.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from ._lib import check, lib, ptr

DSV2L_EXPERT_BYTES = 3 * 2048 * 1408 * 2
QWEN3_EXPERT_BYTES = 3 * 2048 * 768 * 2


@dataclass(frozen=True)
class ExpertShape:
    d_model: int
    d_ff: int
    bytes_per_param: int = 2

    @property
    def expert_bytes(self) -> int:
        # gate, up and down projections of one SwiGLU expert
        return 3 * self.d_model * self.d_ff * self.bytes_per_param


def _stream(s):
    return s.cuda_stream


class ExpertStore:
    """Page-locked host memory with `n_experts` blobs of `expert_bytes` each."""

    def __init__(self, n_experts: int, expert_bytes: int, fill: bool = True):
        if expert_bytes % 16:
            raise ValueError("expert_bytes must be a multiple of 16")
        self.n_experts, self.expert_bytes = n_experts, expert_bytes
        self.host = torch.empty(n_experts * expert_bytes, dtype=torch.uint8, pin_memory=True)
        if fill:
            # distinct byte pattern per expert so a misplaced copy is detectable
            v = self.host.view(n_experts, expert_bytes)
            for e in range(n_experts):
                v[e, :64].fill_(e & 0xFF)
                v[e, -64:].fill_((e * 7 + 3) & 0xFF)

    def blob(self, e: int) -> torch.Tensor:
        return self.host[e * self.expert_bytes:(e + 1) * self.expert_bytes]


class ExpertCache:
    """Device-resident expert slots with an expert -> slot table."""

    def __init__(self, n_slots: int, expert_bytes: int, n_experts: int, device="cuda"):
        self.n_slots, self.expert_bytes = n_slots, expert_bytes
        self.dev = torch.device(device)
        self.data = torch.empty(n_slots * expert_bytes, dtype=torch.uint8, device=self.dev)
        self.slot_of = torch.full((n_experts,), -1, dtype=torch.int32, device=self.dev)
        self.free_slots = torch.arange(n_slots, dtype=torch.int32, device=self.dev)
        self.free_cursor = torch.zeros(1, dtype=torch.int32, device=self.dev)  # next free slot (device)

    def reset(self):
        self.slot_of.fill_(-1)
        self.free_cursor.zero_()

    def slot(self, s: int) -> torch.Tensor:
        return self.data[s * self.expert_bytes:(s + 1) * self.expert_bytes]


class Prefetcher:
    def __init__(self, store: ExpertStore, cache: ExpertCache, copy_stream: torch.cuda.Stream | None = None):
        self.store, self.cache = store, cache
        self.dev = cache.dev
        self.copy = copy_stream or torch.cuda.Stream(self.dev)
        E = store.n_experts
        self.need_list = torch.empty(E, dtype=torch.int32, device=self.dev)
        self.need_slot = torch.empty(E, dtype=torch.int32, device=self.dev)
        self.need_count = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.mask = torch.empty(E, dtype=torch.uint8, device=self.dev)
        self.h_plan = torch.empty(2 * E + 1, dtype=torch.int32, pin_memory=True)
        self.done = torch.cuda.Event()

    def plan(self, ids: torch.Tensor, stream=None):
        """K8 on `stream` (default: current): union of ids minus resident experts."""
        st = stream or torch.cuda.current_stream(self.dev)
        ids = ids.to(device=self.dev, dtype=torch.int32).contiguous()
        c = self.cache
        check(lib().moep_prefetch_plan(ptr(ids), ids.numel(), self.store.n_experts, ptr(c.slot_of),
                                       ptr(c.free_slots), c.free_slots.numel(), ptr(c.free_cursor), ptr(self.mask),
                                       ptr(self.need_list), ptr(self.need_slot), ptr(self.need_count),
                                       _stream(st)), "moep_prefetch_plan")

    def commit(self, stream=None):
        """Mark the planned experts resident: a device-side table update on
        `stream` (default: the copy stream), no host synchronisation."""
        st = stream or self.copy
        c = self.cache
        check(lib().moep_prefetch_commit(ptr(self.need_list), ptr(self.need_slot), ptr(self.need_count),
                                         ptr(c.slot_of), ptr(c.free_cursor), _stream(st)), "moep_prefetch_commit")

    def load_copy_engine(self, ids: torch.Tensor) -> int:
        """Plan on the copy stream, read the plan on the host, one cudaMemcpyAsync
        per missing expert on the copy stream. Returns the number of experts moved."""
        with torch.cuda.stream(self.copy):
            self.plan(ids, self.copy)
            E = self.store.n_experts
            self.h_plan[:E].copy_(self.need_list, non_blocking=True)
            self.h_plan[E:2 * E].copy_(self.need_slot, non_blocking=True)
            self.h_plan[2 * E:].copy_(self.need_count, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.copy)
        ev.synchronize()  # the plan is tiny; in a decoder this overlaps the attention kernels
        n = int(self.h_plan[2 * E].item())
        lst = self.h_plan[:n].tolist()
        slots = self.h_plan[E:E + n].tolist()
        with torch.cuda.stream(self.copy):
            for e, s in zip(lst, slots):
                if s >= 0:
                    self.cache.slot(s).copy_(self.store.blob(e), non_blocking=True)
            self.commit(self.copy)
            self.done.record(self.copy)
        return n

    def load_sm_gather(self, ids: torch.Tensor, n_ctas: int = 64) -> None:
        """K8 + K9 + residency commit on the copy stream; no host round trip.
        Completion: self.done."""
        with torch.cuda.stream(self.copy):
            self.plan(ids, self.copy)
            check(lib().moep_gather_experts(self.store.host.data_ptr(), self.store.expert_bytes,
                                            ptr(self.need_list), ptr(self.need_slot), ptr(self.need_count),
                                            ptr(self.cache.data), n_ctas, _stream(self.copy)),
                  "moep_gather_experts")
            self.commit(self.copy)
            self.done.record(self.copy)


def measure_h2d_peak(n_bytes: int = 1 << 30, reps: int = 10, device="cuda") -> float:
    """Host-link roofline: best-of-`reps` pinned -> device copy-engine bandwidth (GB/s)."""
    h = torch.empty(n_bytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n_bytes, dtype=torch.uint8, device=device)
    s = torch.cuda.Stream(device)
    best = 0.0
    with torch.cuda.stream(s):
        d.copy_(h, non_blocking=True)
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            d.copy_(h, non_blocking=True)
            b.record(s)
            b.synchronize()
            best = max(best, n_bytes / (a.elapsed_time(b) / 1e3) / 1e9)
    return best
