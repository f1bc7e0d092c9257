"""MOEPA1 trace files <-> device arrays (GPU ingestion).

The reference format (pkg/src/moepredict/synthgen.py:8-13, writer :197-216,
reader :219-253), little-endian:
    magic   6 bytes  b"MOEPA1"
    header  5 x u32  version, d, E, k, n
    record  d x f32 activation, E x f32 scores, k x u32 top-k indices

`read_trace_device` streams the records from the file into pinned host
buffers (parallel positional reads), copies them to the GPU on a side stream
double-buffered against K10 (`moep_trace_ingest`), which de-interleaves them
into device arrays and re-checks every record invariant of
TraceFile.validate (synthgen.py:123-145). Header / size problems raise the
reference's exceptions before any transfer; record problems raise
RecordValidationError for the first failing check in the reference's order.
"""

from __future__ import annotations

import os
import struct
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check, lib, ptr
from .data import TraceFile
from .exceptions import (BadMagicError, DataError, RecordValidationError, TraceFormatError, TruncatedFileError,
                         VersionError)

MAGIC = b"MOEPA1"
VERSION = 1
_HEADER = struct.Struct("<5I")  # version, d, E, k, n
HEADER_BYTES = len(MAGIC) + _HEADER.size

# K10 status slots, in TraceFile.validate's check order (synthgen.py:135-145)
_RECORD_ERRORS = (
    "non-finite activation",
    "score outside [0, 1]",
    "scores do not sum to 1 within 1e-5",
    "top-k index out of range",
    "top-k rows must be sorted and distinct",
    "stored top-k inconsistent with scores",
)


@dataclass
class TraceHeader:
    version: int
    hidden_dim: int
    n_experts: int
    k: int
    n: int

    @property
    def record_words(self) -> int:
        return self.hidden_dim + self.n_experts + self.k


@dataclass
class DeviceTrace:
    """A trace resident in HBM: activations [n, d] (fp32 or bf16), scores
    [n, E] fp32, top-k [n, k] int32 (rows ascending)."""

    hidden_dim: int
    n_experts: int
    k: int
    activations: torch.Tensor
    true_scores: torch.Tensor
    true_topk: torch.Tensor

    def __len__(self) -> int:
        return self.activations.shape[0]

    def to_host(self) -> TraceFile:
        return TraceFile(self.hidden_dim, self.n_experts, self.k, self.activations.float().cpu().numpy(),
                         self.true_scores.cpu().numpy(), self.true_topk.cpu().numpy().astype(np.int64))


def parse_header(blob: bytes, file_bytes: int) -> TraceHeader:
    """Header and size checks of read_trace (synthgen.py:222-245), same exceptions."""
    if len(blob) < len(MAGIC):
        raise BadMagicError("file too short for magic")
    if blob[: len(MAGIC)] != MAGIC:
        raise BadMagicError(f"bad magic {blob[:len(MAGIC)]!r}")
    if len(blob) < HEADER_BYTES:
        raise TruncatedFileError("file too short for header")
    version, d, n_experts, k, n = _HEADER.unpack_from(blob, len(MAGIC))
    if version != VERSION:
        raise VersionError(f"unsupported trace version {version}")
    if d < 1 or n_experts < 1 or not 1 <= k <= n_experts or n < 1:
        raise RecordValidationError(f"invalid header dims d={d} E={n_experts} k={k} n={n}")
    h = TraceHeader(version, d, n_experts, k, n)
    expected = n * h.record_words * 4
    got = file_bytes - HEADER_BYTES
    if got < expected:
        raise TruncatedFileError(f"expected {expected} record bytes, found {got}")
    if got > expected:
        raise TraceFormatError(f"{got - expected} trailing bytes after records")
    return h


def _pread_parallel(fd: int, dst: np.ndarray, offset: int, threads: int) -> None:
    """Fill the byte view `dst` from file offset `offset` with positional reads
    on `threads` threads (the page-cache copy is the host-side bottleneck)."""
    n = dst.nbytes
    step = max(1 << 20, -(-n // threads))
    errors = []

    def work(lo, hi):
        try:
            view = memoryview(dst[lo:hi])
            done = 0
            while done < hi - lo:
                got = os.preadv(fd, [view[done:]], offset + lo + done)
                if got <= 0:
                    raise TruncatedFileError("short read")
                done += got
        except Exception as exc:  # noqa: BLE001 - re-raised on the caller's thread
            errors.append(exc)

    ts = [threading.Thread(target=work, args=(lo, min(n, lo + step))) for lo in range(0, n, step)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errors:
        raise errors[0]


def _raise_status(status: torch.Tensor) -> None:
    st = status.cpu().numpy()
    for i, msg in enumerate(_RECORD_ERRORS):
        if st[i]:
            raise RecordValidationError(msg)


def read_trace_device(path, device="cuda", act_dtype=torch.float32, chunk_bytes: int = 64 << 20,
                      threads: int = 8) -> DeviceTrace:
    """Stream a MOEPA1 file into HBM and validate it on the GPU (read_trace,
    synthgen.py:219-253, with the arrays left on the device)."""
    dev = torch.device(device)
    if act_dtype not in (torch.float32, torch.bfloat16):
        raise ValueError("act_dtype must be torch.float32 or torch.bfloat16")
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        head = f.read(HEADER_BYTES)
    h = parse_header(head, size)
    rw = h.record_words
    rec_bytes = rw * 4
    chunk = max(1, min(h.n, chunk_bytes // rec_bytes))
    acts = torch.empty((h.n, h.hidden_dim), dtype=act_dtype, device=dev)
    scores = torch.empty((h.n, h.n_experts), dtype=torch.float32, device=dev)
    topk = torch.empty((h.n, h.k), dtype=torch.int32, device=dev)
    status = torch.zeros(6, dtype=torch.int64, device=dev)
    pinned = [torch.empty(chunk * rw, dtype=torch.int32).pin_memory() for _ in range(2)]
    dbuf = [torch.empty(chunk * rw, dtype=torch.int32, device=dev) for _ in range(2)]
    copy = torch.cuda.Stream(dev)
    main = torch.cuda.current_stream(dev)
    h2d_done = [torch.cuda.Event() for _ in range(2)]
    used = [torch.cuda.Event() for _ in range(2)]
    code = _lib.MOEP_BF16 if act_dtype == torch.bfloat16 else _lib.MOEP_F32
    fd = os.open(path, os.O_RDONLY)
    try:
        for ci, r0 in enumerate(range(0, h.n, chunk)):
            b = ci & 1
            nr = min(chunk, h.n - r0)
            h2d_done[b].synchronize()  # pinned[b] free again
            _pread_parallel(fd, pinned[b].numpy().view(np.uint8)[: nr * rec_bytes],
                            HEADER_BYTES + r0 * rec_bytes, threads)
            with torch.cuda.stream(copy):
                copy.wait_event(used[b])  # dbuf[b] consumed by the previous ingest
                dbuf[b][: nr * rw].copy_(pinned[b][: nr * rw], non_blocking=True)
                h2d_done[b].record(copy)
            main.wait_event(h2d_done[b])
            check(lib().moep_trace_ingest(ptr(dbuf[b]), nr, h.hidden_dim, h.n_experts, h.k, code, ptr(acts),
                                          ptr(scores), ptr(topk), r0, ptr(status), main.cuda_stream),
                  "moep_trace_ingest")
            used[b].record(main)
    finally:
        os.close(fd)
    _raise_status(status)
    return DeviceTrace(h.hidden_dim, h.n_experts, h.k, acts, scores, topk)


def read_trace(path, device="cuda") -> TraceFile:
    """read_trace (synthgen.py:219-253): host TraceFile, validated on the GPU."""
    return read_trace_device(path, device).to_host()


def _records(trace) -> np.ndarray:
    n = len(trace)
    rec = np.empty((n, trace.hidden_dim + trace.n_experts + trace.k), dtype="<u4")
    rec[:, : trace.hidden_dim] = np.ascontiguousarray(trace.activations, dtype=np.float32).view(np.uint32)
    rec[:, trace.hidden_dim: trace.hidden_dim + trace.n_experts] = (
        np.ascontiguousarray(trace.true_scores, dtype=np.float32).view(np.uint32))
    rec[:, trace.hidden_dim + trace.n_experts:] = np.asarray(trace.true_topk).astype(np.uint32)
    return rec


def validate_device(trace, device="cuda") -> None:
    """TraceFile.validate (synthgen.py:123-145) on the GPU (K10 over the records)."""
    n = len(trace)
    if np.asarray(trace.activations).shape != (n, trace.hidden_dim):
        raise RecordValidationError("activation block shape mismatch")
    if np.asarray(trace.true_scores).shape != (n, trace.n_experts):
        raise RecordValidationError("score block shape mismatch")
    if np.asarray(trace.true_topk).shape != (n, trace.k):
        raise RecordValidationError("top-k block shape mismatch")
    if n == 0:
        return
    dev = torch.device(device)
    rec = torch.from_numpy(_records(trace).view(np.int32)).to(dev)
    acts = torch.empty((n, trace.hidden_dim), dtype=torch.float32, device=dev)
    scores = torch.empty((n, trace.n_experts), dtype=torch.float32, device=dev)
    topk = torch.empty((n, trace.k), dtype=torch.int32, device=dev)
    status = torch.zeros(6, dtype=torch.int64, device=dev)
    check(lib().moep_trace_ingest(ptr(rec), n, trace.hidden_dim, trace.n_experts, trace.k, _lib.MOEP_F32, ptr(acts),
                                  ptr(scores), ptr(topk), 0, ptr(status),
                                  torch.cuda.current_stream(dev).cuda_stream), "moep_trace_ingest")
    _raise_status(status)


def write_trace(path, trace, device="cuda") -> None:
    """write_trace (synthgen.py:197-216): same bytes as the reference; the
    record invariants are checked on the GPU first."""
    if len(trace) == 0:
        raise DataError("refusing to write an empty trace")
    validate_device(trace, device)
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(_HEADER.pack(VERSION, trace.hidden_dim, trace.n_experts, trace.k, len(trace)))
        f.write(_records(trace).tobytes())
