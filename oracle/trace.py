"""CPU restatement of the reference's MOEPA1 reader and record invariants
(pkg/src/moepredict/synthgen.py:8-13 format, :219-253 read_trace, :123-145
TraceFile.validate). TEST INFRASTRUCTURE ONLY: the product path
(paper_2511_10676_b200.trace_io) never imports it. Pinned by
tests/test_oracle_golden.py against files and exception kinds produced by the
real reference (tests/golden/make_golden.py -> trace*.moepa, trace.npz).
"""

from __future__ import annotations

import struct

import numpy as np

from .oracle import top_k_batch

MAGIC = b"MOEPA1"
_HEADER = struct.Struct("<5I")


class OracleTraceError(Exception):
    """kind = the reference exception class name (synthgen.py raises)."""

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


def read_trace(blob: bytes):
    """-> (d, E, k, acts f32, scores f32, topk int64) or OracleTraceError."""
    if len(blob) < len(MAGIC):                                        # synthgen.py:223-224
        raise OracleTraceError("BadMagicError", "file too short for magic")
    if blob[: len(MAGIC)] != MAGIC:                                   # :225-226
        raise OracleTraceError("BadMagicError", f"bad magic {blob[:len(MAGIC)]!r}")
    off = len(MAGIC)
    if len(blob) < off + _HEADER.size:                                # :228-229
        raise OracleTraceError("TruncatedFileError", "file too short for header")
    version, d, e, k, n = _HEADER.unpack_from(blob, off)
    off += _HEADER.size
    if version != 1:                                                  # :232-233
        raise OracleTraceError("VersionError", f"unsupported trace version {version}")
    if d < 1 or e < 1 or not 1 <= k <= e or n < 1:                    # :234-237
        raise OracleTraceError("RecordValidationError", f"invalid header dims d={d} E={e} k={k} n={n}")
    rw = d + e + k
    expected, got = n * rw * 4, len(blob) - off                       # :238-244
    if got < expected:
        raise OracleTraceError("TruncatedFileError", f"expected {expected} record bytes, found {got}")
    if got > expected:
        raise OracleTraceError("TraceFormatError", f"{got - expected} trailing bytes after records")
    words = np.frombuffer(blob, dtype="<u4", offset=off).reshape(n, rw)
    acts = np.ascontiguousarray(words[:, :d]).view(np.float32)
    scores = np.ascontiguousarray(words[:, d: d + e]).view(np.float32)
    topk = words[:, d + e:].astype(np.int64)
    validate(acts, scores, topk, e, k)
    return d, e, k, acts, scores, topk


def validate(acts, scores, topk, e, k):
    """TraceFile.validate record checks, in order (synthgen.py:133-145)."""
    if not np.all(np.isfinite(acts)):
        raise OracleTraceError("RecordValidationError", "non-finite activation")
    s64 = scores.astype(np.float64)
    if np.any(s64 < 0) or np.any(s64 > 1):
        raise OracleTraceError("RecordValidationError", "score outside [0, 1]")
    if np.any(np.abs(s64.sum(axis=1) - 1.0) > 1e-5):
        raise OracleTraceError("RecordValidationError", "scores do not sum to 1 within 1e-5")
    if np.any(topk < 0) or np.any(topk >= e):
        raise OracleTraceError("RecordValidationError", "top-k index out of range")
    if k > 1 and np.any(np.diff(topk, axis=1) <= 0):
        raise OracleTraceError("RecordValidationError", "top-k rows must be sorted and distinct")
    if not np.array_equal(top_k_batch(scores.astype(np.float64), k), topk):
        raise OracleTraceError("RecordValidationError", "stored top-k inconsistent with scores")
