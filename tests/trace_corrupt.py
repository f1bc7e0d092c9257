"""Byte-level corruptions of a MOEPA1 trace shared by tests/golden/make_golden.py
(which records the reference's exception for each) and the trace tests."""

import numpy as np


def corruptions(blob: bytes, d: int, e: int, k: int):
    """Byte-level corruptions of a valid trace, mirroring test_synthgen.py:112-172
    plus one per record invariant of TraceFile.validate (synthgen.py:135-145)."""
    hdr = 6 + 20
    rw = d + e + k
    out = {}
    b = bytearray(blob); b[0] ^= 0xFF; out["bad_magic"] = bytes(b)
    b = bytearray(blob); b[6] = 9; out["bad_version"] = bytes(b)
    out["truncated"] = blob[: len(blob) - 8]
    out["missing_record"] = blob[: len(blob) - 4 * rw]
    out["trailing"] = blob + b"\x00\x00\x00\x00"
    out["short_header"] = blob[:10]
    b = bytearray(blob); b[6 + 16: 6 + 20] = (0).to_bytes(4, "little"); out["zero_n"] = bytes(b)
    rec = lambda r, w: hdr + 4 * (r * rw + w)  # byte offset of word w of record r
    b = bytearray(blob); b[rec(3, 5): rec(3, 5) + 4] = np.float32(np.nan).tobytes(); out["nan_activation"] = bytes(b)
    b = bytearray(blob); b[rec(4, d + 1): rec(4, d + 1) + 4] = np.float32(1.5).tobytes(); out["score_range"] = bytes(b)
    b = bytearray(blob); s0 = np.frombuffer(blob[rec(5, d): rec(5, d) + 4], "<f4")[0]
    b[rec(5, d): rec(5, d) + 4] = np.float32(s0 * 0.5 if s0 > 1e-3 else s0 + 0.01).tobytes(); out["score_sum"] = bytes(b)
    b = bytearray(blob); b[rec(6, d + e): rec(6, d + e) + 4] = (e + 3).to_bytes(4, "little"); out["index_range"] = bytes(b)
    t = np.frombuffer(blob[rec(7, d + e): rec(7, d + e) + 4 * k], "<u4").copy()
    b = bytearray(blob); b[rec(7, d + e): rec(7, d + e) + 4 * k] = t[::-1].astype("<u4").tobytes(); out["unsorted"] = bytes(b)
    t = np.frombuffer(blob[rec(8, d + e): rec(8, d + e) + 4 * k], "<u4").copy()
    free = [x for x in range(e) if x not in set(t.tolist())]
    t2 = np.sort(np.concatenate([t[1:], [free[-1]]])).astype("<u4")
    b = bytearray(blob); b[rec(8, d + e): rec(8, d + e) + 4 * k] = t2.tobytes(); out["wrong_set"] = bytes(b)
    return out
