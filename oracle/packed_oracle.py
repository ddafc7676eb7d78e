"""ORACLE — test infrastructure only; never imported by the product package.

CPU restatement of the reference packed-data algorithms the training feed
depends on (reference: /root/reference/pkg/src/corpusforge/packed_data.py).
Used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
checker. Parity is pinned against golden vectors produced by importing the
reference itself (tests/golden/make_golden.py -> tests/golden/packed_golden.json).

Functions and the reference lines they restate:
  token_width(vocab)          packed_data.py:49-59
  parse_header(buf)           packed_data.py:26, :147-165 (header + invariants)
  sample_count(n_tok, L)      packed_data.py:188-194
  sample_window(payload,s,L)  packed_data.py:196-203
  batch_windows(...)          get_sample per id, stacked, split into ids[:L]/ids[1:]
  splitmix64_first(seed, k)   packed_data.py:226-238
  permutation(n, seed)        packed_data.py:257-282 (pure Python; small n only)
  chunk_sizes(n, k)           packed_data.py:322-333
"""

from __future__ import annotations

import struct

import numpy as np

M64 = (1 << 64) - 1
HEADER = struct.Struct("<8sIIQQQ")


class OracleFormatError(Exception):
    pass


def token_width(vocab: int) -> int:
    if vocab < 1:
        raise ValueError(vocab)
    for w, cap in ((1, 1 << 8), (2, 1 << 16), (4, 1 << 32)):
        if vocab <= cap:
            return w
    raise ValueError(vocab)


def parse_header(buf: bytes, file_size: int):
    if file_size < HEADER.size:
        raise OracleFormatError("short")
    magic, ver, w, count, ndocs, off = HEADER.unpack(buf[: HEADER.size])
    if magic != b"CFPKD001" or ver != 1 or w not in (1, 2, 4):
        raise OracleFormatError("header")
    if off != HEADER.size + count * w or file_size != off + 16 * ndocs:
        raise OracleFormatError("length")
    return w, count, ndocs, off


def sample_count(n_tok: int, L: int) -> int:
    if L < 1:
        raise ValueError(L)
    return 0 if n_tok == 0 else (n_tok - 1) // L


def sample_window(payload: np.ndarray, s: int, L: int) -> np.ndarray:
    if not 0 <= s < sample_count(payload.size, L):
        raise IndexError(s)
    return payload[s * L : s * L + L + 1]


def batch_windows(payload: np.ndarray, ids, L: int):
    """(inputs, targets) int64 [B, L] for sample ids, via one get_sample per id."""
    rows = [sample_window(payload, int(s), L).astype(np.int64) for s in ids]
    if not rows:
        z = np.zeros((0, L), np.int64)
        return z, z.copy()
    win = np.stack(rows)
    return win[:, :L].copy(), win[:, 1:].copy()


def _mix(state: int):
    state = (state + 0x9E3779B97F4A7C15) & M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return state, z ^ (z >> 31)


def splitmix64_first(seed: int, k: int) -> list[int]:
    st = seed & M64
    out = []
    for _ in range(k):
        st, x = _mix(st)
        out.append(x)
    return out


def permutation(n: int, seed: int) -> np.ndarray:
    order = list(range(n))
    st = seed & M64
    for i in range(n - 1, 0, -1):
        b = i + 1
        lim = ((1 << 64) // b) * b
        while True:
            st, x = _mix(st)
            if x < lim:
                break
        j = x % b
        order[i], order[j] = order[j], order[i]
    return np.asarray(order, dtype=np.uint64)


def chunk_sizes(n: int, k: int) -> list[int]:
    if not 1 <= k <= max(1, n):
        raise ValueError(k)
    q, r = divmod(n, k)
    return [q + 1 if c < r else q for c in range(k)]


def materialize_bytes(buf: bytes, docs) -> bytes:
    """ORACLE: the CFPKD001 file materialize_chunk (packed_data.py:336-344) writes for
    the documents ``docs`` of the packed file ``buf``: header, the documents' tokens
    in order, the rebuilt contiguous span index (packed_data.py:62-131 writer layout)."""
    width, count, ndoc, index_off = parse_header(buf, len(buf))
    dt = {1: "<u1", 2: "<u2", 4: "<u4"}[width]
    payload = np.frombuffer(buf, dt, count, 40)
    spans = np.frombuffer(buf, "<u8", 2 * ndoc, index_off).reshape(ndoc, 2)
    parts, lens = [], []
    for d in docs:
        s, n = int(spans[int(d), 0]), int(spans[int(d), 1])
        parts.append(payload[s:s + n])
        lens.append(n)
    body = np.concatenate(parts).astype(dt).tobytes() if parts else b""
    lens = np.asarray(lens, dtype="<u8")
    out_spans = np.zeros((len(lens), 2), dtype="<u8")
    out_spans[:, 1] = lens
    if len(lens) > 1:
        out_spans[1:, 0] = np.cumsum(lens[:-1])
    total = int(lens.sum()) if len(lens) else 0
    hdr = struct.pack("<8sIIQQQ", b"CFPKD001", 1, width, total, len(lens), 40 + total * width)
    return hdr + body + out_spans.tobytes()
