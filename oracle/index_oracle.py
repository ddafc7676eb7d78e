"""ORACLE -- test infrastructure only (tests/ may import it; the product never does).

Restatement of corpusforge.corpus_index.build_index (reference corpus_index.py:68-107):
a document is every maximal run of bytes between newline (0x0A) bytes that is
non-empty; a final run without a trailing newline counts. Pinned to the
reference by tests/golden/packed_golden.json["corpus_index"].
"""

from __future__ import annotations

import numpy as np


def spans(data: bytes) -> np.ndarray:
    """(doc_count, 2) uint64 (byte_offset, byte_length) of the non-empty lines of ``data``."""
    out = []
    start = 0
    for i, b in enumerate(data):
        if b == 0x0A:
            if i > start:
                out.append((start, i - start))
            start = i + 1
    if start < len(data):
        out.append((start, len(data) - start))
    return np.asarray(out, dtype=np.uint64).reshape(-1, 2)


def spans_fast(data: bytes) -> np.ndarray:
    """Same answer as ``spans`` vectorised with numpy (for large property tests)."""
    a = np.frombuffer(data, dtype=np.uint8)
    nl = np.flatnonzero(a == 0x0A).astype(np.int64)
    starts = np.concatenate([[0], nl[:-1] + 1]) if nl.size else np.zeros(0, np.int64)
    lens = nl - starts
    keep = lens > 0
    starts, lens = starts[keep], lens[keep]
    tail = int(nl[-1]) + 1 if nl.size else 0
    if tail < a.size:
        starts, lens = np.append(starts, tail), np.append(lens, a.size - tail)
    return np.stack([starts, lens], 1).astype(np.uint64).reshape(-1, 2)
