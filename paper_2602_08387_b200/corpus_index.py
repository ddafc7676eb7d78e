"""Byte-span index of a raw JSONL corpus, built by a GPU newline scan.

Same surface and file format as the reference ``corpusforge.corpus_index``
(corpus_index.py:1-148): ``build_index`` records the (byte_offset, byte_length)
of every non-empty newline-terminated line (0x0A is the only boundary; a final
line without a trailing newline still counts; zero-length lines are dropped),
``write_index`` / ``load_index`` use the CFIDX001 sidecar
(``<8sIQQ`` = magic, version, source_size, doc_count, then doc_count x 2 u64).

The O(bytes) part -- finding the newlines -- runs on the GPU
(``b2s_newline_count`` / ``b2s_newline_positions``): the file is streamed to HBM
in pieces, each piece scanned with 16-byte vector loads; spans follow from the
ordered newline positions with one vectorised diff on the host. The result does
not depend on ``buffer_size`` (the reference's read-chunk size, kept for API
parity) nor on the piece size.
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from . import _lib

INDEX_MAGIC = b"CFIDX001"
INDEX_VERSION = 1
DEFAULT_BUFFER_SIZE = 1 << 20
_IDX_HDR = struct.Struct("<8sIQQ")
_PIECE = 1 << 28  # bytes streamed to the GPU per scan


class FormatError(Exception):
    """Malformed index sidecar."""


class OutOfRangeError(IndexError):
    """Document ordinal outside the index."""


class DocSpan(NamedTuple):
    byte_offset: int
    byte_length: int


@dataclass(eq=False)
class DocumentIndex:
    source_size: int
    spans: np.ndarray  # (doc_count, 2) uint64: byte_offset, byte_length

    @property
    def doc_count(self) -> int:
        return int(self.spans.shape[0])

    def span(self, i: int) -> DocSpan:
        if not 0 <= i < self.doc_count:
            raise OutOfRangeError(f"document {i} out of range [0, {self.doc_count})")
        return DocSpan(int(self.spans[i, 0]), int(self.spans[i, 1]))

    def __eq__(self, other) -> bool:
        if not isinstance(other, DocumentIndex):
            return NotImplemented
        return self.source_size == other.source_size and np.array_equal(self.spans, other.spans)


def _newline_positions_gpu(data: np.ndarray, device) -> np.ndarray:
    """Ascending byte positions of 0x0A in ``data`` (uint8), scanned on the GPU."""
    import torch

    n_total = int(data.size)
    out = []
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ValueError("the corpus index scan runs on a CUDA device (no CPU fallback)")
    buf = torch.empty(min(n_total, _PIECE) + 16, dtype=torch.uint8, device=dev)
    for p0 in range(0, n_total, _PIECE):
        n = min(_PIECE, n_total - p0)
        buf[:n].copy_(torch.from_numpy(data[p0:p0 + n]))
        nblocks = max(1, min(148 * 8, (n + 4095) // 4096))
        chunk = ((-(-n // nblocks)) + 15) // 16 * 16
        nblocks = -(-n // chunk)
        counts = torch.empty(nblocks, dtype=torch.int32, device=dev)
        st = _lib.stream_ptr()
        _lib.call("b2s_newline_count", buf.data_ptr(), n, chunk, counts.data_ptr(), nblocks, st)
        c = counts.cpu().numpy().astype(np.int64)
        offs = np.zeros(nblocks, dtype=np.int64)
        np.cumsum(c[:-1], out=offs[1:])
        total = int(c.sum())
        pos = torch.empty(max(1, total), dtype=torch.int64, device=dev)
        if total:
            d_offs = torch.from_numpy(offs).to(dev)
            _lib.call("b2s_newline_positions", buf.data_ptr(), n, chunk, d_offs.data_ptr(), nblocks, p0,
                      pos.data_ptr(), st)
            out.append(pos[:total].cpu().numpy().view(np.uint64))
    return np.concatenate(out) if out else np.zeros(0, dtype=np.uint64)


def build_index(raw_path, buffer_size: int = DEFAULT_BUFFER_SIZE, device="cuda") -> DocumentIndex:
    """Index every non-empty line of ``raw_path`` (reference corpus_index.py:68-107)."""
    if buffer_size < 1:
        raise ValueError(f"buffer_size must be >= 1, got {buffer_size}")
    size = os.path.getsize(raw_path)
    data = np.fromfile(raw_path, dtype=np.uint8) if size else np.zeros(0, dtype=np.uint8)
    nl = _newline_positions_gpu(data, device).astype(np.int64)
    starts = np.empty(nl.size, dtype=np.int64)
    starts[:1] = 0
    starts[1:] = nl[:-1] + 1
    lens = nl - starts
    keep = lens > 0
    starts, lens = starts[keep], lens[keep]
    tail = int(nl[-1]) + 1 if nl.size else 0
    if tail < size:  # final line without a trailing newline
        starts = np.append(starts, tail)
        lens = np.append(lens, size - tail)
    spans = np.empty((starts.size, 2), dtype="<u8")
    spans[:, 0] = starts
    spans[:, 1] = lens
    return DocumentIndex(source_size=size, spans=spans)


def write_index(index: DocumentIndex, path) -> None:
    with open(path, "wb") as f:
        f.write(_IDX_HDR.pack(INDEX_MAGIC, INDEX_VERSION, index.source_size, index.doc_count))
        f.write(np.ascontiguousarray(index.spans, dtype="<u8").tobytes())


def load_index(path) -> DocumentIndex:
    data = open(path, "rb").read()
    if len(data) < _IDX_HDR.size:
        raise FormatError(f"{path}: truncated index header")
    magic, version, source_size, n = _IDX_HDR.unpack_from(data)
    if magic != INDEX_MAGIC:
        raise FormatError(f"{path}: bad magic {magic!r}")
    if version != INDEX_VERSION:
        raise FormatError(f"{path}: unsupported version {version}")
    if len(data) != _IDX_HDR.size + 16 * n:
        raise FormatError(f"{path}: truncated span table")
    spans = np.frombuffer(data, "<u8", 2 * n, _IDX_HDR.size).reshape(n, 2).copy()
    return DocumentIndex(source_size=source_size, spans=spans)


def index_sidecar_path(raw_path) -> str:
    return os.fspath(raw_path) + ".didx"


def verify_index(index: DocumentIndex, raw_path) -> bool:
    """Size-only staleness check (reference corpus_index.py:131-138)."""
    return os.path.getsize(raw_path) == index.source_size


def read_document(raw_path, index: DocumentIndex, i: int) -> bytes:
    off, n = index.span(i)
    with open(raw_path, "rb") as f:
        f.seek(off)
        return f.read(n)
