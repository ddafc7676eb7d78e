"""CFPKD001 packed token stream: host reader/writer and the GPU sample indexer.

Mirrors the public surface of the reference ``corpusforge.packed_data`` so a
caller can switch imports (same names, argument meaning and exceptions):

===========================  ======================================
reference (packed_data.py)   here
===========================  ======================================
FormatError :37-38           FormatError
OutOfRangeError :41-42       OutOfRangeError (an IndexError)
InvalidKError :45-46         InvalidKError (a ValueError)
token_width_for_vocab :49    token_width_for_vocab -> C-ABI
PackedWriter :62-131         PackedWriter
PackedReader :134-215        PackedReader
open_packed :218-220         open_packed
splitmix64 :226-238          splitmix64 -> C-ABI (host)
make_permutation :257-282    make_permutation -> C-ABI (host)
write/load_permutation       write_permutation / load_permutation
chunk :322-333               chunk -> C-ABI bounds
materialize_chunk :336-344   materialize_chunk
===========================  ======================================

The training step does not call ``get_sample`` per sample. It uploads the
payload to HBM once (:class:`DevicePackedStream`) and gathers a whole batch
of windows with one kernel (``b2s_gather_samples``), bit-exact with
``get_sample`` followed by the ids[:L] / ids[1:] split.
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib

PACKED_MAGIC = b"CFPKD001"
PACKED_VERSION = 1
PERM_MAGIC = b"CFPRM001"
PERM_VERSION = 1
HEADER_SIZE = 40  # <8sIIQQQ: magic, version, width, token_count, doc_count, index_offset
SPAN_BYTES = 16
_HDR = struct.Struct("<8sIIQQQ")
_PERM_HDR = struct.Struct("<8sIQQ")
_WIDTH_DTYPE = {1: np.dtype("<u1"), 2: np.dtype("<u2"), 4: np.dtype("<u4")}
_MASK64 = (1 << 64) - 1


class FormatError(Exception):
    """Malformed packed file or permutation sidecar."""


class OutOfRangeError(IndexError):
    """Document or sample ordinal outside the file's range."""


class InvalidKError(ValueError):
    """Chunk count outside [1, max(1, n)]."""


def token_width_for_vocab(vocab_size: int) -> int:
    if vocab_size < 1 or vocab_size > (1 << 32):
        # same message family as the reference; the C-ABI rejects both cases
        raise ValueError(f"vocab_size {vocab_size} is not representable in a 1/2/4-byte token")
    w = _lib.c_int()
    _lib.call("b2s_token_width_for_vocab", vocab_size, _lib.ctypes.byref(w))
    return w.value


class PackedWriter:
    """Streaming CFPKD001 writer: placeholder header, payload, span index, header patch."""

    def __init__(self, path, token_width: int):
        if token_width not in _WIDTH_DTYPE:
            raise ValueError(f"token_width must be one of 1, 2, 4; got {token_width}")
        self.path = os.fspath(path)
        self.token_width = token_width
        self._f = open(self.path, "wb")
        self._f.write(bytes(HEADER_SIZE))
        self._lengths: list[int] = []
        self._token_count = 0
        self._closed = False

    def write_document(self, ids) -> None:
        arr = np.asarray(ids, dtype=_WIDTH_DTYPE[self.token_width])
        if arr.ndim != 1:
            raise ValueError("token ids must be a flat sequence")
        self._lengths.append(int(arr.size))
        self._token_count += int(arr.size)
        self._f.write(arr.tobytes())

    def write_stream(self, tokens, doc_len: int) -> None:
        """Bulk form of write_document: consecutive documents of ``doc_len`` tokens."""
        arr = np.ascontiguousarray(tokens, dtype=_WIDTH_DTYPE[self.token_width])
        n = int(arr.size)
        full, rem = divmod(n, doc_len)
        self._lengths.extend([doc_len] * full + ([rem] if rem else []))
        self._token_count += n
        self._f.write(arr.tobytes())

    @property
    def doc_count(self) -> int:
        return len(self._lengths)

    @property
    def token_count(self) -> int:
        return self._token_count

    def close(self) -> None:
        if self._closed:
            return
        lengths = np.asarray(self._lengths, dtype="<u8")
        spans = np.empty((lengths.size, 2), dtype="<u8")
        spans[:, 1] = lengths
        spans[:, 0] = np.cumsum(lengths) - lengths if lengths.size else lengths
        self._f.write(spans.tobytes())
        self._f.seek(0)
        index_offset = HEADER_SIZE + self._token_count * self.token_width
        self._f.write(_HDR.pack(PACKED_MAGIC, PACKED_VERSION, self.token_width,
                                self._token_count, lengths.size, index_offset))
        self._f.close()
        self._closed = True

    def __enter__(self):
        return self

    def __exit__(self, exc_type, exc, tb):
        if exc_type is None:
            self.close()
        else:  # leave an unpatched (invalid) file behind, like the reference (:126-131)
            self._f.close()
            self._closed = True


class PackedReader:
    """Read-only memory-mapped view of a CFPKD001 file; immutable after open."""

    def __init__(self, path):
        self.path = os.fspath(path)
        size = os.path.getsize(self.path)
        if size < HEADER_SIZE:
            raise FormatError(f"{self.path}: file shorter than the {HEADER_SIZE}-byte header")
        with open(self.path, "rb") as f:
            magic, version, width, count, ndocs, index_offset = _HDR.unpack(f.read(HEADER_SIZE))
        if magic != PACKED_MAGIC:
            raise FormatError(f"{self.path}: bad magic {magic!r}")
        if version != PACKED_VERSION:
            raise FormatError(f"{self.path}: unsupported version {version}")
        if width not in _WIDTH_DTYPE:
            raise FormatError(f"{self.path}: invalid token width {width}")
        if index_offset != HEADER_SIZE + count * width:
            raise FormatError(f"{self.path}: index_offset {index_offset} does not match "
                              f"{HEADER_SIZE} + {count} * {width}")
        if size != index_offset + ndocs * SPAN_BYTES:
            raise FormatError(f"{self.path}: file length {size} does not match header "
                              f"(expected {index_offset + ndocs * SPAN_BYTES})")
        self.token_width = width
        self.token_count = count
        self.doc_count = ndocs
        mm = np.memmap(self.path, dtype=np.uint8, mode="r")
        self._mm = mm
        self._payload = mm[HEADER_SIZE:index_offset].view(_WIDTH_DTYPE[width])
        self._spans = mm[index_offset:].view("<u8").reshape(ndocs, 2)

    @property
    def payload(self) -> np.ndarray:
        return self._payload

    @property
    def spans(self) -> np.ndarray:
        return self._spans

    def get_document_tokens(self, i: int) -> np.ndarray:
        if not 0 <= i < self.doc_count:
            raise OutOfRangeError(f"document {i} out of range [0, {self.doc_count})")
        start, length = (int(x) for x in self._spans[i])
        return self._payload[start:start + length]

    def sample_count(self, seq_len: int) -> int:
        if seq_len < 1:
            raise ValueError(f"seq_len must be >= 1, got {seq_len}")
        n = _lib.c_uint64()
        _lib.call("b2s_sample_count", self.token_count, seq_len, _lib.ctypes.byref(n))
        return n.value

    def get_sample(self, s: int, seq_len: int) -> np.ndarray:
        n = self.sample_count(seq_len)
        if not 0 <= s < n:
            raise OutOfRangeError(f"sample {s} out of range [0, {n}) for L={seq_len}")
        lo = s * seq_len
        return self._payload[lo:lo + seq_len + 1]

    def max_token(self) -> int:
        """Largest token id in the payload (-1 if empty); one host scan, cached (the reader is
        immutable). The training feed checks it against the model's vocabulary once."""
        if getattr(self, "_max_token", None) is None:
            self._max_token = int(self._payload.max()) if self.token_count else -1
        return self._max_token

    def close(self) -> None:
        self._payload = self._spans = None
        self._mm = None

    def __enter__(self):
        return self

    def __exit__(self, exc_type, exc, tb):
        self.close()


def open_packed(path) -> PackedReader:
    return PackedReader(path)


# --- seeded shuffling (host C++) -------------------------------------------------


def splitmix64(state: int, count: int) -> np.ndarray:
    """First ``count`` SplitMix64 outputs for ``state`` (the reference yields lazily)."""
    out = np.empty(count, dtype="<u8")
    _lib.call("b2s_splitmix64", state & _MASK64, count, out.ctypes.data)
    return out


@dataclass
class Permutation:
    seed: int
    order: np.ndarray

    def __eq__(self, other):
        if not isinstance(other, Permutation):
            return NotImplemented
        return self.seed == other.seed and np.array_equal(self.order, other.order)

    def __len__(self):
        return len(self.order)


def make_permutation(n: int, seed: int) -> Permutation:
    if n < 0:
        raise ValueError(f"n must be >= 0, got {n}")
    order = np.empty(n, dtype="<u8")
    _lib.call("b2s_make_permutation", n, seed & _MASK64, order.ctypes.data)
    return Permutation(seed=seed, order=order)


def write_permutation(perm: Permutation, path) -> None:
    if not 0 <= perm.seed <= _MASK64:
        # the reference fails inside struct.pack here; say why
        raise ValueError(f"permutation seed {perm.seed} is not a uint64; mask it first")
    with open(path, "wb") as f:
        f.write(_PERM_HDR.pack(PERM_MAGIC, PERM_VERSION, perm.seed, len(perm.order)))
        f.write(np.asarray(perm.order, dtype="<u8").tobytes())


def load_permutation(path) -> Permutation:
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < _PERM_HDR.size:
        raise FormatError(f"{path}: truncated permutation header")
    magic, version, seed, n = _PERM_HDR.unpack_from(data)
    if magic != PERM_MAGIC:
        raise FormatError(f"{path}: bad magic {magic!r}")
    if version != PERM_VERSION:
        raise FormatError(f"{path}: unsupported version {version}")
    if len(data) != _PERM_HDR.size + 8 * n:
        raise FormatError(f"{path}: truncated permutation body")
    return Permutation(seed=seed, order=np.frombuffer(data, "<u8", n, _PERM_HDR.size).copy())


@dataclass
class ChunkSpec:
    chunk_count: int
    assignments: list


def chunk(perm: Permutation, k: int) -> ChunkSpec:
    n = len(perm.order)
    if not 1 <= k <= max(1, n):
        raise InvalidKError(f"k must be in [1, {max(1, n)}], got {k}")
    lo = np.empty(k + 1, dtype="<u8")
    _lib.call("b2s_chunk_bounds", n, k, lo.ctypes.data)
    return ChunkSpec(k, [perm.order[int(lo[c]):int(lo[c + 1])] for c in range(k)])


def materialize_chunk(reader: PackedReader, docs, out_path) -> None:
    with PackedWriter(out_path, reader.token_width) as w:
        for d in docs:
            w.write_document(reader.get_document_tokens(int(d)))


def materialize_chunk_gpu(reader: PackedReader, docs, out_path, device="cuda", stream=None) -> None:
    """``materialize_chunk`` with the token copy on the GPU.

    Same output bytes as the host path (reference packed_data.py:336-344): the
    documents ``docs`` (ordinals into ``reader``), in order, as a standalone
    CFPKD001 file with a rebuilt contiguous span index. ``stream`` may be a
    ``DevicePackedStream`` of ``reader`` whose payload is already resident in HBM
    (the training-time case); otherwise the payload is copied to ``device``.
    """
    import torch

    docs = np.asarray(docs, dtype=np.int64).reshape(-1)
    n = reader.doc_count
    bad = docs[(docs < 0) | (docs >= n)]
    if bad.size:
        raise OutOfRangeError(f"document {int(bad[0])} out of range [0, {n})")
    ds = stream if stream is not None else DevicePackedStream(reader, device)
    spans = np.asarray(reader.spans, dtype=np.uint64)
    src = spans[docs, 0] if docs.size else np.zeros(0, np.uint64)
    lens = spans[docs, 1] if docs.size else np.zeros(0, np.uint64)
    dst = np.zeros(docs.size, dtype=np.uint64)
    if docs.size > 1:
        np.cumsum(lens[:-1], out=dst[1:])
    total = int(lens.sum()) if docs.size else 0
    w = reader.token_width
    dev = ds.payload.device
    out = torch.empty(max(16, total * w), dtype=torch.uint8, device=dev)
    if docs.size:
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)  # noqa: E731
        d_src, d_len, d_dst = t(src), t(lens), t(dst)
        _lib.call("b2s_gather_documents", ds.payload.data_ptr(), w, d_src.data_ptr(), d_len.data_ptr(),
                  d_dst.data_ptr(), int(docs.size), out.data_ptr(), _lib.stream_ptr())
    payload = out[: total * w].cpu().numpy()
    out_spans = np.empty((docs.size, 2), dtype="<u8")
    out_spans[:, 0] = dst
    out_spans[:, 1] = lens
    with open(out_path, "wb") as f:
        f.write(_HDR.pack(PACKED_MAGIC, PACKED_VERSION, w, total, int(docs.size), HEADER_SIZE + total * w))
        f.write(payload.tobytes())
        f.write(out_spans.tobytes())


# --- GPU side ---------------------------------------------------------------------


class DevicePackedStream:
    """The packed payload resident in HBM plus the batched sample gather (K1).

    ``gather(ids)`` returns ``(inputs, targets)`` int64 tensors of shape [B, L]
    equal to ``get_sample(s, L)[:L]`` / ``[1:]`` for every id, computed by
    ``b2s_gather_samples`` on the current stream.
    """

    def __init__(self, reader: PackedReader, device="cuda"):
        import torch

        self.token_width = reader.token_width
        self.token_count = reader.token_count
        nbytes = reader.token_count * reader.token_width
        host = torch.from_numpy(np.asarray(reader.payload).view(np.uint8)[:nbytes].copy())
        # pad to 16 B so vectorised readers may overrun the tail safely
        self.payload = torch.zeros(((nbytes + 15) // 16) * 16, dtype=torch.uint8, device=device)
        self.payload[:nbytes].copy_(host)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        self._reader = reader

    def sample_count(self, seq_len: int) -> int:
        return self._reader.sample_count(seq_len)

    @staticmethod
    def _check(host_ids: np.ndarray, n: int, seq_len: int) -> None:
        bad = host_ids[host_ids >= n]
        if bad.size:
            raise OutOfRangeError(f"sample {int(bad[0])} out of range [0, {n}) for L={seq_len}")

    def gather(self, sample_ids, seq_len: int, out=None, check: bool = True):
        import torch

        n = self.sample_count(seq_len)
        if isinstance(sample_ids, torch.Tensor):
            ids = sample_ids.view(torch.int64)
            if check:  # device ids: validate on the host copy (a sync; tests only)
                self._check(ids.detach().cpu().numpy().view(np.uint64), n, seq_len)
        else:
            host_ids = np.ascontiguousarray(sample_ids, dtype=np.uint64)
            if check:
                self._check(host_ids, n, seq_len)
            ids = torch.from_numpy(host_ids.view(np.int64))
        ids = ids.to(self.payload.device, non_blocking=True)
        B = ids.numel()
        if out is None:
            inputs = torch.empty(B, seq_len, dtype=torch.int64, device=self.payload.device)
            targets = torch.empty_like(inputs)
        else:
            inputs, targets = out
        _lib.call("b2s_gather_samples", self.payload.data_ptr(), self.token_width, self.token_count,
                  ids.data_ptr(), B, seq_len, inputs.data_ptr(), targets.data_ptr(),
                  self.status.data_ptr(), _lib.stream_ptr())
        return inputs, targets
