"""The ``dataset`` / ``sampler`` / ``dataloader`` components of the training step.

The reference leaves sample order and the rank split to consumers
(SPEC.md:490); this build fixes them so that W ranks with per-rank batch B see
exactly the samples of a 1-rank run with batch W*B:

    position q = (step * W + rank) * B + b,   sample id = order[q]

with order = identity (sequential) or make_permutation(sample_count, seed)
(packed_data.py:257-282). The remainder that does not fill a global batch
is dropped.

Two feeds, both ending in the same widening kernel:
  * resident: the packed payload is uploaded to HBM once; per step only the
    B sample ids cross PCIe and ``b2s_gather_samples`` reads the windows.
  * staged (end-to-end): per step the B windows of L+1 tokens are copied from
    the host memory map into pinned memory, then H2D, then
    ``b2s_unpack_windows`` widens/splits them.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib
from .packed import DevicePackedStream, OutOfRangeError, PackedReader, PackedWriter, make_permutation, open_packed


class Sampler:
    """Global sample order over a packed stream (sequential or seeded permutation)."""

    def __init__(self, shuffle: bool = False, seed: int = 0):
        self.shuffle = shuffle
        self.seed = seed

    def order(self, n: int) -> np.ndarray:
        if self.shuffle:
            return make_permutation(n, self.seed).order
        return np.arange(n, dtype=np.uint64)


class PackedDataLoader:
    def __init__(self, dataset: PackedReader, batch_size: int, seq_len: int, sampler: Sampler | None = None,
                 feed: str = "resident"):
        if batch_size < 1 or seq_len < 1:
            raise ValueError("batch_size and seq_len must be >= 1")
        if feed not in ("resident", "staged"):
            raise ValueError(f"feed must be resident or staged, got {feed!r}")
        self.dataset = dataset
        self.batch_size = batch_size
        self.seq_len = seq_len
        self.sampler = sampler or Sampler()
        self.feed = feed
        self.rank, self.world, self.device = 0, 1, None
        self._order = None
        self._dev = None

    def bind(self, rank: int, world: int, device, vocab_size: int | None = None) -> "PackedDataLoader":
        """Attach to (rank, world, device). With ``vocab_size`` (the trainer passes the model's),
        a corpus holding any token id >= vocab_size is rejected here: the embedding and
        cross-entropy kernels index weight rows by token id and would otherwise read or
        scatter-add outside the tables."""
        if vocab_size is not None:
            mx = self.dataset.max_token()
            if mx >= vocab_size:
                raise ValueError(f"dataset holds token id {mx}, outside the model's vocabulary of {vocab_size}")
        self.rank, self.world, self.device = rank, world, torch.device(device)
        n = self.dataset.sample_count(self.seq_len)
        self._order = self.sampler.order(n)
        if self.device.type != "cuda":  # host-side use (sample_ids only), e.g. gloo tests
            return self
        B, L = self.batch_size, self.seq_len
        self._in = torch.empty(B, L, dtype=torch.int64, device=self.device)
        self._tg = torch.empty(B, L, dtype=torch.int64, device=self.device)
        # Pinned host staging is a ring: the host may run several steps ahead of
        # the GPU (CUDA-graph replay makes a step a handful of launches), so a
        # buffer is rewritten only after the H2D copy that last read it has run.
        self._ring = [None] * self.RING
        self._slot = 0
        if self.feed == "resident":
            self._dev = DevicePackedStream(self.dataset, self.device)
            self._ids_host = [torch.empty(B, dtype=torch.int64, pin_memory=True) for _ in range(self.RING)]
            self._ids_dev = torch.empty(B, dtype=torch.int64, device=self.device)
        else:
            w = self.dataset.token_width
            self._stage_host = [torch.empty(B * (L + 1) * w, dtype=torch.uint8, pin_memory=True)
                                for _ in range(self.RING)]
            self._stage_dev = torch.empty(B * (L + 1) * w + 16, dtype=torch.uint8, device=self.device)
        return self

    RING = 4

    def _host_slot(self) -> int:
        """Next pinned staging buffer, waiting for the copy that last read it."""
        i = self._slot
        self._slot = (i + 1) % self.RING
        if self._ring[i] is not None:
            self._ring[i].synchronize()
        return i

    def _copied(self, i: int) -> None:
        ev = torch.cuda.Event()
        ev.record()
        self._ring[i] = ev

    @property
    def steps_available(self) -> int:
        return len(self._order) // (self.world * self.batch_size)

    def sample_ids(self, step: int) -> np.ndarray:
        B, W = self.batch_size, self.world
        if not 0 <= step < self.steps_available:
            raise OutOfRangeError(f"step {step} out of range [0, {self.steps_available})")
        q0 = (step * W + self.rank) * B
        return self._order[q0:q0 + B]

    def h2d_bytes_per_step(self) -> int:
        if self.feed == "resident":
            return self.batch_size * 8
        return self.batch_size * (self.seq_len + 1) * self.dataset.token_width

    def batch(self, step: int):
        """(inputs, targets) int64 [B, L] on the bound device for global step `step`."""
        ids = self.sample_ids(step)
        B, L = self.batch_size, self.seq_len
        stream = _lib.stream_ptr()
        i = self._host_slot()
        if self.feed == "resident":
            self._ids_host[i].numpy()[:] = ids.view(np.int64)
            self._ids_dev.copy_(self._ids_host[i], non_blocking=True)
            self._copied(i)
            _lib.call("b2s_gather_samples", self._dev.payload.data_ptr(), self._dev.token_width,
                      self._dev.token_count, self._ids_dev.data_ptr(), B, L, self._in.data_ptr(),
                      self._tg.data_ptr(), self._dev.status.data_ptr(), stream)
        else:
            w = self.dataset.token_width
            pay = self.dataset.payload
            host = self._stage_host[i].numpy().view(pay.dtype).reshape(B, L + 1)
            for b, s in enumerate(ids):
                lo = int(s) * L
                host[b] = pay[lo:lo + L + 1]
            self._stage_dev[: B * (L + 1) * w].copy_(self._stage_host[i], non_blocking=True)
            self._copied(i)
            _lib.call("b2s_unpack_windows", self._stage_dev.data_ptr(), w, B, L, self._in.data_ptr(),
                      self._tg.data_ptr(), stream)
        return self._in, self._tg


def open_dataset(path: str) -> PackedReader:
    return open_packed(path)


def make_synthetic_packed(path: str, n_tokens: int, vocab_size: int, doc_len: int = 1024, kind: str = "markov",
                          seed: int = 0) -> str:
    """Seeded synthetic CFPKD001 corpus.

    markov: each token has 8 fixed random successors, starts are Zipf-like and
    every document ends with eod = vocab-1, so the loss is learnable.
    uniform: i.i.d. uniform ids (pure throughput runs).
    """
    from .packed import token_width_for_vocab

    rng = np.random.default_rng(seed)
    V = vocab_size
    ndocs = -(-n_tokens // doc_len)
    if kind == "uniform":
        toks = rng.integers(0, V - 1, size=(ndocs, doc_len), dtype=np.int64)
    elif kind == "markov":
        succ = rng.integers(0, V - 1, size=(V, 8), dtype=np.int64)
        ranks = np.arange(1, V, dtype=np.float64)
        p = 1.0 / ranks
        p /= p.sum()
        toks = np.empty((ndocs, doc_len), dtype=np.int64)
        toks[:, 0] = rng.choice(V - 1, size=ndocs, p=p)
        choice = rng.integers(0, 8, size=(ndocs, doc_len), dtype=np.int64)
        for t in range(1, doc_len):
            toks[:, t] = succ[toks[:, t - 1], choice[:, t]]
    else:
        raise ValueError(f"unknown synthetic kind {kind!r}")
    toks[:, -1] = V - 1  # eod
    flat = toks.reshape(-1)[:n_tokens]
    with PackedWriter(path, token_width_for_vocab(V)) as w:
        w.write_stream(flat, doc_len)
    return path


def synthetic_path(root: str, n_tokens: int, vocab_size: int, kind: str = "markov", seed: int = 0) -> str:
    os.makedirs(root, exist_ok=True)
    path = os.path.join(root, f"synthetic_{kind}_v{vocab_size}_n{n_tokens}_s{seed}.cfpk")
    if not os.path.exists(path):
        tmp = path + f".tmp{os.getpid()}"
        make_synthetic_packed(tmp, n_tokens, vocab_size, kind=kind, seed=seed)
        os.replace(tmp, path)
    return path
