"""Tokenization of an indexed JSONL corpus into a packed file.

Same surface as the reference ``corpusforge.pipeline`` (pipeline.py:1-422):
``run_pipeline(raw_path, index, tokenizer, cfg) -> PipelineStats`` with
``PipelineConfig`` / ``PipelineError`` / ``StaleIndexError`` / ``Skip`` /
``extract_text``. The producer is the library's C++ thread pool
(``b2s_tokenize_corpus``): ``cfg.workers`` threads tokenize batches of
``cfg.batch_size`` documents (the reference forks worker processes and pickles
batches through queues) and the writer restores batch order, so the CFPKD001
output is byte-identical for any worker count -- and to the reference's.
The reorder window is bounded by construction (workers wait when they run
``4 * workers + 8`` batches ahead of the writer), so ``reorder_cap`` /
``ReorderOverflowError`` are kept for API parity only.
"""

from __future__ import annotations

import ctypes
import enum
import json
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .corpus_index import DocumentIndex, verify_index
from .packed import token_width_for_vocab
from .tokenizers import Tokenizer


class PipelineError(Exception):
    """A pipeline stage failed; the packed output is not usable."""


class StaleIndexError(PipelineError):
    """The raw file changed size since its index was built."""


class ReorderOverflowError(PipelineError):
    """Kept for API parity (the C++ writer's reorder window is bounded by construction)."""


class Skip(enum.Enum):
    MALFORMED = "malformed"
    MISSING_TEXT = "missing_text"


def extract_text(raw: bytes, text_key: str = "text"):
    """The text field of one raw JSONL document, or a Skip reason (reference pipeline.py:50-68).
    Host helper for API parity; the C++ producer applies the same rules per document."""
    try:
        obj = json.loads(raw)
    except ValueError:
        return Skip.MALFORMED
    if not isinstance(obj, dict):
        return Skip.MALFORMED
    value = obj.get(text_key)
    return value if isinstance(value, str) else Skip.MISSING_TEXT


def default_workers() -> int:
    return max(1, (os.cpu_count() or 1) - 2)


@dataclass
class PipelineConfig:
    out_path: str
    workers: int = field(default_factory=default_workers)
    batch_size: int = 128
    queue_capacity: int = 8
    append_eod: bool = True
    text_key: str = "text"
    reorder_cap: int | None = None

    def __post_init__(self) -> None:
        if self.workers < 1:
            raise ValueError(f"workers must be >= 1, got {self.workers}")
        if self.batch_size < 1:
            raise ValueError(f"batch_size must be >= 1, got {self.batch_size}")
        if self.queue_capacity < 1:
            raise ValueError(f"queue_capacity must be >= 1, got {self.queue_capacity}")

    def resolved_reorder_cap(self) -> int:
        if self.reorder_cap is not None:
            return self.reorder_cap
        return max(4 * self.queue_capacity, self.workers + 2 * self.queue_capacity)


@dataclass
class PipelineStats:
    documents: int
    skipped: int
    malformed: int
    tokens: int
    elapsed: float
    throughput: float

    def summary(self) -> dict:
        return {"documents": self.documents, "skipped": self.skipped, "malformed": self.malformed,
                "tokens": self.tokens, "seconds": round(self.elapsed, 3),
                "tokens_per_sec": round(self.throughput, 1)}


def run_pipeline(raw_path, index: DocumentIndex, tokenizer: Tokenizer, cfg: PipelineConfig) -> PipelineStats:
    """Tokenize every indexed document of ``raw_path`` into ``cfg.out_path``."""
    if not verify_index(index, raw_path):
        raise StaleIndexError(f"{raw_path}: size changed since indexing; rebuild the index")
    if cfg.append_eod and tokenizer.eod_token_id is None:
        raise ValueError("append_eod is enabled but the tokenizer has no eod_token_id")
    width = token_width_for_vocab(tokenizer.vocab_size)
    spans = np.ascontiguousarray(index.spans, dtype=np.uint64)
    stats = (ctypes.c_int64 * 4)()
    t0 = time.perf_counter()
    rc = _lib.load().b2s_tokenize_corpus(
        os.fsencode(raw_path), spans.ctypes.data, int(spans.shape[0]), tokenizer.handle,
        cfg.text_key.encode("utf-8"), int(cfg.append_eod), width, cfg.workers, cfg.batch_size,
        os.fsencode(cfg.out_path), ctypes.addressof(stats))
    elapsed = time.perf_counter() - t0
    if rc != 0:
        raise PipelineError(f"tokenization failed: {_lib.last_error()}")
    docs, skipped, malformed, tokens = (int(x) for x in stats)
    return PipelineStats(docs, skipped, malformed, tokens, elapsed, tokens / elapsed if elapsed > 0 else 0.0)
