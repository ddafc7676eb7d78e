"""Corpus index: GPU newline scan vs the reference build_index goldens."""

import hashlib
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import index_oracle as orc
from paper_2602_08387_b200 import corpus_index as CI


def test_oracle_pinned_to_reference(golden):
    for name, g in golden["corpus_index"].items():
        data = open(os.path.join(GOLDEN, name), "rb").read()
        exp = np.asarray(g["spans"], dtype=np.uint64).reshape(-1, 2)
        assert np.array_equal(orc.spans(data), exp), name
        assert np.array_equal(orc.spans_fast(data), exp), name


def test_sidecar_format_matches_reference(golden, tmp_path):
    for name, g in golden["corpus_index"].items():
        ix = CI.DocumentIndex(g["source_size"], np.asarray(g["spans"], dtype="<u8").reshape(-1, 2))
        p = tmp_path / (name + ".didx")
        CI.write_index(ix, p)
        assert hashlib.sha256(p.read_bytes()).hexdigest() == g["didx_sha256"], name
        assert CI.load_index(p) == ix
    bad = tmp_path / "bad.didx"
    bad.write_bytes(b"XXXXXXXX" + bytes(20))
    with pytest.raises(CI.FormatError):
        CI.load_index(bad)
    bad.write_bytes(b"CFIDX001")
    with pytest.raises(CI.FormatError):
        CI.load_index(bad)
    with pytest.raises(ValueError):
        CI.build_index(bad, buffer_size=0)


@pytest.mark.gpu
def test_build_index_gpu_matches_reference(cuda, golden, tmp_path):
    for name, g in golden["corpus_index"].items():
        path = os.path.join(GOLDEN, name)
        for bs in (1, 7, 1 << 20):
            ix = CI.build_index(path, buffer_size=bs)
            assert ix.source_size == g["source_size"]
            assert np.array_equal(ix.spans, np.asarray(g["spans"], dtype=np.uint64).reshape(-1, 2)), (name, bs)
        p = tmp_path / "x.didx"
        CI.write_index(ix, p)
        assert hashlib.sha256(p.read_bytes()).hexdigest() == g["didx_sha256"], name
        assert CI.verify_index(ix, path)
    ix = CI.build_index(os.path.join(GOLDEN, "idx_mixed.jsonl"))
    assert CI.read_document(os.path.join(GOLDEN, "idx_mixed.jsonl"), ix, 1) == b'{"text":"bc"}\r'
    with pytest.raises(CI.OutOfRangeError):
        ix.span(ix.doc_count)


@pytest.mark.gpu
def test_build_index_gpu_full_size(cuda, tmp_path, monkeypatch):
    """64 MiB of ragged lines (empty lines, CR bytes, no trailing newline) vs the oracle; the
    answer is independent of how the file is cut into GPU scan pieces."""
    rng = np.random.default_rng(3)
    n = 64 << 20
    data = rng.integers(32, 127, size=n, dtype=np.uint8)
    nl = rng.integers(0, n, size=n // 300)
    data[nl] = 10
    data[rng.integers(0, n, size=1000)] = 13
    data[-1] = ord("x")
    path = tmp_path / "big.jsonl"
    data.tofile(path)
    exp = orc.spans_fast(data.tobytes())
    ix = CI.build_index(path)
    assert np.array_equal(ix.spans, exp) and ix.source_size == n
    monkeypatch.setattr(CI, "_PIECE", (1 << 20) + 16 * 7)  # pieces not aligned to anything in the file
    assert np.array_equal(CI.build_index(path).spans, exp)
