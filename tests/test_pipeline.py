"""Tokenization pipeline: the C++ thread-pool producer vs reference goldens.

Goldens (tests/golden/pipeline_golden.json) were produced by running the reference
run_pipeline / tokenizers (tests/golden/make_pipeline_golden.py). Host only (no GPU).
"""

import hashlib
import json
import os

import pytest

from conftest import GOLDEN
from paper_2602_08387_b200 import corpus_index as CI
from paper_2602_08387_b200 import pipeline as PL
from paper_2602_08387_b200 import tokenizers as TK


@pytest.fixture(scope="module")
def pg():
    with open(os.path.join(GOLDEN, "pipeline_golden.json")) as f:
        return json.load(f)


def _tok(pg, kind):
    s = pg["specs"][kind]
    return TK.load_tokenizer(TK.TokenizerSpec(kind, os.path.join(GOLDEN, s["vocab"]) if s["vocab"] else None,
                                              os.path.join(GOLDEN, s["merges"]) if s["merges"] else None,
                                              eod_token_id=s["eod"], unk_token_id=s["unk"]))


def _index(path):
    """Host restatement of build_index for these host-only tests (the GPU scan is tested in
    test_corpus_index.py); spans of the non-empty lines."""
    data = open(path, "rb").read()
    spans, start = [], 0
    for i, b in enumerate(data):
        if b == 10:
            if i > start:
                spans.append((start, i - start))
            start = i + 1
    if start < len(data):
        spans.append((start, len(data) - start))
    import numpy as np

    return CI.DocumentIndex(len(data), np.asarray(spans, dtype=np.uint64).reshape(-1, 2))


@pytest.mark.parametrize("kind", ["byte", "whitespace", "bpe"])
def test_tricky_documents_match_reference(pg, kind):
    """extract_text + encode per document: Python json semantics (NaN, BOM, duplicate keys,
    strict strings, escapes, surrogate pairs), Unicode whitespace splitting, BPE merge order."""
    tok = _tok(pg, kind)
    for raw_hex, exp in zip(pg["tricky_raw_hex"], pg["tricky"][kind]):
        raw = bytes.fromhex(raw_hex)
        t = PL.extract_text(raw)
        if "skip" in exp:
            assert isinstance(t, PL.Skip) and t.value == exp["skip"], raw
            continue
        assert isinstance(t, str), raw
        if "error" in exp:
            with pytest.raises(UnicodeEncodeError):
                tok.encode(t)
        else:
            assert tok.encode(t) == exp["ids"], raw


@pytest.mark.parametrize("kind", ["byte", "whitespace", "bpe"])
@pytest.mark.parametrize("workers", [1, 4, 16])
def test_pipeline_bytes_match_reference(pg, tmp_path, kind, workers):
    """The C++ producer writes the reference's bytes for every worker count."""
    corpus = os.path.join(GOLDEN, "pipeline_corpus.jsonl")
    out = tmp_path / "out.cfpk"
    st = PL.run_pipeline(corpus, _index(corpus), _tok(pg, kind), PL.PipelineConfig(str(out), workers=workers,
                                                                                    batch_size=37))
    g = pg["runs"][kind]
    assert hashlib.sha256(out.read_bytes()).hexdigest() == g["sha256"]
    assert (st.documents, st.skipped, st.malformed, st.tokens) == (g["documents"], g["skipped"], g["malformed"],
                                                                   g["tokens"])


@pytest.mark.parametrize("kind", ["byte", "whitespace", "bpe"])
def test_lone_surrogate_fails_like_reference(pg, tmp_path, kind):
    corpus = os.path.join(GOLDEN, "pipeline_surrogate.jsonl")
    cfg = PL.PipelineConfig(str(tmp_path / "s.cfpk"), workers=2)
    if pg["surrogate_run_fails"][kind]:
        with pytest.raises(PL.PipelineError):
            PL.run_pipeline(corpus, _index(corpus), _tok(pg, kind), cfg)
    else:
        PL.run_pipeline(corpus, _index(corpus), _tok(pg, kind), cfg)


def test_pipeline_errors(pg, tmp_path):
    corpus = os.path.join(GOLDEN, "pipeline_corpus.jsonl")
    ix = _index(corpus)
    stale = CI.DocumentIndex(ix.source_size + 1, ix.spans)
    with pytest.raises(PL.StaleIndexError):
        PL.run_pipeline(corpus, stale, _tok(pg, "byte"), PL.PipelineConfig(str(tmp_path / "a.cfpk")))
    with pytest.raises(ValueError):
        PL.run_pipeline(corpus, ix, TK.ByteTokenizer(), PL.PipelineConfig(str(tmp_path / "b.cfpk")))
    for bad in (dict(workers=0), dict(batch_size=0), dict(queue_capacity=0)):
        with pytest.raises(ValueError):
            PL.PipelineConfig(str(tmp_path / "c.cfpk"), **bad)
    with pytest.raises(TK.OutOfVocabError):
        TK.ByteTokenizer().decode([256])
    v = tmp_path / "v.txt"
    v.write_text("a\na\n")
    with pytest.raises(TK.VocabFormatError):
        TK.load_tokenizer(TK.TokenizerSpec("whitespace", str(v), unk_token_id=0))
    v.write_text("a\nb\n")
    m = tmp_path / "m.txt"
    m.write_text("a b\n")
    with pytest.raises(TK.MergeFormatError):  # "ab" absent from the vocabulary
        TK.load_tokenizer(TK.TokenizerSpec("bpe", str(v), str(m), unk_token_id=2))
