"""CLI data commands (reference SPEC cli: index / tokenize / shuffle / chunk / sample)."""

import hashlib
import json
import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2602_08387_b200 import cli
from paper_2602_08387_b200 import corpus_index as CI
from paper_2602_08387_b200 import packed as P


def _tok_yaml(tmp_path, raw):
    y = tmp_path / "tok.yaml"
    y.write_text(f"""tok:
  interface: tokenizer
  variant: bpe
  config: {{vocab_path: {GOLDEN}/tok_bpe_vocab.txt, merges_path: {GOLDEN}/tok_bpe_merges.txt, unk_token_id: 115, eod_token_id: 116}}
pipeline:
  interface: pipeline
  variant: tokenize
  config: {{raw_path: {raw}, out_path: {tmp_path}/out.cfpk, tokenizer: !ref tok, workers: 3, batch_size: 37}}
""")
    return y


def test_cli_tokenize_sample_shuffle(tmp_path, capsys):
    from test_pipeline import _index

    raw = tmp_path / "corpus.jsonl"
    shutil.copy(os.path.join(GOLDEN, "pipeline_corpus.jsonl"), raw)
    CI.write_index(_index(str(raw)), CI.index_sidecar_path(raw))  # host index (the GPU scan: test below)
    assert cli.main(["tokenize", "-c", str(_tok_yaml(tmp_path, raw)), "--root", "pipeline", "--json"]) == 0
    st = json.loads(capsys.readouterr().out)
    g = json.load(open(os.path.join(GOLDEN, "pipeline_golden.json")))["runs"]["bpe"]
    assert st["tokens"] == g["tokens"] and st["documents"] == g["documents"]
    out = tmp_path / "out.cfpk"
    assert hashlib.sha256(out.read_bytes()).hexdigest() == g["sha256"]
    assert cli.main(["sample", str(out), "0", "8", "--json"]) == 0
    ids = json.loads(capsys.readouterr().out)["ids"]
    assert ids == [int(x) for x in P.open_packed(out).get_sample(0, 8)] and len(ids) == 9
    assert cli.main(["shuffle", str(out), "--seed", "3"]) == 0
    capsys.readouterr()
    assert P.load_permutation(str(out) + ".perm") == P.make_permutation(P.open_packed(out).doc_count, 3)
    assert cli.main(["sample", str(out), "99999999", "8"]) == 1  # OutOfRangeError -> runtime failure


@pytest.mark.gpu
def test_cli_index_and_chunk_gpu(cuda, tmp_path, capsys, golden):
    raw = tmp_path / "idx.jsonl"
    shutil.copy(os.path.join(GOLDEN, "idx_random.jsonl"), raw)
    assert cli.main(["index", str(raw)]) == 0
    capsys.readouterr()
    ix = CI.load_index(CI.index_sidecar_path(raw))
    exp = golden["corpus_index"]["idx_random.jsonl"]
    assert np.array_equal(ix.spans, np.asarray(exp["spans"], dtype=np.uint64))
    src = os.path.join(GOLDEN, "ref_w2.cfpk")
    pk = tmp_path / "p.cfpk"
    shutil.copy(src, pk)
    assert cli.main(["shuffle", str(pk), "--seed", "3"]) == 0
    assert cli.main(["chunk", str(pk), str(pk) + ".perm", "3", str(tmp_path / "chunks")]) == 0
    capsys.readouterr()
    for c in range(3):
        key = f"w2_seed3_k3_c{c}"
        data = (tmp_path / "chunks" / f"chunk_{c:05d}.cfpk").read_bytes()
        assert hashlib.sha256(data).hexdigest() == golden["materialize"][key]["sha256"], key
