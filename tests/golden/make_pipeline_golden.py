"""Generate tests/golden/pipeline_* by running the REFERENCE tokenizers and pipeline (this container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_pipeline_golden.py

Writes:
  pipeline_corpus.jsonl        tricky + random JSONL documents (one per line)
  pipeline_surrogate.jsonl     a corpus with a lone-surrogate text (the byte/bpe runs fail)
  tok_ws_vocab.txt, tok_bpe_vocab.txt, tok_bpe_merges.txt
  pipeline_golden.json         per tokenizer kind: sha256 + stats of run_pipeline output
                               (workers 1 and 3 give the same bytes), per-document
                               extract_text / encode answers for the tricky documents
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from corpusforge import corpus_index as RI  # noqa: E402
from corpusforge import pipeline as RP  # noqa: E402
from corpusforge import tokenizers as RT  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

TRICKY = [
    b'{"text":"hello world"}',
    '{"text":"héllo wörld — naïve café 日本語 \U0001F600"}'.encode("utf-8"),
    b'{"text":"tab\\tsep\\u3000ideo\\u00a0nbsp\\u2028ls\\u0085nel x\\u200by"}',
    b'{"text":"\\ud83d\\ude00 pair"}',
    b'{"text": "", "x": 1}',
    b'{"text": "   "}',
    b'{"text": 5}',
    b'{"other": "x"}',
    b'[1,2,3]',
    b'"just a string"',
    b'{"text": "a",}',
    b'{"text": "bad \\x escape"}',
    b'{"text": "ctrl char \x01 raw"}',
    b'{"text": "\xff\xfe bad utf8"}',
    b'{"text": "dup1", "text": "dup2"}',
    b'{"text": "nan", "v": NaN, "w": -Infinity, "x": 1e999, "y": Infinity}',
    b'\xef\xbb\xbf{"text":"bom"}',
    b'{"text":"x"} extra',
    b'  {"text" :  "spaces around"  }  ',
    b'{"text": "nested", "obj": {"a": [1, {"b": null}], "c": true, "d": []}, "e": {}}',
    b'{"text": "\\u0000 null char escaped"}',
    b'{"text":"n", "a": 01}',
    b'{"text":"n", "a": -}',
    b'{"text":"n", "a": 1.}',
    b'{"text":"n", "a": .5}',
    b'{"text":"n", "a": -0.5e-7, "b": 12E+3}',
    b'{"text":"line\\nbreak escaped"}',
    b'{"TEXT":"case"}',
    '{"text":"unicode key", "ключ": "значение"}'.encode("utf-8"),
    b'{"text":"the then theme other thither"}',
    b'{"text": "x\\\\u00e9 \\/ \\" \\b\\f\\r"}',
    b'{}',
    b'{"text":null}',
    b'   ',
    b'{"text":"crlf"}\r',
    b'true',
    b'{"text":"tail}',
    b'{"text":"a\\ud83dz"}',  # lone high surrogate escape followed by a letter: whitespace ok, byte/bpe fail
]
SURROGATE_IDX = len(TRICKY) - 1


def main() -> None:
    rng = np.random.default_rng(2026)
    words = ["the", "then", "theme", "other", "in", "ing", "and", "an", "er", "on", "re", "data", "token",
             "café", "日本", "\U0001F600", "x", "thing", "another", "rather"]
    docs = [d for i, d in enumerate(TRICKY) if i != SURROGATE_IDX]
    for _ in range(1500):
        n = int(rng.integers(0, 40))
        sep = [" ", "  ", "\t", "　", "  "]
        text = "".join(words[int(rng.integers(0, len(words)))] + sep[int(rng.integers(0, len(sep)))] for _ in range(n))
        docs.append(json.dumps({"id": int(rng.integers(0, 1 << 30)), "text": text},
                               ensure_ascii=bool(rng.integers(0, 2))).encode("utf-8"))
    corpus = os.path.join(HERE, "pipeline_corpus.jsonl")
    with open(corpus, "wb") as f:
        f.write(b"\n".join(docs) + b"\n")
    sur = os.path.join(HERE, "pipeline_surrogate.jsonl")
    with open(sur, "wb") as f:
        f.write(b'{"text":"ok"}\n' + TRICKY[SURROGATE_IDX] + b"\n")

    ws_vocab = ["the", "then", "other", "data", "token", "café", "日本", "\U0001F600", "hello", "world"]
    with open(os.path.join(HERE, "tok_ws_vocab.txt"), "w", encoding="utf-8", newline="\n") as f:
        f.write("\n".join(ws_vocab) + "\n")
    base = [chr(c) for c in range(33, 127)]
    merges = [("t", "h"), ("th", "e"), ("i", "n"), ("in", "g"), ("a", "n"), ("an", "d"), ("e", "r"), ("o", "n"),
              ("r", "e"), ("the", "n"), ("the", "m"), ("o", "th"), ("oth", "er"), ("d", "a"), ("da", "t"),
              ("dat", "a"), ("t", "o"), ("to", "k"), ("e", "n")]
    bpe_vocab = base + [a + b for a, b in merges] + ["caf", "é"]
    with open(os.path.join(HERE, "tok_bpe_vocab.txt"), "w", encoding="utf-8", newline="\n") as f:
        f.write("\n".join(bpe_vocab) + "\n")
    with open(os.path.join(HERE, "tok_bpe_merges.txt"), "w", encoding="utf-8", newline="\n") as f:
        f.write("\n".join(f"{a} {b}" for a, b in merges) + "\n")

    specs = {
        "byte": RT.TokenizerSpec("byte", eod_token_id=256),
        "whitespace": RT.TokenizerSpec("whitespace", os.path.join(HERE, "tok_ws_vocab.txt"), unk_token_id=10,
                                       eod_token_id=11),
        "bpe": RT.TokenizerSpec("bpe", os.path.join(HERE, "tok_bpe_vocab.txt"),
                                os.path.join(HERE, "tok_bpe_merges.txt"), unk_token_id=len(bpe_vocab),
                                eod_token_id=len(bpe_vocab) + 1),
    }
    g = {"specs": {k: {"vocab": os.path.basename(s.vocab_path) if s.vocab_path else None,
                       "merges": os.path.basename(s.merges_path) if s.merges_path else None,
                       "unk": s.unk_token_id, "eod": s.eod_token_id} for k, s in specs.items()},
         "runs": {}, "tricky": {}, "surrogate_run_fails": {}}
    index = RI.build_index(corpus)
    for kind, spec in specs.items():
        tok = RT.load_tokenizer(spec)
        shas = set()
        for workers in (1, 3):
            out = os.path.join(HERE, f"_pipe_{kind}_{workers}.cfpk")
            st = RP.run_pipeline(corpus, index, tok, RP.PipelineConfig(out, workers=workers, batch_size=37))
            shas.add(hashlib.sha256(open(out, "rb").read()).hexdigest())
            os.remove(out)
        assert len(shas) == 1
        g["runs"][kind] = {"sha256": shas.pop(), "documents": st.documents, "skipped": st.skipped,
                           "malformed": st.malformed, "tokens": st.tokens}
        per = []
        for raw in TRICKY:
            t = RP.extract_text(raw)
            if isinstance(t, RP.Skip):
                per.append({"skip": t.value})
                continue
            try:
                per.append({"ids": tok.encode(t)})
            except UnicodeEncodeError:
                per.append({"error": "UnicodeEncodeError"})
        g["tricky"][kind] = per
        sidx = RI.build_index(sur)
        try:
            RP.run_pipeline(sur, sidx, tok, RP.PipelineConfig(os.path.join(HERE, "_s.cfpk"), workers=2))
            g["surrogate_run_fails"][kind] = False
        except RP.PipelineError:
            g["surrogate_run_fails"][kind] = True
        if os.path.exists(os.path.join(HERE, "_s.cfpk")):
            os.remove(os.path.join(HERE, "_s.cfpk"))
    g["tricky_raw_hex"] = [r.hex() for r in TRICKY]
    with open(os.path.join(HERE, "pipeline_golden.json"), "w") as f:
        json.dump(g, f, indent=1)
    print(json.dumps(g["runs"]), g["surrogate_run_fails"])


if __name__ == "__main__":
    main()
