"""Tokenize pipeline throughput (SPEC.md:670 W=4 >= 2 x W=1): the C++ thread
pool at W = 1, 2, 4, 8 and, when /root/reference is importable (this container only), the
reference run_pipeline on the same corpus.   python tools/bench_pipeline.py [n_docs]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_08387_b200 import pipeline as PL  # noqa: E402
from paper_2602_08387_b200 import tokenizers as TK  # noqa: E402
from paper_2602_08387_b200.corpus_index import DocumentIndex  # noqa: E402

G = os.path.join(ROOT, "tests", "golden")
n_docs = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
rng = np.random.default_rng(0)
words = ["the", "then", "theme", "other", "in", "ing", "and", "an", "er", "on", "re", "data", "token", "café",
         "日本", "thing", "another", "rather", "tokenization", "pipeline"]
path = "/tmp/b2s_pipe_corpus.jsonl"
lines = []
for _ in range(n_docs):
    k = int(rng.integers(50, 400))
    lines.append(json.dumps({"text": " ".join(words[i] for i in rng.integers(0, len(words), size=k))}).encode())
data = b"\n".join(lines) + b"\n"
open(path, "wb").write(data)
offs = np.cumsum([0] + [len(x) + 1 for x in lines[:-1]])
index = DocumentIndex(len(data), np.stack([offs, [len(x) for x in lines]], 1).astype(np.uint64))
vocab = os.path.join(G, "tok_bpe_vocab.txt")
nv = sum(1 for _ in open(vocab, encoding="utf-8"))
tok = TK.load_tokenizer(TK.TokenizerSpec("bpe", vocab, os.path.join(G, "tok_bpe_merges.txt"), unk_token_id=nv,
                                         eod_token_id=nv + 1))
res = {"docs": n_docs, "bytes": len(data), "tokenizer": "bpe", "ours": {}}
for w in (1, 2, 4, 8):
    st = PL.run_pipeline(path, index, tok, PL.PipelineConfig("/tmp/b2s_pipe_out.cfpk", workers=w))
    res["ours"][w] = round(st.throughput, 1)
res["speedup_w4_over_w1"] = round(res["ours"][4] / res["ours"][1], 2)
res["host_cpus"] = os.cpu_count()
if os.path.isdir("/root/reference/pkg/src"):
    sys.path.insert(0, "/root/reference/pkg/src")
    from corpusforge import corpus_index as RI
    from corpusforge import pipeline as RP
    from corpusforge import tokenizers as RT

    rt = RT.load_tokenizer(RT.TokenizerSpec("bpe", vocab, os.path.join(G, "tok_bpe_merges.txt"), unk_token_id=nv,
                                            eod_token_id=nv + 1))
    sub = 2000  # bounded sample: the reference's pure-Python BPE is slow
    sp = "/tmp/b2s_pipe_small.jsonl"
    open(sp, "wb").write(b"\n".join(lines[:sub]) + b"\n")
    for w in (1, 4):
        t0 = time.perf_counter()
        st = RP.run_pipeline(sp, RI.build_index(sp), rt, RP.PipelineConfig("/tmp/b2s_ref_out.cfpk", workers=w))
        res.setdefault("reference", {})[w] = round(st.tokens / (time.perf_counter() - t0), 1)
    res["reference_sample_docs"] = sub
print(json.dumps(res))
