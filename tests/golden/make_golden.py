"""Generate tests/golden/* by running the REFERENCE implementation (this container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes:
  packed_golden.json   splitmix64 / make_permutation / chunk / token_width /
                       sample_count answers computed by corpusforge.packed_data
  ref_w{1,2,4}.cfpk    small packed files written by the reference PackedWriter
  ref_w{1,2,4}.npz     get_sample(s, L) for a grid of (s, L), from the reference reader
  (json) materialize   sha256 of materialize_chunk outputs for seeded permutation chunks
  (json) perm_sidecar  sha256 of write_permutation .perm files
  idx_*.jsonl          raw fixtures; (json) corpus_index = build_index spans + .didx sha256
The GPU box never runs this script (the reference does not travel).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from corpusforge import packed_data as ref  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    g: dict = {}
    sm = {}
    for seed in (0, 42, 1234, (1 << 64) - 1):
        it = ref.splitmix64(seed)
        sm[str(seed)] = [hex(next(it)) for _ in range(8)]
    g["splitmix64"] = sm

    perms = []
    for n, seed in [(0, 0), (1, 0), (2, 7), (4, 42), (10, 0), (16, 1234), (5, (1 << 64) - 1),
                    (5, -1), (7, -1), (33, 99), (257, 3), (1000, 2026)]:
        perms.append({"n": n, "seed": seed, "order": [int(x) for x in ref.make_permutation(n, seed).order]})
    g["permutations"] = perms
    big = ref.make_permutation(1_000_000, 0).order.astype("<u8").tobytes()
    g["perm_1m_seed0_sha256"] = hashlib.sha256(big).hexdigest()

    g["chunks"] = []
    for n, k in [(10, 3), (3, 3), (10, 1), (7, 7), (0, 1), (100, 8), (5, 4)]:
        spec = ref.chunk(ref.make_permutation(n, 0), k)
        g["chunks"].append({"n": n, "k": k, "sizes": [len(a) for a in spec.assignments],
                            "flat": [int(x) for a in spec.assignments for x in a]})
    g["chunk_invalid"] = [[10, 0], [10, 11], [0, 2]]

    g["token_width"] = {str(v): ref.token_width_for_vocab(v)
                        for v in (1, 255, 256, 257, 4096, 50257, 65536, 65537, 128256, 1 << 32)}

    # small files written by the reference writer; samples read by the reference reader
    rng = np.random.default_rng(7)
    files = {}
    for w, vocab in ((1, 256), (2, 50257), (4, 128256)):
        path = os.path.join(HERE, f"ref_w{w}.cfpk")
        with ref.PackedWriter(path, w) as wr:
            for _ in range(23):
                wr.write_document(rng.integers(0, vocab, size=int(rng.integers(1, 300))))
            wr.write_document([])  # zero-length document is legal in the format
            wr.write_document([vocab - 1])
        rd = ref.open_packed(path)
        samples = {}
        for L in (1, 2, 3, 7, 64, 255, 1000):
            n = rd.sample_count(L)
            for s in sorted({0, 1, n // 2, n - 1} & set(range(n))):
                samples[f"L{L}_s{s}"] = np.array(rd.get_sample(s, L), dtype=np.int64)
        np.savez(os.path.join(HERE, f"ref_w{w}.npz"), **samples)
        files[str(w)] = {"token_count": rd.token_count, "doc_count": rd.doc_count,
                         "sample_count": {str(L): rd.sample_count(L) for L in (1, 2, 3, 7, 64, 255, 1000, 10**9)},
                         "spans": [[int(a), int(b)] for a, b in rd.spans]}
        rd.close()
    g["files"] = files

    # the SPEC's 9-token example
    path = os.path.join(HERE, "ref_nine.cfpk")
    with ref.PackedWriter(path, 2) as wr:
        wr.write_document(list(range(100, 109)))
    rd = ref.open_packed(path)
    g["nine"] = {"sample_count_4": rd.sample_count(4), "s0": rd.get_sample(0, 4).tolist(),
                 "s1": rd.get_sample(1, 4).tolist(), "file_len": os.path.getsize(path)}
    rd.close()

    # materialize_chunk (packed_data.py:336-344) of each chunk of a seeded document
    # permutation, and the .perm sidecar bytes (write_permutation, :285-290)
    mat = {}
    for w in (1, 2, 4):
        rd = ref.open_packed(os.path.join(HERE, f"ref_w{w}.cfpk"))
        for seed, k in ((0, 1), (3, 3), (11, 4)):
            perm = ref.make_permutation(rd.doc_count, seed) if seed else ref.Permutation(
                seed=0, order=np.arange(rd.doc_count, dtype="<u8"))
            for c, docs in enumerate(ref.chunk(perm, k).assignments):
                out = os.path.join(HERE, f"_mat_tmp_{w}.cfpk")
                ref.materialize_chunk(rd, docs, out)
                mat[f"w{w}_seed{seed}_k{k}_c{c}"] = {"docs": [int(d) for d in docs],
                                                     "sha256": hashlib.sha256(open(out, "rb").read()).hexdigest()}
                os.remove(out)
        rd.close()
    g["materialize"] = mat
    side = {}
    for n, seed in ((0, 0), (10, 0), (1000, 2026), (5, (1 << 64) - 1)):
        out = os.path.join(HERE, "_perm_tmp.perm")
        ref.write_permutation(ref.make_permutation(n, seed), out)
        side[f"{n}_{seed}"] = hashlib.sha256(open(out, "rb").read()).hexdigest()
        os.remove(out)
    g["perm_sidecar_sha256"] = side

    # corpus_index.build_index (corpus_index.py:68-107) on small raw fixtures
    from corpusforge import corpus_index as cidx

    fixtures = {
        "idx_mixed.jsonl": b'{"text":"a"}\n\n{"text":"bc"}\r\n\n\n{"x":1}\n{"text":"no newline at end"}',
        "idx_trailing.jsonl": b'{"text":"one"}\n{"text":"two"}\n',
        "idx_only_newlines.jsonl": b"\n\n\n",
        "idx_empty.jsonl": b"",
    }
    rng = np.random.default_rng(11)
    lines = []
    for _ in range(3000):
        k = int(rng.integers(0, 200))
        lines.append(bytes(rng.integers(32, 127, size=k, dtype=np.uint8)) + (b"\r" if rng.random() < 0.1 else b""))
    fixtures["idx_random.jsonl"] = b"\n".join(lines)
    idx = {}
    for name, data in fixtures.items():
        path = os.path.join(HERE, name)
        with open(path, "wb") as f:
            f.write(data)
        ix = cidx.build_index(path, buffer_size=7)
        out = os.path.join(HERE, "_idx_tmp.didx")
        cidx.write_index(ix, out)
        idx[name] = {"source_size": ix.source_size, "spans": [[int(a), int(b)] for a, b in ix.spans],
                     "didx_sha256": hashlib.sha256(open(out, "rb").read()).hexdigest()}
        os.remove(out)
    g["corpus_index"] = idx

    with open(os.path.join(HERE, "packed_golden.json"), "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", os.path.join(HERE, "packed_golden.json"))


if __name__ == "__main__":
    main()
