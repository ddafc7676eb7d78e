"""Packed token stream: oracle pinned to reference goldens, host C-ABI, GPU gather parity."""

import hashlib
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import packed_oracle as orc
from paper_2602_08387_b200 import packed as P

# ---------------------------------------------------------------- oracle vs reference goldens


def test_oracle_splitmix_matches_reference(golden):
    for seed, outs in golden["splitmix64"].items():
        assert [hex(x) for x in orc.splitmix64_first(int(seed), len(outs))] == outs


def test_oracle_permutation_matches_reference(golden):
    for case in golden["permutations"]:
        assert orc.permutation(case["n"], case["seed"]).tolist() == case["order"]


def test_oracle_c_permutation_sha_1m(golden):
    import oracle

    lib = oracle.clib()
    out = np.empty(1_000_000, dtype="<u8")
    lib.oracle_permutation(1_000_000, 0, out.ctypes.data)
    assert hashlib.sha256(out.tobytes()).hexdigest() == golden["perm_1m_seed0_sha256"]


def test_oracle_samples_match_reference_files(golden):
    for w in ("1", "2", "4"):
        path = os.path.join(GOLDEN, f"ref_w{w}.cfpk")
        buf = open(path, "rb").read()
        width, count, ndocs, off = orc.parse_header(buf, len(buf))
        payload = np.frombuffer(buf, {1: "<u1", 2: "<u2", 4: "<u4"}[width], count, 40)
        exp = np.load(os.path.join(GOLDEN, f"ref_w{w}.npz"))
        for key in exp.files:
            L, s = (int(x[1:]) for x in key.split("_"))
            assert np.array_equal(orc.sample_window(payload, s, L).astype(np.int64), exp[key])
        for L, n in golden["files"][w]["sample_count"].items():
            assert orc.sample_count(count, int(L)) == n


def test_oracle_chunks(golden):
    for c in golden["chunks"]:
        assert orc.chunk_sizes(c["n"], c["k"]) == c["sizes"]


# ---------------------------------------------------------------- product host side vs goldens


def test_token_width(golden):
    for v, w in golden["token_width"].items():
        assert P.token_width_for_vocab(int(v)) == w
    for bad in (0, (1 << 32) + 1):
        with pytest.raises(ValueError):
            P.token_width_for_vocab(bad)


def test_splitmix_and_permutation(golden):
    for seed, outs in golden["splitmix64"].items():
        assert [hex(int(x)) for x in P.splitmix64(int(seed), len(outs))] == outs
    for case in golden["permutations"]:
        perm = P.make_permutation(case["n"], case["seed"])
        assert perm.order.dtype == np.dtype("<u8")
        assert perm.order.tolist() == case["order"]
    big = P.make_permutation(1_000_000, 0).order
    assert hashlib.sha256(big.astype("<u8").tobytes()).hexdigest() == golden["perm_1m_seed0_sha256"]
    with pytest.raises(ValueError):
        P.make_permutation(-1, 0)


def test_permutation_properties():
    rng = np.random.default_rng(0)
    for _ in range(200):
        n, seed = int(rng.integers(0, 3000)), int(rng.integers(0, 1 << 63))
        a = P.make_permutation(n, seed).order
        assert np.array_equal(np.sort(a), np.arange(n, dtype=np.uint64))
        assert np.array_equal(a, P.make_permutation(n, seed).order)
    assert not np.array_equal(P.make_permutation(64, 1).order, P.make_permutation(64, 2).order)


def test_chunk(golden):
    for c in golden["chunks"]:
        spec = P.chunk(P.make_permutation(c["n"], 0), c["k"])
        assert [len(a) for a in spec.assignments] == c["sizes"]
        assert [int(x) for a in spec.assignments for x in a] == c["flat"]
    for n, k in golden["chunk_invalid"]:
        with pytest.raises(P.InvalidKError):
            P.chunk(P.make_permutation(n, 0), k)


def test_reader_on_reference_files(golden):
    for w in ("1", "2", "4"):
        r = P.open_packed(os.path.join(GOLDEN, f"ref_w{w}.cfpk"))
        g = golden["files"][w]
        assert (r.token_count, r.doc_count) == (g["token_count"], g["doc_count"])
        assert r.spans.tolist() == g["spans"]
        exp = np.load(os.path.join(GOLDEN, f"ref_w{w}.npz"))
        for key in exp.files:
            L, s = (int(x[1:]) for x in key.split("_"))
            got = r.get_sample(s, L)
            assert np.array_equal(got.astype(np.int64), exp[key])
            assert got.dtype == np.dtype({"1": "<u1", "2": "<u2", "4": "<u4"}[w])
            assert not got.flags.writeable
        for L, n in g["sample_count"].items():
            assert r.sample_count(int(L)) == n
        with pytest.raises(P.OutOfRangeError):
            r.get_sample(r.sample_count(7), 7)
        with pytest.raises(P.OutOfRangeError):
            r.get_document_tokens(r.doc_count)
        with pytest.raises(ValueError):
            r.sample_count(0)


def test_nine_token_example(golden):
    r = P.open_packed(os.path.join(GOLDEN, "ref_nine.cfpk"))
    nine = golden["nine"]
    assert r.sample_count(4) == nine["sample_count_4"]
    assert r.get_sample(0, 4).tolist() == nine["s0"]
    assert r.get_sample(1, 4).tolist() == nine["s1"]
    with pytest.raises(IndexError):
        r.get_sample(2, 4)


def test_writer_matches_reference_bytes(tmp_path):
    # our writer must produce byte-identical files to the reference writer's output
    src = P.open_packed(os.path.join(GOLDEN, "ref_w2.cfpk"))
    out = tmp_path / "copy.cfpk"
    P.materialize_chunk(src, range(src.doc_count), out)
    assert out.read_bytes() == open(os.path.join(GOLDEN, "ref_w2.cfpk"), "rb").read()


def test_format_errors(tmp_path):
    p = tmp_path / "short.cfpk"
    p.write_bytes(b"CFPKD001")
    with pytest.raises(P.FormatError):
        P.open_packed(p)
    good = open(os.path.join(GOLDEN, "ref_nine.cfpk"), "rb").read()
    for mutate in (lambda b: b"XFPKD001" + b[8:], lambda b: b + b"\x00", lambda b: b[:-1],
                   lambda b: b[:8] + (2).to_bytes(4, "little") + b[12:],
                   lambda b: b[:12] + (3).to_bytes(4, "little") + b[16:]):
        p = tmp_path / "bad.cfpk"
        p.write_bytes(mutate(good))
        with pytest.raises(P.FormatError):
            P.open_packed(p)


def test_perm_sidecar_roundtrip(tmp_path):
    rng = np.random.default_rng(1)
    for i in range(100):
        perm = P.make_permutation(int(rng.integers(0, 500)), int(rng.integers(0, 1 << 63)))
        path = tmp_path / f"p{i}.perm"
        P.write_permutation(perm, path)
        assert P.load_permutation(path) == perm
    with pytest.raises(ValueError):
        P.write_permutation(P.make_permutation(3, -1), tmp_path / "neg.perm")


# ---------------------------------------------------------------- GPU gather (K1) parity


def _oracle_batch(path, ids, L):
    buf = open(path, "rb").read()
    width, count, _, _ = orc.parse_header(buf, len(buf))
    payload = np.frombuffer(buf, {1: "<u1", 2: "<u2", 4: "<u4"}[width], count, 40)
    return orc.batch_windows(payload, ids, L)


@pytest.mark.gpu
def test_gather_matches_oracle_on_reference_files(cuda):
    for w in ("1", "2", "4"):
        path = os.path.join(GOLDEN, f"ref_w{w}.cfpk")
        r = P.open_packed(path)
        ds = P.DevicePackedStream(r)
        for L in (1, 2, 3, 7, 64, 255, 1000):
            n = r.sample_count(L)
            if n == 0:
                continue
            rng = np.random.default_rng(L)
            for B in (1, 2, 5, 8):
                ids = rng.integers(0, n, size=B).astype(np.uint64)
                ei, et = _oracle_batch(path, ids, L)
                gi, gt = ds.gather(ids, L)
                assert gi.dtype == gt.dtype == __import__("torch").int64
                assert np.array_equal(gi.cpu().numpy(), ei)
                assert np.array_equal(gt.cpu().numpy(), et)


@pytest.mark.gpu
def test_gather_out_of_range_and_empty(cuda):
    import torch

    r = P.open_packed(os.path.join(GOLDEN, "ref_nine.cfpk"))
    ds = P.DevicePackedStream(r)
    with pytest.raises(P.OutOfRangeError):
        ds.gather(np.array([0, 2], dtype=np.uint64), 4)
    # unchecked path: the kernel flags the bad id on the device instead
    ds.gather(np.array([2], dtype=np.uint64), 4, check=False)
    torch.cuda.synchronize()
    assert int(ds.status.item()) == 1
    gi, gt = ds.gather(np.zeros(0, dtype=np.uint64), 4)
    assert gi.shape == (0, 4)


@pytest.mark.gpu
def test_gather_full_size_tiling_property(cuda, tmp_path):
    """At bench sizes: samples s=0..n-1 tile the payload with a one-token overlap."""
    import torch

    rng = np.random.default_rng(3)
    V, L = 50257, 2048
    toks = rng.integers(0, V, size=(1 << 22) + 1, dtype=np.int64)
    path = tmp_path / "big.cfpk"
    with P.PackedWriter(path, 2) as w:
        w.write_stream(toks, 1024)
    r = P.open_packed(path)
    ds = P.DevicePackedStream(r)
    n = r.sample_count(L)
    ids = np.arange(n, dtype=np.uint64)
    gi, gt = ds.gather(ids, L)
    flat_in = gi.reshape(-1)
    expect = torch.from_numpy(toks[: n * L + 1]).cuda()
    assert torch.equal(flat_in, expect[: n * L])
    assert torch.equal(gt.reshape(-1), expect[1 : n * L + 1])
    perm = P.make_permutation(n, 11).order
    pi, pt = ds.gather(perm, L)
    assert torch.equal(pi, gi[torch.from_numpy(perm.astype(np.int64)).cuda()])


# ---------------------------------------------------------------------------- materialize / sidecar


def _sha(b: bytes) -> str:
    import hashlib

    return hashlib.sha256(b).hexdigest()


def test_materialize_oracle_pinned_to_reference(golden):
    """The oracle's materialize_chunk bytes equal the reference's (sha256 goldens)."""
    for key, g in golden["materialize"].items():
        w = key.split("_")[0][1:]
        buf = open(os.path.join(GOLDEN, f"ref_w{w}.cfpk"), "rb").read()
        assert _sha(orc.materialize_bytes(buf, g["docs"])) == g["sha256"], key


def test_materialize_host_path_matches_reference(golden, tmp_path):
    for key, g in golden["materialize"].items():
        w = key.split("_")[0][1:]
        r = P.open_packed(os.path.join(GOLDEN, f"ref_w{w}.cfpk"))
        out = tmp_path / f"{key}.cfpk"
        P.materialize_chunk(r, np.asarray(g["docs"], dtype=np.uint64), out)
        assert _sha(out.read_bytes()) == g["sha256"], key


def test_perm_sidecar_bytes_match_reference(golden, tmp_path):
    for key, sha in golden["perm_sidecar_sha256"].items():
        n, seed = (int(x) for x in key.split("_"))
        path = tmp_path / f"{key}.perm"
        P.write_permutation(P.make_permutation(n, seed), path)
        assert _sha(path.read_bytes()) == sha, key
        assert P.load_permutation(path) == P.make_permutation(n, seed)


@pytest.mark.gpu
def test_materialize_gpu_matches_reference(cuda, golden, tmp_path):
    """b2s_gather_documents: the GPU materialize_chunk writes the reference's bytes."""
    for key, g in golden["materialize"].items():
        w = key.split("_")[0][1:]
        r = P.open_packed(os.path.join(GOLDEN, f"ref_w{w}.cfpk"))
        out = tmp_path / f"{key}.cfpk"
        P.materialize_chunk_gpu(r, np.asarray(g["docs"], dtype=np.uint64), out)
        assert _sha(out.read_bytes()) == g["sha256"], key
    r = P.open_packed(os.path.join(GOLDEN, "ref_w2.cfpk"))
    with pytest.raises(P.OutOfRangeError):
        P.materialize_chunk_gpu(r, [0, r.doc_count], tmp_path / "bad.cfpk")
    P.materialize_chunk_gpu(r, [], tmp_path / "empty.cfpk")  # zero documents: valid empty file
    e = P.open_packed(tmp_path / "empty.cfpk")
    assert e.doc_count == 0 and e.token_count == 0


@pytest.mark.gpu
def test_materialize_gpu_full_size(cuda, tmp_path):
    """2^24 tokens, ragged documents (incl. empty ones), a seeded global shuffle split in 8
    chunks: every chunk equals the oracle's bytes; re-opened chunks concatenate to the
    permuted corpus (span contiguity); identity permutation, k=1 -> byte copy."""
    rng = np.random.default_rng(5)
    path = tmp_path / "corpus.cfpk"
    lens = rng.integers(0, 4000, size=8192)
    lens[::97] = 0
    with P.PackedWriter(path, 4) as w:
        for n in lens:
            w.write_document(rng.integers(0, 128256, size=int(n)))
    r = P.open_packed(path)
    ds = P.DevicePackedStream(r)
    buf = path.read_bytes()
    perm = P.make_permutation(r.doc_count, 2026)
    for c, docs in enumerate(P.chunk(perm, 8).assignments):
        out = tmp_path / f"c{c}.cfpk"
        P.materialize_chunk_gpu(r, docs, out, stream=ds)
        assert out.read_bytes() == orc.materialize_bytes(buf, docs), c
        cr = P.open_packed(out)
        sp = np.asarray(cr.spans)
        assert np.array_equal(sp[1:, 0], sp[:-1, 0] + sp[:-1, 1]) and int(sp[:, 1].sum()) == cr.token_count
    ident = tmp_path / "ident.cfpk"
    P.materialize_chunk_gpu(r, np.arange(r.doc_count), ident, stream=ds)
    assert ident.read_bytes() == buf
