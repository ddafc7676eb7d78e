"""Host-side checks of the training feed (no GPU): the vocabulary guard in PackedDataLoader.bind."""

import pytest


def test_bind_rejects_token_ids_outside_the_vocabulary(tmp_path):
    from paper_2602_08387_b200.data import PackedDataLoader
    from paper_2602_08387_b200.packed import PackedWriter, open_packed

    path = str(tmp_path / "w2.cfpk")
    with PackedWriter(path, 2) as w:  # width 2 holds ids up to 65535
        w.write_document([1, 2, 3, 5000, 7])
        w.write_document([9, 10, 11, 12])
    r = open_packed(path)
    assert r.max_token() == 5000
    PackedDataLoader(r, 1, 2).bind(0, 1, "cpu", vocab_size=5001)  # ok: max id 5000 < 5001
    with pytest.raises(ValueError, match="token id 5000"):
        PackedDataLoader(r, 1, 2).bind(0, 1, "cpu", vocab_size=4096)
    PackedDataLoader(r, 1, 2).bind(0, 1, "cpu")  # no vocabulary given: no check
