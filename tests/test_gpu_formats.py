"""Device-formatted writers against the reference's own output
bytes (tests/golden/formats.json, made from /root/reference by make_golden.py)."""

import base64
import json

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

G = json.loads((GOLDEN / "formats.json").read_text())


class _Vocab:
    def __init__(self, lex):
        self.lex = lex

    def lexical(self, t):
        return self.lex[t]


@pytest.mark.parametrize("name", ["f64", "f32"])
@pytest.mark.parametrize("kind", ["text", "tsv"])
def test_embedding_writers_byte_exact(tmp_path, name, kind):
    import torch

    from paper_2508_01073_b200 import formats

    m = np.array(G[f"{name}_matrix"], dtype=np.float64)
    vocab = _Vocab(G[f"{name}_lexicals"])
    fn = formats.save_embeddings_text if kind == "text" else formats.save_embeddings_tsv
    want = base64.b64decode(G[f"{name}_{kind}"])
    fn(m, vocab, tmp_path / "a")
    assert (tmp_path / "a").read_bytes() == want
    if name == "f32":  # the fp32 parameter store, formatted from the device tensor
        fn(torch.from_numpy(m.astype(np.float32)).cuda(), vocab, tmp_path / "b")
        assert (tmp_path / "b").read_bytes() == want


def test_fmt_g8_random_values_match_python(tmp_path):
    """200k random doubles over 1e-30..1e15 (both signs): every cell equals format(x, '.8g')."""
    from paper_2508_01073_b200 import formats

    rng = np.random.default_rng(5)
    sign = np.where(rng.random(200_000) < 0.5, -1.0, 1.0)
    x = sign * (1.0 + 9.0 * rng.random(200_000)) * 10.0 ** rng.integers(-30, 15, 200_000)
    x[::97] = np.round(x[::97], 3)  # short decimals and exact ties in binary
    x[x == 0] = 0.5
    m = x.reshape(-1, 4)
    formats.save_embeddings_text(m, _Vocab([str(i) for i in range(len(m))]), tmp_path / "r")
    lines = (tmp_path / "r").read_text().splitlines()[1:]
    got = [c for line in lines for c in line.split(" ")[1:]]
    assert got == [format(v, ".8g") for v in x.tolist()]


def test_wvc1_writer_byte_exact(tmp_path):
    import paper_2508_01073_b200 as wv
    from paper_2508_01073_b200 import formats

    c = wv.WalkCorpus(np.array(G["wvc1_tokens"]), np.array(G["wvc1_offsets"]), wv.BFS, wv.ENTITY)
    formats.save_corpus_binary(c, tmp_path / "c.wvc")
    assert (tmp_path / "c.wvc").read_bytes() == base64.b64decode(G["wvc1"])


def _wvc1_bytes(seqs, strategy=0, projection=0, count=None):
    import struct

    body = []
    for s in seqs:
        body.append(len(s))
        body.extend(s)
    hdr = b"WVC1" + struct.pack("<BBHI", strategy, projection, 0, len(seqs) if count is None else count)
    return hdr + np.array(body, dtype="<u4").tobytes()


def test_wvc1_reader_reference_fixture(tmp_path):
    """The reference's own WVC1 file (tests/golden/formats.json) reads back to its corpus."""
    import paper_2508_01073_b200 as wv
    from paper_2508_01073_b200 import formats

    (tmp_path / "c.wvc").write_bytes(base64.b64decode(G["wvc1"]))
    c = formats.load_corpus_binary(tmp_path / "c.wvc")
    assert np.array_equal(c.tokens, np.array(G["wvc1_tokens"])) and np.array_equal(c.offsets, G["wvc1_offsets"])
    assert c.strategy == wv.BFS and c.projection == wv.ENTITY


@pytest.mark.parametrize("n,maxlen,seed", [(0, 1, 0), (1, 5, 1), (1000, 9, 2), (200_000, 33, 3), (30_000, 300, 4),
                                           (50_000, 140, 5)])
def test_wvc1_reader_round_trip(tmp_path, n, maxlen, seed):
    """Random corpora across chunk boundaries (8192-word chunks, 128-word speculation window),
    empty walks, and records longer than the window (the sequential path) read back exactly,
    equal to the reference's reader restated (walks.py:368-389)."""
    from paper_2508_01073_b200 import formats

    rng = np.random.default_rng(seed)
    seqs = [rng.integers(0, 2**31 - 1, rng.integers(0, maxlen + 1)).tolist() for _ in range(n)]
    (tmp_path / "r.wvc").write_bytes(_wvc1_bytes(seqs, 1, 2))
    c = formats.load_corpus_binary(tmp_path / "r.wvc")
    lens = np.array([len(s) for s in seqs], dtype=np.int64)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    tok = np.array([t for s in seqs for t in s], dtype=np.int64)
    assert len(c) == n and np.array_equal(c.offsets, off) and np.array_equal(c.tokens, tok)


def test_wvc1_reader_errors(tmp_path):
    """Reference error behaviour: bad magic -> ValueError; words left after `count` records or a
    record running past the body -> ValueError; the body ending before `count` records -> IndexError."""
    from paper_2508_01073_b200 import formats

    p = tmp_path / "e.wvc"
    p.write_bytes(b"WVCX" + _wvc1_bytes([[1]])[4:])
    with pytest.raises(ValueError, match="not a walk corpus file"):
        formats.load_corpus_binary(p)
    p.write_bytes(_wvc1_bytes([[1, 2], [3]], count=1))  # trailing record
    with pytest.raises(ValueError, match="corrupt"):
        formats.load_corpus_binary(p)
    good = _wvc1_bytes([[1, 2], [3]])
    p.write_bytes(good[:-4])  # the last record runs past the body
    with pytest.raises(ValueError):
        formats.load_corpus_binary(p)
    p.write_bytes(_wvc1_bytes([[1, 2], [3]], count=3))  # fewer records than the header says
    with pytest.raises(IndexError):
        formats.load_corpus_binary(p)


def test_vocabulary_tsv_byte_exact(tmp_path):
    """Vocabulary.save_tsv's bytes (reference output in tests/golden/formats.json): escaped
    tabs / newlines / backslashes / CR, UTF-8, an empty lexical, roles e / p / ep, frequencies."""
    from paper_2508_01073_b200 import formats

    class Voc:
        lexical_of = G["vocab_lexicals"]
        _entity_tokens = set(G["vocab_entities"])
        _predicate_tokens = set(G["vocab_predicates"])
        frequency = np.array(G["vocab_frequency"])

    formats.save_vocabulary_tsv(Voc(), tmp_path / "v.tsv")
    assert (tmp_path / "v.tsv").read_bytes() == base64.b64decode(G["vocab_tsv"])
