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
