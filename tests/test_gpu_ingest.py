"""GPU ingest against the reference's own parse + build_vocabulary
outputs (tests/golden/ingest.json, made by tests/golden/make_golden.py from
/root/reference): tokens, lexical keys, roles, edges and errors, exactly."""

import json

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

CASES = json.loads((GOLDEN / "ingest.json").read_text())


TRIPLES = [c for c in CASES if "triples" in c]
CASES = [c for c in CASES if "triples" not in c]


@pytest.mark.parametrize("case", TRIPLES, ids=[c["name"] for c in TRIPLES])
def test_build_vocabulary_on_triples_matches_reference(case):
    """Triple streams with keys holding spaces, '>', backslashes, newlines, quotes, non-ASCII."""
    from collections import namedtuple

    import paper_2508_01073_b200 as wv

    Tr = namedtuple("Tr", "subject predicate object object_kind")
    vocab, edges = wv.build_vocabulary([Tr(*r) for r in case["triples"]], include_literals=case["include_literals"])
    assert vocab.lexical_of == case["lexicals"] and edges.tolist() == case["edges"]
    assert vocab.entity_tokens().tolist() == case["entities"]
    assert sorted(vocab._predicate_tokens) == case["predicates"]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_ingest_matches_reference(case):
    from paper_2508_01073_b200.ingest import ParseError, load_triples_device

    kw = dict(format=case["format"], strict=case["strict"], include_literals=case["include_literals"],
              has_header=case.get("has_header", False))
    data = case["text"].encode("utf-8")
    if "error" in case:
        with pytest.raises(ParseError) as err:
            load_triples_device(data, **kw)
        assert [err.value.line, err.value.reason] == case["error"]
        return
    if "value_error" in case:
        with pytest.raises(ValueError, match=case["value_error"]):
            load_triples_device(data, **kw)
        return
    sink = []
    vocab, edges = load_triples_device(data, error_sink=sink, **kw)
    assert vocab.lexical_of == case["lexicals"]
    assert edges.tolist() == case["edges"]
    assert vocab.entity_tokens().tolist() == case["entities"]
    assert sorted(vocab._predicate_tokens) == case["predicates"]
    assert [[e.line, e.reason] for e in sink] == case.get("errors", [])


def test_ingest_synthetic_scale_matches_integer_encoding():
    """A 200k-statement N-Triples document: tokens equal the vectorised encoder's."""
    from paper_2508_01073_b200.ingest import encode_integer_triples, load_triples_device

    rng = np.random.default_rng(4)
    n, E, P = 20_000, 200_000, 37
    src, dst, pk = rng.integers(0, n, E), rng.integers(0, n, E), rng.integers(0, P, E)
    text = "".join(f"<v{s}> <P{p}> <v{d}> .\n" for s, p, d in zip(src.tolist(), pk.tolist(), dst.tolist()))
    vocab, edges = load_triples_device(text.encode())
    ref_edges, V, ents, preds, lex = encode_integer_triples(src, pk, dst, n, with_lexicals=True)
    assert np.array_equal(edges, ref_edges) and vocab.lexical_of == lex
    assert np.array_equal(vocab.entity_tokens(), ents)


def test_load_data_file_and_errors(tmp_path):
    """pipeline.load_data (pipeline.py:117-135): format from the extension, PipelineError('ingest')."""
    import paper_2508_01073_b200 as wv

    case = CASES[0]
    f = tmp_path / "g.nt"
    f.write_bytes(case["text"].encode("utf-8"))
    vocab, edges = wv.load_data(str(f))
    assert vocab.lexical_of == case["lexicals"] and edges.tolist() == case["edges"]
    with pytest.raises(ValueError, match="format unsupported: parquet"):
        wv.load_data(str(tmp_path / "g.parquet"))
    bad = tmp_path / "bad.nt"
    bad.write_bytes(b"<a> <p> <b>\n")
    with pytest.raises(wv.PipelineError):
        wv.load_data(str(bad), strict=True)
