"""End to end through the drop-in API (pipeline.py:117-219): GPU ingest of an .nt file,
graph, walks (random / BFS, duplicate_free, projections), skip-gram / CBOW training
replaying the reference's numpy streams in float64 -- against the reference's own
load_data + fit_transform outputs (tests/golden/pipeline.json)."""

import json

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

G = json.loads((GOLDEN / "pipeline.json").read_text())


@pytest.mark.parametrize("name", sorted(G["cases"]))
def test_fit_transform_matches_reference(tmp_path, name):
    import paper_2508_01073_b200 as wv

    case = G["cases"][name]
    f = tmp_path / "g.nt"
    f.write_text(G["text"])
    vocab, edges = wv.load_data(str(f))
    assert vocab.lexical_of == case["lexicals"]
    table = wv.fit_transform(edges, vocab, wv.PipelineConfig(**case["cfg"]), precision="fp64", pairs="numpy")
    np.testing.assert_allclose(table.vectors, np.array(case["vectors"]), rtol=0, atol=1e-10)
    np.testing.assert_allclose(table.losses, case["losses"], rtol=1e-10)
    assert table.trained_mask.tolist() == case["trained"]
    assert vocab.frequency.tolist() == case["frequency"]
