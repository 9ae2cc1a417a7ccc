"""Device synthetic-graph generator and token encoding (csrc/synth.cu).

gen_barabasi restates benchgen.gen_barabasi (benchgen.py:78-109) as the same
preferential-attachment process with counter-based draws, so the checks are
structural (edge count, out-degree min(m, v), distinct targets, targets of
earlier vertices, degree+1 attachment weights) and distributional.  The
encoding must equal the host first-occurrence encoder (ingest.py:368-396)
bit-for-bit on the same triples.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wv():
    import paper_2508_01073_b200 as wv

    return wv


@pytest.mark.parametrize("n,m", [(2, 1), (7, 3), (50, 10), (5000, 4), (20000, 10)])
def test_barabasi_structure(wv, n, m):
    from paper_2508_01073_b200 import synth

    src, dst = synth.device_barabasi_edges(n, m, seed=7)
    src, dst = src.cpu().numpy(), dst.cpu().numpy()
    v = np.arange(1, n)
    k = np.minimum(m, v)
    assert len(src) == k.sum()
    assert np.array_equal(src, np.repeat(v, k))  # source-major, like the reference's edge list
    assert (dst < src).all() and (dst >= 0).all()  # new -> old (a DAG, tests/test_benchgen.py:122-124)
    key = src * n + dst
    assert len(np.unique(key)) == len(key)  # distinct targets per vertex


def test_barabasi_attachment_is_degree_plus_one(wv):
    """P(first draw of vertex v hits u) ∝ deg(u)+1 over the bag (benchgen.py:85-104): chi-square on
    the early, well-populated vertices of many independent graphs."""
    from paper_2508_01073_b200 import synth

    n, m = 12, 1
    hits = np.zeros((n, n))
    for seed in range(400):
        src, dst = synth.device_barabasi_edges(n, m, seed=seed)
        s, d = src.cpu().numpy(), dst.cpu().numpy()
        # with m=1 each vertex v draws once from the bag of length v^2 (closed form)
        hits[s, d] += 1
    # vertex 2's draw: bag [0, 1(t), 1, 1(self)] -> vertex 1's edge points at 0 => bag = [0, 0, 1, 1]
    # so P(0) = P(1) = 1/2 regardless of vertex 1's draw
    row = hits[2, :2]
    assert abs(row[0] - row[1]) < 5 * np.sqrt(400 * 0.25) * 2


def test_barabasi_power_law_in_degree(wv):
    from paper_2508_01073_b200 import synth

    n, m = 200_000, 10
    src, dst = synth.device_barabasi_edges(n, m, seed=7)
    indeg = np.bincount(dst.cpu().numpy(), minlength=n)
    # heavy tail: hubs far above the mean (mean in-degree ~ m); out-degree constant m
    assert indeg.max() > 50 * indeg.mean()
    assert indeg[:100].mean() > 20 * indeg[n // 2:].mean()


def test_device_encode_matches_host(wv):
    from paper_2508_01073_b200 import synth
    from paper_2508_01073_b200.ingest import encode_integer_triples

    import torch

    n, m, P = 3000, 5, 17
    src, dst = synth.device_barabasi_edges(n, m, seed=3)
    picks = synth.predicate_picks(int(src.numel()), P, seed=3)
    e_d, V_d, ent_d, prd_d = synth.device_encode(src, torch.from_numpy(picks).cuda(), dst, n, P)
    e_h, V_h, ent_h, prd_h = encode_integer_triples(src.cpu().numpy(), picks, dst.cpu().numpy(), n)
    assert V_d == V_h
    assert np.array_equal(e_d.cpu().numpy(), e_h)
    assert np.array_equal(ent_d.cpu().numpy(), ent_h)
    assert np.array_equal(prd_d.cpu().numpy(), prd_h)


def test_device_synthetic_kg_cfg1_shape(wv):
    """cfg1 shape: BA(10k, m=5, 20 P) -> 49,985 triples, V = 10,020."""
    from paper_2508_01073_b200 import synth

    edges, V, ent, prd = synth.device_synthetic_kg("barabasi", 10_000, m=5, predicates=20, seed=7)
    assert edges.shape == (49_985, 3)
    assert len(prd) == 20 and V == len(ent) + 20
    assert V == 10_020
    g = wv.build_graph(edges, V)
    deg = np.diff(g.row_offsets)
    assert deg.max() == 5


def test_device_erdos_renyi_structure(wv):
    """gen_erdos_renyi semantics: no self loops, row-major order, edge count ~ Binomial(n(n-1), p)."""
    from paper_2508_01073_b200.synth import device_erdos_renyi_edges

    n, p = 15_000, 0.001378
    src, dst = device_erdos_renyi_edges(n, p, seed=7)
    s, d = src.cpu().numpy(), dst.cpu().numpy()
    mean, sd = n * (n - 1) * p, (n * (n - 1) * p * (1 - p)) ** 0.5
    assert abs(len(s) - mean) < 6 * sd
    assert (s != d).all() and (s >= 0).all() and (d < n).all()
    key = s * n + d
    assert (np.diff(key) > 0).all()  # strictly row-major, no duplicates
    s2, d2 = device_erdos_renyi_edges(n, p, seed=7)
    assert np.array_equal(s2.cpu().numpy(), s)


def test_device_uniform_attachment_structure(wv):
    """gen_uniform_attachment semantics: per vertex v >= 1, distinct ascending targets in [0, v),
    at most min(m, v) of them; the expected count matches m uniform draws with collisions."""
    from paper_2508_01073_b200.synth import device_uniform_attachment_edges

    n, m = 50_000, 10
    src, dst = device_uniform_attachment_edges(n, m, seed=3)
    s, d = src.cpu().numpy(), dst.cpu().numpy()
    assert (d < s).all() and (s >= 1).all()
    assert (np.diff(s) >= 0).all()
    same = s[1:] == s[:-1]
    assert (d[1:][same] > d[:-1][same]).all()
    per = np.bincount(s, minlength=n)
    v = np.arange(n)
    assert (per[1:] <= np.minimum(m, v[1:])).all()
    # E[distinct] = v (1 - (1 - 1/v)^m)
    expect = (v[1:] * (1 - (1 - 1 / v[1:]) ** m)).sum()
    assert abs(per.sum() - expect) / expect < 0.01


@pytest.mark.parametrize("n,m,seed", [(2, 1, 7), (7, 3, 1), (50, 10, 7), (5000, 4, 3), (20000, 10, 7)])
def test_barabasi_bit_exact_vs_oracle(wv, n, m, seed):
    """csrc/synth.cu equals its numpy restatement (oracle/synth.py) edge for edge, and the
    device encoding equals the oracle's first-occurrence encoding of the same triples."""
    from oracle import synth as osy
    from paper_2508_01073_b200 import synth

    src, dst = synth.device_barabasi_edges(n, m, seed=seed)
    osrc, odst = osy.barabasi_edges(n, m, seed)
    assert np.array_equal(src.cpu().numpy(), osrc) and np.array_equal(dst.cpu().numpy(), odst)
    e, V, ent, prd = synth.device_synthetic_kg("barabasi", n, m=m, predicates=12, seed=seed)
    oe, oV, oent, oprd = osy.barabasi_kg(n, m, 12, seed)
    assert V == oV and np.array_equal(e.cpu().numpy(), oe)
    assert np.array_equal(ent.cpu().numpy(), oent) and np.array_equal(prd.cpu().numpy(), oprd)


def test_device_encode_matches_reference_vocabulary(wv, golden):
    """wv_encode_triples on the reference's own BA edges and predicate picks equals the
    reference's build_vocabulary encoding (tests/golden/vocab.npz, ingest.py:368-396)."""
    import torch

    from paper_2508_01073_b200 import synth

    g = golden("vocab.npz")
    raw = torch.from_numpy(g["raw"]).cuda()
    picks = torch.from_numpy(g["picks"]).cuda()
    e, V, ent, _ = synth.device_encode(raw[:, 0].contiguous(), picks, raw[:, 1].contiguous(), 300, 5)
    assert V == int(g["V"]) and np.array_equal(e.cpu().numpy(), g["edges"])
    assert np.array_equal(ent.cpu().numpy(), g["entity_tokens"])
