"""The CPU oracle against the reference's own outputs (golden fixtures) and known answers."""

import json
import math

import numpy as np
import pytest

from oracle import rng as orng
from oracle import walks as ow
from oracle import w2v as ov
from conftest import GOLDEN


def test_seedseq_and_streams_match_numpy_golden(golden):
    g = golden("seedseq.npz")
    ents = json.loads(str(g["entropies"]))
    for i, e in enumerate(ents):
        assert orng.generate_state_u64(e, 4) == [int(x) for x in g[f"state4_{i}"]]
        pcg = orng.PCG64(e)
        for k, want in zip([0, 1, 2, 3, 999, 1000, 1099], g[f"pcg_{i}"]):
            assert pcg.u64_at(k) == int(want)
        ph = orng.Philox(e)
        for k, want in zip([0, 1, 2, 3, 4, 5, 999, 1000, 1099], g[f"philox_{i}"]):
            assert ph.u64_at(k) == int(want)


def test_double_conversion_matches_numpy():
    gen = np.random.default_rng(np.random.SeedSequence([42, 0, 3]))
    want = gen.random(5)
    pcg = orng.PCG64([42, 0, 3])
    assert [orng.to_double(pcg.u64_at(k)) for k in range(5)] == want.tolist()


def _walk_case(g, i):
    p = g[f"c{i}_params"]
    seed = int(str(g[f"c{i}_seed"]))
    return g[f"c{i}_edges"], int(g[f"c{i}_V"]), g[f"c{i}_roots"], int(p[0]), int(p[1]), seed, bool(p[3])


@pytest.mark.parametrize("kind", ["pcg64", "philox"])
def test_walk_oracle_matches_reference(golden, kind):
    g = golden("walks.npz")
    tag = "pcg" if kind == "pcg64" else "philox"
    for i in range(int(g["n_cases"])):
        edges, V, roots, depth, number, seed, dup = _walk_case(g, i)
        off, tgt, prd = ow.csr(edges, V)
        assert np.array_equal(off, g[f"c{i}_row_offsets"])
        assert np.array_equal(tgt, g[f"c{i}_col_targets"])
        assert np.array_equal(prd, g[f"c{i}_col_predicates"])
        tok, offs = ow.random_walks(off, tgt, prd, roots, depth, number, seed, kind, dup)
        assert np.array_equal(tok, g[f"c{i}_{tag}_tokens"]), i
        assert np.array_equal(offs, g[f"c{i}_{tag}_offsets"]), i


def test_counter_addressed_draws_equal_sequential_stream(golden):
    """The GPU addressing (k = hop * n_shard + row) restated with jump-ahead, vs numpy's sequential stream."""
    g = golden("walks.npz")
    edges, V, roots, depth, number, seed, _ = _walk_case(g, 0)
    off, tgt, prd = ow.csr(edges, V)
    work = np.repeat(roots, number)
    n_sh = -(-len(work) // ow.SHARD)
    s = n_sh - 1  # the partial shard
    n_s = len(work) - s * ow.SHARD
    pcg = orng.PCG64([seed, 0, s])
    seq = np.random.default_rng(np.random.SeedSequence([seed, 0, s])).random(3 * n_s)
    for h in range(3):
        for i in (0, 1, n_s - 1):
            assert orng.to_double(pcg.u64_at(h * n_s + i)) == seq[h * n_s + i]


def test_bfs_oracle_matches_reference(golden):
    g = golden("bfs.npz")
    for i in range(int(g["n_cases"])):
        off, tgt, prd = ow.csr(g[f"c{i}_edges"], int(g[f"c{i}_V"]))
        tok, offs, rows = ow.bfs_walks(off, tgt, prd, g[f"c{i}_roots"], int(g[f"c{i}_depth"]))
        assert np.array_equal(tok, g[f"c{i}_tokens"])
        assert np.array_equal(offs, g[f"c{i}_offsets"])
        assert np.array_equal(np.array(rows, dtype=np.int64).reshape(-1, 3), g[f"c{i}_table"])


def test_init_and_pairs_match_reference(golden):
    g = golden("w2v.npz")
    a, b = ov.init(37, 13, 5)
    assert np.array_equal(a, g["init_in"]) and np.array_equal(b, g["init_out"])
    toks, offs = g["pairs_tokens"], g["pairs_offsets"]
    freq = ov.frequencies(toks, 12)
    assert np.array_equal(freq, g["pairs_freq"])
    ft, fo = ov.filtered(toks, offs, freq >= 6)
    assert np.array_equal(ov.pairs(ft, fo, 3), g["pairs"])


@pytest.mark.parametrize("name", ["sparse", "dense", "auto"])
def test_train_oracle_matches_reference(golden, name):
    g = golden("w2v.npz")
    kw = json.loads(str(g[f"{name}_cfg"]))
    r = ov.train(g["train_tokens"], g["train_offsets"], int(g["train_V"]), kw["vector_size"], kw["window_size"],
                 kw["negative_samples"], kw.get("learning_rate", 0.01), kw["min_count"], kw["epochs"], 42,
                 batch=kw.get("batch_size"), sparse=kw.get("use_sparse", True))
    np.testing.assert_allclose(r["inp"], g[f"{name}_in"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(r["out"], g[f"{name}_out"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(r["losses"], g[f"{name}_losses"], rtol=1e-12)
    assert np.array_equal(r["touched_in"], g[f"{name}_touched_in"])
    assert np.array_equal(r["touched_out"], g[f"{name}_touched_out"])


def test_zero_state_loss_known_answer():
    """SGNS loss with all-zero embeddings is (1+k) ln 2 = 6 ln 2 for k=5 (reference test_w2v.py:151-160)."""
    z = np.zeros((4, 3))
    loss, *_ = ov.sgns_step(z, z, np.array([0, 1]), np.array([2, 3]), np.array([[0, 1, 2, 3, 0]] * 2))
    assert abs(loss - 6 * math.log(2)) < 1e-12
    assert abs(ov.scalar_loss(z, z, [0, 1], [2, 3], [[0, 1, 2, 3, 0]] * 2) - 6 * math.log(2)) < 1e-12


def test_batch_rule_known_answers():
    # reference SPEC.md:335-337 examples, and the 1 GiB rule at cfg1 / cfg2
    assert ov.batch_size(10**6, 100, 5, budget=1 << 62) == 50_000
    assert ov.batch_size(5_737_534, 100, 5) == 47_798
    assert ov.batch_size(10**10, 200, 5) == 23_933


def test_two_clique_reference_statistics():
    runs = json.loads((GOLDEN / "two_clique.json").read_text())["runs"]
    m = np.array([r["margin"] for r in runs])
    assert len(runs) == 10 and m.min() > 0.3 and all(r["loss_last"] < r["loss0"] for r in runs)


def test_cbow_instances_match_reference(golden):
    g = golden("cbow.npz")
    toks, offs = g["inst_tokens"], g["inst_offsets"]
    freq = ov.frequencies(toks, 12)
    assert np.array_equal(freq, g["inst_freq"])
    ft, fo = ov.filtered(toks, offs, freq >= 6)
    ctx, lens, tg = ov.cbow_instances(ft, fo, 3)
    assert np.array_equal(ctx, g["inst_ctx"]) and np.array_equal(lens, g["inst_lengths"])
    assert np.array_equal(tg, g["inst_targets"])


@pytest.mark.parametrize("name", ["sparse", "dense", "auto"])
def test_cbow_train_oracle_matches_reference(golden, name):
    g = golden("cbow.npz")
    kw = json.loads(str(g[f"{name}_cfg"]))
    r = ov.train(g["train_tokens"], g["train_offsets"], int(g["train_V"]), kw["vector_size"], kw["window_size"],
                 0, kw.get("learning_rate", 0.01), kw["min_count"], kw["epochs"], 42,
                 batch=kw.get("batch_size"), sparse=kw.get("use_sparse", True), model="cbow")
    np.testing.assert_allclose(r["inp"], g[f"{name}_in"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(r["out"], g[f"{name}_out"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(r["losses"], g[f"{name}_losses"], rtol=1e-12)
    assert np.array_equal(r["touched_in"], g[f"{name}_touched_in"])
    assert np.array_equal(r["touched_out"], g[f"{name}_touched_out"])


def test_synth_oracle_structure_and_encoding():
    """oracle/synth.py: BA structure (benchgen.py:78-109 invariants) and the first-occurrence
    encoding equal to the reference vocabulary fixture's rule (ingest.py:368-396)."""
    from oracle import synth as osy

    n, m = 3000, 6
    src, dst = osy.barabasi_edges(n, m, 11)
    v = np.arange(1, n)
    assert np.array_equal(src, np.repeat(v, np.minimum(m, v)))
    assert (dst < src).all() and (dst >= 0).all()
    assert len(np.unique(src * n + dst)) == len(src)
    assert osy.ba_edge_count(n, m) == len(src)
    # in-degree + 1 attachment: old vertices collect far more edges than young ones
    indeg = np.bincount(dst, minlength=n)
    assert indeg[:30].mean() > 10 * indeg[-1000:].mean()
    # encoding: tokens by first occurrence over (s, p, o), shared space, entity/predicate split
    edges, V, ent, prd = osy.encode(np.array([5, 2, 5]), np.array([1, 0, 1]), np.array([2, 7, 7]), 10)
    assert edges.tolist() == [[0, 1, 2], [2, 3, 4], [0, 1, 4]]
    assert V == 5 and ent.tolist() == [0, 2, 4] and prd.tolist() == [1, 3]


def test_synth_oracle_mulhi_and_philox():
    from oracle import synth as osy

    rng = np.random.default_rng(0)
    a = rng.integers(0, 2**63, 1000, dtype=np.int64).astype(np.uint64) * np.uint64(2) + np.uint64(1)
    b = rng.integers(0, 2**63, 1000, dtype=np.int64).astype(np.uint64)
    got = osy.mulhi64(a, b)
    want = [(int(x) * int(y)) >> 64 for x, y in zip(a, b)]
    assert [int(x) for x in got] == want
    # Philox4x32-10 known-answer vectors (Random123 kat_vectors: philox4x32 10 rounds)
    c = osy.philox4x32_10([0], [0], [0], [0], 0, 0)
    assert [int(x[0]) for x in c] == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    c = osy.philox4x32_10([0xFFFFFFFF] * 1, [0xFFFFFFFF], [0xFFFFFFFF], [0xFFFFFFFF], 0xFFFFFFFF, 0xFFFFFFFF)
    assert [int(x[0]) for x in c] == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]


def test_synth_encoding_matches_reference_vocabulary(golden):
    """oracle/synth.encode on the reference's own BA edges and predicate picks reproduces the
    reference's build_vocabulary encoding (tests/golden/vocab.npz, ingest.py:368-396)."""
    from oracle import synth as osy

    g = golden("vocab.npz")
    raw = g["raw"]
    edges, V, ent, _ = osy.encode(raw[:, 0], g["picks"], raw[:, 1], 300)
    assert np.array_equal(edges, g["edges"]) and V == int(g["V"])
    assert np.array_equal(ent, g["entity_tokens"])
