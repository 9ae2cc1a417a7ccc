"""GPU parity for SGNS training: replay of the reference streams, tolerances stated per test."""

import json
import math

import numpy as np
import pytest

from oracle import w2v as ov
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wv():
    import paper_2508_01073_b200 as wv

    return wv


def _corpus(wv, g):
    return wv.WalkCorpus(g["train_tokens"], g["train_offsets"])


def test_init_bit_exact(golden, wv):
    g = golden("w2v.npz")
    for prec in ("fp64", "fp32"):
        m = wv.init_embeddings(37, 13, 5, precision=prec)
        if prec == "fp64":
            assert np.array_equal(m.input_matrix, g["init_in"]) and np.array_equal(m.output_matrix, g["init_out"])
        else:  # fp32 store: values are the rounded init
            np.testing.assert_array_equal(m.input_matrix, g["init_in"].astype(np.float32).astype(np.float64))


def test_generate_pairs_matches_reference(golden, wv):
    g = golden("w2v.npz")
    corpus = wv.WalkCorpus(g["pairs_tokens"], g["pairs_offsets"])
    pairs, freq = wv.generate_pairs(corpus, 3, 6, 12)
    assert np.array_equal(pairs, g["pairs"]) and np.array_equal(freq, g["pairs_freq"])


# fp64 replay of the reference's own streams: 1e-10 absolute on parameters of magnitude <~1
@pytest.mark.parametrize("name", ["sparse", "dense", "auto", "multi", "multi3"])
def test_train_replay_fp64_matches_reference(golden, wv, name):
    g = golden("w2v.npz")
    kw = json.loads(str(g[f"{name}_cfg"]))
    model, losses = wv.train(_corpus(wv, g), int(g["train_V"]), wv.TrainConfig(**kw), 42, precision="fp64",
                             pairs="numpy")
    np.testing.assert_allclose(model.input_matrix, g[f"{name}_in"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(model.output_matrix, g[f"{name}_out"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(losses, g[f"{name}_losses"], rtol=1e-10)
    assert np.array_equal(model.touched_input, g[f"{name}_touched_in"])
    assert np.array_equal(model.touched_output, g[f"{name}_touched_out"])


# fp32 parameter store, same streams: 1e-4 absolute, loss 1e-5 relative
@pytest.mark.parametrize("name", ["sparse", "auto"])
def test_train_replay_fp32_within_tolerance(golden, wv, name):
    g = golden("w2v.npz")
    kw = json.loads(str(g[f"{name}_cfg"]))
    model, losses = wv.train(_corpus(wv, g), int(g["train_V"]), wv.TrainConfig(**kw), 42, precision="fp32",
                             pairs="numpy")
    np.testing.assert_allclose(model.input_matrix, g[f"{name}_in"], rtol=0, atol=1e-4)
    np.testing.assert_allclose(model.output_matrix, g[f"{name}_out"], rtol=0, atol=1e-4)
    np.testing.assert_allclose(losses, g[f"{name}_losses"], rtol=1e-5)


def test_device_mode_deterministic_and_untouched_rows_exact(golden, wv):
    g = golden("w2v.npz")
    cfg = wv.TrainConfig(min_count=2, vector_size=12, epochs=2, window_size=3, negative_samples=4, batch_size=64)
    a, la = wv.train(_corpus(wv, g), int(g["train_V"]) + 5, cfg, 11)
    b, lb = wv.train(_corpus(wv, g), int(g["train_V"]) + 5, cfg, 11)
    assert np.array_equal(a.input_matrix, b.input_matrix) and np.array_equal(a.output_matrix, b.output_matrix)
    assert la == lb
    fresh_in, fresh_out = ov.init(int(g["train_V"]) + 5, 12, 11)
    assert np.array_equal(a.input_matrix[~a.touched_input], fresh_in[~a.touched_input])
    assert np.array_equal(a.output_matrix[~a.touched_output], fresh_out[~a.touched_output])
    assert (~a.touched_input[-5:]).all()


def test_zero_lr_keeps_init(golden, wv):
    g = golden("w2v.npz")
    cfg = wv.TrainConfig(min_count=0, vector_size=6, epochs=1, learning_rate=0.0, window_size=2, negative_samples=2)
    m, _ = wv.train(_corpus(wv, g), int(g["train_V"]), cfg, 7)
    a, b = ov.init(int(g["train_V"]), 6, 7)
    assert np.array_equal(m.input_matrix, a) and np.array_equal(m.output_matrix, b)


def test_divergence_raises(golden, wv):
    g = golden("w2v.npz")
    cfg = wv.TrainConfig(min_count=0, vector_size=4, epochs=5, learning_rate=1e200, window_size=2,
                         negative_samples=2)
    with pytest.raises(wv.TrainingDiverged) as err:
        wv.train(_corpus(wv, g), int(g["train_V"]), cfg, 0)
    assert "divergence at epoch" in str(err.value)


def test_empty_training_set_and_batch_halving(golden, wv):
    g = golden("w2v.npz")
    with pytest.raises(ValueError, match="empty training set"):
        wv.train(_corpus(wv, g), int(g["train_V"]), wv.TrainConfig(min_count=10**6, vector_size=4, epochs=1), 0)
    events = []
    cfg = wv.TrainConfig(min_count=0, vector_size=8, epochs=1, window_size=2, negative_samples=2, batch_size=4096,
                         memory_budget_bytes=wv.estimate_per_sample_bytes("skipgram", 8, 2, 2) * 64)
    _, losses = wv.train(_corpus(wv, g), int(g["train_V"]), cfg, 1, on_event=lambda k, **i: events.append(k))
    assert "batch_halved" in events and len(losses) == 1


def test_sparse_isolation_below_min_count(wv):
    corpus = [[0, 1, 2]] * 10 + [[0, 3, 4]] * 2
    cfg = wv.TrainConfig(min_count=5, vector_size=8, epochs=3, window_size=2, negative_samples=2)
    m, _ = wv.train(corpus, 5, cfg, 5)
    a, b = ov.init(5, 8, 5)
    assert m.trained_mask.tolist() == [True, True, True, False, False]
    for r in (3, 4):
        assert np.array_equal(m.input_matrix[r], a[r]) and np.array_equal(m.output_matrix[r], b[r])


@pytest.mark.parametrize("pairs", ["device", "numpy"])
def test_two_clique_separation_within_reference_band(wv, pairs):
    """Downstream check (reference test_acceptance.py:256-276): margin and final loss within mean +- 4 sigma."""
    ref = json.loads((GOLDEN / "two_clique.json").read_text())
    margins = np.array([r["margin"] for r in ref["runs"]])
    finals = np.array([r["loss_last"] for r in ref["runs"]])
    graph = wv.build_graph(np.array(ref["edges"]), ref["V"])
    got_m, got_l = [], []
    for r in ref["runs"][:5]:
        corpus = wv.random_walks(graph, ref["roots"], walk_depth=4, walk_number=25, rng_seed=r["seed"])
        cfg = wv.TrainConfig(min_count=1, vector_size=16, epochs=10, learning_rate=0.01, window_size=5,
                             negative_samples=5)
        model, losses = wv.train(corpus, ref["V"], cfg, r["seed"], pairs=pairs)
        v = model.input_matrix

        def cos(a, b):
            return float(np.dot(v[a], v[b]) / (np.linalg.norm(v[a]) * np.linalg.norm(v[b])))

        x, y = ref["x"], ref["y"]
        intra = [cos(a, b) for grp in (x, y) for a in grp for b in grp if a < b]
        inter = [cos(a, b) for a in x for b in y]
        got_m.append(np.mean(intra) - np.mean(inter))
        got_l.append(losses[-1])
        assert losses[-1] < losses[0]
    assert abs(np.mean(got_m) - margins.mean()) < 4 * margins.std() + 1e-3
    assert abs(np.mean(got_l) - finals.mean()) < 4 * finals.std() + 1e-3


def test_device_mode_loss_tracks_oracle_statistics(wv):
    """Device RNG streams vs numpy streams: same corpus, epoch-1 loss within 1%."""
    from paper_2508_01073_b200.synth import synthetic_kg

    edges, V, ents, _ = synthetic_kg("barabasi", 3000, m=5, predicates=20, seed=7)
    graph = wv.build_graph(edges, V)
    corpus = wv.random_walks(graph, ents, walk_depth=4, walk_number=10, rng_seed=42)
    cfg = wv.TrainConfig(min_count=1, vector_size=32, epochs=1, window_size=5, negative_samples=5)
    _, l_dev = wv.train(corpus, V, cfg, 42, pairs="device")
    _, l_np = wv.train(corpus, V, cfg, 42, pairs="numpy")
    assert abs(l_dev[0] - l_np[0]) / l_np[0] < 0.01


def test_pipelined_batches_equal_sequential(wv):
    """wv_sgns_batches (decode/group of batch i+1 overlapping batch i, two workspace
    halves; CUDA-graph replayed or eager) is bit-identical to one wv_sgns_batch call
    per batch (the profiled path)."""
    from paper_2508_01073_b200.synth import synthetic_kg

    edges, V, ents, _ = synthetic_kg("barabasi", 2000, m=5, predicates=20, seed=3)
    graph = wv.build_graph(edges, V)
    corpus = wv.random_walks(graph, ents, walk_depth=4, walk_number=4, rng_seed=9)
    cfg = wv.TrainConfig(min_count=1, vector_size=24, epochs=1, window_size=3, negative_samples=4, batch_size=997)
    out = []
    for graph_batches, profile in ((8, False), (1, False), (8, True)):
        sess = wv.SkipGramSession(V, cfg, 5, graph_batches=graph_batches)
        losses = sess.fit(corpus, 2, profile=profile)
        out.append((sess.model.input_matrix, sess.model.output_matrix, losses))
    for a in out[1:]:
        assert np.array_equal(out[0][0], a[0]) and np.array_equal(out[0][1], a[1]) and out[0][2] == a[2]


# ---------------------------------------------------------------- CBOW --
def test_cbow_instances_match_reference(golden, wv):
    g = golden("cbow.npz")
    corpus = wv.WalkCorpus(g["inst_tokens"], g["inst_offsets"])
    ctx, lens, tg, freq = wv.generate_cbow_instances(corpus, 3, 6, 12)
    assert np.array_equal(ctx, g["inst_ctx"]) and np.array_equal(lens, g["inst_lengths"])
    assert np.array_equal(tg, g["inst_targets"]) and np.array_equal(freq, g["inst_freq"])


# fp64 replay of the reference's CBOW streams: 1e-10 absolute on parameters
@pytest.mark.parametrize("name", ["sparse", "dense", "auto", "multi"])
def test_cbow_replay_fp64_matches_reference(golden, wv, name):
    g = golden("cbow.npz")
    kw = json.loads(str(g[f"{name}_cfg"]))
    corpus = wv.WalkCorpus(g["train_tokens"], g["train_offsets"])
    model, losses = wv.train(corpus, int(g["train_V"]), wv.TrainConfig(**kw), 42, precision="fp64", pairs="numpy")
    np.testing.assert_allclose(model.input_matrix, g[f"{name}_in"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(model.output_matrix, g[f"{name}_out"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(losses, g[f"{name}_losses"], rtol=1e-10)
    assert np.array_equal(model.touched_input, g[f"{name}_touched_in"])
    assert np.array_equal(model.touched_output, g[f"{name}_touched_out"])


# fp32 store, same streams: 1e-4 absolute, loss 1e-5 relative
def test_cbow_replay_fp32_within_tolerance(golden, wv):
    g = golden("cbow.npz")
    kw = json.loads(str(g["sparse_cfg"]))
    corpus = wv.WalkCorpus(g["train_tokens"], g["train_offsets"])
    model, losses = wv.train(corpus, int(g["train_V"]), wv.TrainConfig(**kw), 42, precision="fp32", pairs="numpy")
    np.testing.assert_allclose(model.input_matrix, g["sparse_in"], rtol=0, atol=1e-4)
    np.testing.assert_allclose(model.output_matrix, g["sparse_out"], rtol=0, atol=1e-4)
    np.testing.assert_allclose(losses, g["sparse_losses"], rtol=1e-5)


def test_cbow_device_mode_deterministic_and_learns(golden, wv):
    g = golden("cbow.npz")
    corpus = wv.WalkCorpus(g["train_tokens"], g["train_offsets"])
    cfg = wv.TrainConfig(model="cbow", min_count=1, vector_size=16, epochs=4, window_size=3, batch_size=50)
    a, la = wv.train(corpus, int(g["train_V"]), cfg, 3)
    b, lb = wv.train(corpus, int(g["train_V"]), cfg, 3)
    assert np.array_equal(a.input_matrix, b.input_matrix) and la == lb
    assert la[-1] < la[0]


def test_large_batch_replay_matches_oracle(wv):
    """Batches beyond the shared-memory slot bitmap (> 393,216 items): heavy rows take the
    CTA radix-sort path; fp64 replay of the reference streams still matches the oracle."""
    from paper_2508_01073_b200.synth import synthetic_kg

    edges, V, ents, _ = synthetic_kg("barabasi", 4000, m=4, predicates=12, seed=5)
    graph = wv.build_graph(edges, V)
    corpus = wv.random_walks(graph, ents, walk_depth=4, walk_number=20, rng_seed=3)
    cfg = wv.TrainConfig(min_count=1, vector_size=8, epochs=1, window_size=3, negative_samples=5,
                         batch_size=70_000)
    model, losses = wv.train(corpus, V, cfg, 42, precision="fp64", pairs="numpy")
    ref = ov.train(corpus.tokens, corpus.offsets, V, 8, 3, 5, 0.01, 1, 1, 42, batch=70_000)
    assert 70_000 * 7 > 393_216
    np.testing.assert_allclose(model.input_matrix, ref["inp"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(model.output_matrix, ref["out"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(losses, ref["losses"], rtol=1e-10)


def _two_clique_margin(wv, ref, v):
    def cos(a, b):
        return float(np.dot(v[a], v[b]) / (np.linalg.norm(v[a]) * np.linalg.norm(v[b])))

    x, y = ref["x"], ref["y"]
    intra = [cos(a, b) for grp in (x, y) for a in grp for b in grp if a < b]
    inter = [cos(a, b) for a in x for b in y]
    return np.mean(intra) - np.mean(inter)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_two_clique_d200_device_streams_within_reference_band(wv, precision):
    """The downstream check at the benchmark's width (d 200, reference band from 10 reference
    runs in tests/golden/two_clique.json runs_d200): device streams, both stores."""
    ref = json.loads((GOLDEN / "two_clique.json").read_text())
    margins = np.array([r["margin"] for r in ref["runs_d200"]])
    finals = np.array([r["loss_last"] for r in ref["runs_d200"]])
    graph = wv.build_graph(np.array(ref["edges"]), ref["V"])
    got_m, got_l = [], []
    for r in ref["runs_d200"][:5]:
        corpus = wv.random_walks(graph, ref["roots"], walk_depth=4, walk_number=25, rng_seed=r["seed"])
        cfg = wv.TrainConfig(min_count=1, vector_size=200, epochs=10, learning_rate=0.01, window_size=5,
                             negative_samples=5)
        model, losses = wv.train(corpus, ref["V"], cfg, r["seed"], precision=precision)
        got_m.append(_two_clique_margin(wv, ref, model.input_matrix))
        got_l.append(losses[-1])
    assert abs(np.mean(got_m) - margins.mean()) < 4 * margins.std() + 1e-3, (np.mean(got_m), margins.mean())
    assert abs(np.mean(got_l) - finals.mean()) < 4 * finals.std() + 1e-3, (np.mean(got_l), finals.mean())


@pytest.mark.parametrize("blocks", ["strided", "whole"])
def test_blockwise_session_within_reference_band(wv, blocks):
    """SkipGramSession (the benchmark's trainer) streaming the corpus in root blocks -- a fresh
    permutation per block, the session's resident parameters and RowAdam state -- against the
    reference's downstream band at equal epochs (each epoch visits every block once; the batch
    size is the reference's whole-corpus rule value).  Blocks must sample the roots (strided):
    contiguous root ranges of a graph whose clusters follow the token order train one cluster at
    a time and measured a margin of 0.29 against the band's 0.59 +- 0.04."""
    ref = json.loads((GOLDEN / "two_clique.json").read_text())
    margins = np.array([r["margin"] for r in ref["runs"]])
    graph = wv.build_graph(np.array(ref["edges"]), ref["V"])
    got = []
    for r in ref["runs"][:5]:
        roots = np.array(ref["roots"])
        full = wv.random_walks(graph, roots, walk_depth=4, walk_number=25, rng_seed=r["seed"])
        n_pairs = len(wv.generate_pairs(full, 5, 1, ref["V"])[0])
        B = wv.suggest_batch_size(wv.estimate_per_sample_bytes("skipgram", 16, 5, 5), 1 << 30, n_pairs)
        parts = [roots[i::3] for i in range(3)] if blocks == "strided" else [roots]
        blks = [wv.random_walks(graph, part, walk_depth=4, walk_number=25, rng_seed=r["seed"]) for part in parts]
        cfg = wv.TrainConfig(min_count=1, vector_size=16, epochs=1, learning_rate=0.01, window_size=5,
                             negative_samples=5, batch_size=B)
        sess = wv.SkipGramSession(ref["V"], cfg, r["seed"], precision="fp64")
        for _ in range(10):
            for blk in blks:
                sess.fit(blk, 1)
        got.append(_two_clique_margin(wv, ref, sess.model.input_matrix))
    assert abs(np.mean(got) - margins.mean()) < 4 * margins.std() + 1e-3, (np.mean(got), margins.mean())
