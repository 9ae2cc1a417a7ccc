"""Multi-rank SGNS on the device: two ranks (processes on one GPU, gloo with host
staging) against in-process references.

* ``train(exchange=RankExchange())`` -- each rank trains its worker span as a
  local replica and the ranks merge per-row deltas every sync round -- equals
  the in-process ``train(workers=2)`` (the reference's _train_multi contract,
  w2v.py:579-746) bit for bit: with two ranks the cross-rank sums have two
  addends, so the order cannot matter.
* ``SkipGramSession.sync`` after each rank fits a different corpus equals the
  reference merge (_merge_bundles, w2v.py:642-659) recomputed in numpy from
  the ranks' pre-sync parameters, and leaves both ranks identical; the merge
  goes through the sparse touched-row path or the dense all-reduce as asked.
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _corpus(wv, seed):
    from paper_2508_01073_b200.synth import synthetic_kg

    edges, V, ents, _ = synthetic_kg("barabasi", 6000, m=4, predicates=10, seed=3)
    graph = wv.build_graph(edges, V)
    return wv.random_walks(graph, ents[::4], walk_depth=4, walk_number=3, rng_seed=seed), V


CFG = dict(min_count=1, vector_size=24, epochs=2, window_size=3, negative_samples=4, batch_size=256, workers=2,
           reproducible=True)


def _worker(rank, world, port, out_dir, sparse_fraction):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    import paper_2508_01073_b200 as wv
    from paper_2508_01073_b200.dist import RankExchange

    corpus, V = _corpus(wv, 11)
    for precision in ("fp64", "fp32"):
        model, losses = wv.train(corpus, V, wv.TrainConfig(**CFG), 42, precision=precision,
                                 exchange=RankExchange())
        np.savez(os.path.join(out_dir, f"train_{precision}_rank{rank}.npz"), inp=model.input_matrix,
                 out=model.output_matrix, losses=np.array(losses))
    # SkipGramSession: different corpora per rank, then one merge
    cfg = wv.TrainConfig(min_count=0, vector_size=16, epochs=1, window_size=3, negative_samples=3, batch_size=128)
    sess = wv.SkipGramSession(V, cfg, 5, precision="fp64")
    ex = RankExchange()
    sess.attach_exchange(ex)
    orig = ex.merge_deltas_
    ex.merge_deltas_ = lambda d, c, dim: orig(d, c, dim, sparse_fraction=sparse_fraction)
    small = wv.WalkCorpus(*_first_walks(_corpus(wv, 20 + rank)[0], 8 if rank == 0 else 12))
    snap_in = sess.params.inp.double().cpu().numpy().copy()
    snap_out = sess.params.out.double().cpu().numpy().copy()
    sess.fit(small, 1)
    pre_in = sess.params.inp.cpu().numpy().copy()
    pre_out = sess.params.out.cpu().numpy().copy()
    t_in = sess._round_in.cpu().numpy().copy()
    t_out = sess._round_out.cpu().numpy().copy()
    sess.sync()
    np.savez(os.path.join(out_dir, f"sess_rank{rank}.npz"), snap_in=snap_in, snap_out=snap_out, pre_in=pre_in,
             pre_out=pre_out, t_in=t_in, t_out=t_out, post_in=sess.params.inp.cpu().numpy(),
             post_out=sess.params.out.cpu().numpy(), merge=np.array(sess.last_merge))
    dist.barrier()
    dist.destroy_process_group()


def _first_walks(corpus, n):
    off = corpus.offsets[: n + 1]
    return corpus.tokens[: off[-1]], off


@pytest.mark.parametrize("sparse_fraction,expect", [(0.99, "sparse,sparse"), (1e-9, "dense,dense")])
def test_two_rank_training_and_session_merge(tmp_path, sparse_fraction, expect):
    import torch.multiprocessing as mp

    import paper_2508_01073_b200 as wv

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), sparse_fraction), nprocs=world,
                       join=True, start_method="spawn")
    corpus, V = _corpus(wv, 11)
    for precision in ("fp64", "fp32"):
        model, losses = wv.train(corpus, V, wv.TrainConfig(**CFG), 42, precision=precision)
        for r in range(world):
            got = np.load(tmp_path / f"train_{precision}_rank{r}.npz")
            assert np.array_equal(got["inp"], model.input_matrix), (precision, r)
            assert np.array_equal(got["out"], model.output_matrix), (precision, r)
            np.testing.assert_allclose(got["losses"], losses, rtol=1e-12)
    a, b = (np.load(tmp_path / f"sess_rank{r}.npz") for r in range(world))
    assert str(a["merge"]) == expect and str(b["merge"]) == expect
    for side in ("in", "out"):
        snap = a[f"snap_{side}"].ravel()
        d = snap.size // V
        # the reference merge: shared += mean over the ranks that touched the row of their deltas
        deltas = [x[f"pre_{side}"] - snap for x in (a, b)]
        cnt = a[f"t_{side}"].astype(np.float32) + b[f"t_{side}"].astype(np.float32)
        expect_p = snap.copy().reshape(V, d)
        dsum = (deltas[0] + deltas[1]).reshape(V, d)
        hit = cnt > 0
        expect_p[hit] = snap.reshape(V, d)[hit] + dsum[hit] / cnt[hit, None]
        for x in (a, b):
            assert np.array_equal(x[f"post_{side}"].reshape(V, d), expect_p), side


def _bfs_worker(rank, world, port, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    import paper_2508_01073_b200 as wv
    from paper_2508_01073_b200.dist import bfs_walks_rank
    from paper_2508_01073_b200.synth import synthetic_kg

    edges, V, ents, _ = synthetic_kg("barabasi", 3000, m=4, predicates=8, seed=9)
    graph = wv.build_graph(edges, V)
    corpus, table, base = bfs_walks_rank(graph, ents[::7], 3, max_walks_per_root=40)
    np.savez(os.path.join(out_dir, f"bfs_rank{rank}.npz"), tokens=corpus.tokens, offsets=corpus.offsets,
             src=table.sources, dst=table.targets, wid=table.walk_ids, base=np.array(base))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_bfs_root_ranges_with_global_walk_ids(tmp_path, world):
    """Rank-sharded BFS (root ranges, walk ids by an exclusive scan of the ranks' counts)
    concatenates to the single-process bfs_walks corpus and PathTable."""
    import torch.multiprocessing as mp

    import paper_2508_01073_b200 as wv
    from paper_2508_01073_b200.synth import synthetic_kg

    mp.start_processes(_bfs_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    edges, V, ents, _ = synthetic_kg("barabasi", 3000, m=4, predicates=8, seed=9)
    graph = wv.build_graph(edges, V)
    corpus, table = wv.bfs_walks(graph, ents[::7], 3, max_walks_per_root=40)
    parts = [np.load(tmp_path / f"bfs_rank{r}.npz") for r in range(world)]
    toks = np.concatenate([p["tokens"] for p in parts])
    offs = [np.zeros(1, dtype=np.int64)]
    for p in parts:
        offs.append(p["offsets"][1:] + offs[-1][-1])
    assert np.array_equal(toks, corpus.tokens) and np.array_equal(np.concatenate(offs), corpus.offsets)
    assert np.array_equal(np.concatenate([p["src"] for p in parts]), table.sources)
    assert np.array_equal(np.concatenate([p["dst"] for p in parts]), table.targets)
    assert np.array_equal(np.concatenate([p["wid"] for p in parts]), table.walk_ids)
    assert [int(p["base"]) for p in parts] == [int(sum(len(q["offsets"]) - 1 for q in parts[:r])) for r in
                                               range(world)]
