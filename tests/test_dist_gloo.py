"""Multi-process host logic of the multi-GPU path, on CPU with gloo (world_size 2).

SURVEY §8e: walks shard by contiguous entity (root) ranges with no
communication; SGNS replicas exchange per-row deltas and touch counts with one
all-reduce(sum) per sync round and apply shared += sum / count
(_merge_bundles, /root/reference/pkg/src/walkvec/w2v.py:642-659).  The device
kernels are covered by the -m gpu tests; here the rank arithmetic and the
exchange semantics run for real over torch.distributed (gloo).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_01073_b200.dist import RankExchange, rank_slice, walk_work_range


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, fn, *args):
    port = _free_port()
    mp.spawn(_entry, args=(world, port, fn, args), nprocs=world, join=True)


def _entry(rank, world, port, fn, args):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_roots,walk_number,world", [(10, 3, 2), (7, 100, 4), (1, 5, 3), (10_000, 10, 8)])
def test_walk_ranges_partition_root_major_work(n_roots, walk_number, world):
    """Union of the rank ranges = repeat(roots, walk_number) (walks.py:166), whole root groups per rank."""
    got = []
    for r in range(world):
        b, e = walk_work_range(n_roots, walk_number, r, world)
        assert b % walk_number == 0 and e % walk_number == 0  # duplicate_free needs whole groups
        got.append((b, e))
    assert got[0][0] == 0 and got[-1][1] == n_roots * walk_number
    for (b0, e0), (b1, e1) in zip(got, got[1:]):
        assert e0 == b1 and b0 <= e0


def test_rank_slice_granule():
    spans = [rank_slice(100_003, r, 4, granule=8192) for r in range(4)]
    assert spans[0][0] == 0 and spans[-1][1] == 100_003
    assert all(s[1] % 8192 == 0 for s in spans[:-1] if s[1] < 100_003)


def _exchange_worker(rank, world):
    ex = RankExchange()
    assert ex.rank == rank and ex.world_size == world
    V, d = 6, 3
    rng = np.random.default_rng(rank)
    snap = np.arange(V * d, dtype=np.float64).reshape(V, d) / 10  # identical round-start values on all ranks
    touched = np.zeros(V, dtype=bool)
    touched[[rank, 3]] = True  # rank r touches row r and the shared row 3
    params = snap.copy()
    params[touched] += rng.normal(size=(touched.sum(), d))
    delta = torch.from_numpy(params - snap)
    cnt = torch.from_numpy(touched.astype(np.float32))
    ex.all_reduce_(delta, cnt)
    merged = snap.copy()
    hit = cnt.numpy() > 0
    merged[hit] = snap[hit] + delta.numpy()[hit] / cnt.numpy()[hit, None]
    # reference semantics: mean over the workers that touched the row of their deltas
    all_params = []
    for r in range(world):
        rr = np.random.default_rng(r)
        t = np.zeros(V, dtype=bool)
        t[[r, 3]] = True
        p = snap.copy()
        p[t] += rr.normal(size=(t.sum(), d))
        all_params.append((p, t))
    expect = snap.copy()
    for row in range(V):
        ds = [p[row] - snap[row] for p, t in all_params if t[row]]
        if ds:
            expect[row] = snap[row] + np.mean(ds, axis=0)
    np.testing.assert_allclose(merged, expect, rtol=0, atol=1e-12)
    # epoch loss reduction and first divergence over ranks
    loss, count, div = ex.reduce_epoch(1.5 * (rank + 1), 10 * (rank + 1), (2, 7) if rank == 1 else None)
    assert count == sum(10 * (r + 1) for r in range(world))
    assert abs(loss - sum(1.5 * (r + 1) for r in range(world))) < 1e-12
    assert div == ((2, 7) if world > 1 else None)
    flags = torch.zeros(V, dtype=torch.uint8)
    flags[rank] = 1
    ex.or_flags_(flags)
    assert flags.tolist() == [1 if r < world else 0 for r in range(V)]


def test_replica_exchange_matches_reference_merge():
    _run(2, _exchange_worker)


def _merge_worker(rank, world, V, d, frac_rows):
    """merge_deltas_: the sparse (touched rows only) and dense paths give the reference merge."""
    ex = RankExchange()
    results = {}
    for mode, frac in (("sparse", 0.99), ("dense", 1e-9)):
        rng = np.random.default_rng(100 + rank)
        touched = np.zeros(V, dtype=bool)
        touched[rng.choice(V, int(frac_rows * V), replace=False)] = True
        touched[0] = True  # a row every rank touches
        delta = np.zeros((V, d))
        delta[touched] = rng.normal(size=(touched.sum(), d))
        dl = torch.from_numpy(delta.ravel().copy())
        cnt = torch.from_numpy(touched.astype(np.float32))
        got = ex.merge_deltas_((dl,), (cnt,), d, sparse_fraction=frac)
        assert got == mode, (got, mode)  # one matrix: one path
        results[mode] = (dl.numpy().reshape(V, d).copy(), cnt.numpy().copy())
        # expected: sum over ranks of their deltas, counts summed
        exp_d = np.zeros((V, d))
        exp_c = np.zeros(V, dtype=np.float32)
        for r in range(world):
            rr = np.random.default_rng(100 + r)
            t = np.zeros(V, dtype=bool)
            t[rr.choice(V, int(frac_rows * V), replace=False)] = True
            t[0] = True
            dd = np.zeros((V, d))
            dd[t] = rr.normal(size=(t.sum(), d))
            exp_d = exp_d + dd
            exp_c += t
        np.testing.assert_allclose(results[mode][0], exp_d, rtol=0, atol=1e-12)
        assert np.array_equal(results[mode][1], exp_c)
    if world == 2:  # two addends: both paths are exact and identical
        assert np.array_equal(results["sparse"][0], results["dense"][0])


@pytest.mark.parametrize("world", [2, 3])
def test_sparse_touched_row_merge(world):
    _run(world, _merge_worker, 50, 4, 0.1)
