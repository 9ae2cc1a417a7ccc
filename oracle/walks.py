"""Walk-corpus oracle -- TEST INFRASTRUCTURE ONLY.

Restates /root/reference/pkg/src/walkvec/graph.py:74-98 (stable CSR) and
walks.py (random_walks :144-204 with _walk_shard :117-141, duplicate_free
:186-202, _bfs_tree/bfs_walks :207-310, project_corpus :323-341) in numpy.
The random-walk oracle draws from the *same* numpy generators the
reference uses: PCG64 (default_rng) or Philox, per 8192-walk shard.
"""

from __future__ import annotations

import numpy as np

SHARD = 8192


def csr(edges: np.ndarray, vertex_count: int):
    """graph.py:74-98 -> (row_offsets, col_targets, col_predicates), stable by source."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 3)
    perm = np.argsort(e[:, 0], kind="stable")
    off = np.zeros(vertex_count + 1, dtype=np.int64)
    np.cumsum(np.bincount(e[:, 0], minlength=vertex_count), out=off[1:])
    return off, e[perm, 2].copy(), e[perm, 1].copy()


def _shard_rng(seed: int, shard: int, kind: str) -> np.random.Generator:
    ss = np.random.SeedSequence([int(seed), 0, int(shard)])
    if kind == "pcg64":
        return np.random.default_rng(ss)
    if kind == "philox":
        return np.random.Generator(np.random.Philox(ss))
    raise ValueError(kind)


def walk_rows(off, tgt, prd, starts: np.ndarray, depth: int, rng: np.random.Generator):
    """One shard, hop-synchronous (walks.py:117-141): -1 padded rows [n, 2*depth+1]."""
    n = len(starts)
    rows = np.full((n, 2 * depth + 1), -1, dtype=np.int64)
    rows[:, 0] = starts
    at = starts.astype(np.int64).copy()
    live = np.ones(n, dtype=bool)
    for h in range(depth):
        lo, hi = off[at], off[at + 1]
        deg = hi - lo
        live &= deg > 0
        if not live.any():
            break
        u = rng.random(n)  # consumed for every row, dead or alive
        pick = np.minimum((u * deg).astype(np.int64), np.maximum(deg - 1, 0))
        e = (lo + pick)[live]
        rows[live, 2 * h + 1] = prd[e]
        rows[live, 2 * h + 2] = tgt[e]
        at[live] = tgt[e]
    return rows


def random_walks(off, tgt, prd, roots, depth: int, number: int, seed: int, kind: str = "pcg64",
                 duplicate_free: bool = False, shards=None):
    """(tokens, offsets) exactly as walks.random_walks; ``shards`` restricts to a subset."""
    roots = np.asarray(roots, dtype=np.int64)
    work = np.repeat(roots, number)
    n_sh = -(-len(work) // SHARD)
    pieces, lens = [], []
    for s in (range(n_sh) if shards is None else shards):
        rows = walk_rows(off, tgt, prd, work[s * SHARD:(s + 1) * SHARD], depth, _shard_rng(seed, s, kind))
        keep = rows != -1
        pieces.append(rows[keep])
        lens.append(keep.sum(axis=1))
    tokens = np.concatenate(pieces) if pieces else np.empty(0, dtype=np.int64)
    lengths = np.concatenate(lens).astype(np.int64) if lens else np.empty(0, dtype=np.int64)
    offsets = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    if duplicate_free:
        keep_walk = np.zeros(len(lengths), dtype=bool)
        for g0 in range(0, len(lengths), number):
            seen = set()
            for i in range(g0, min(g0 + number, len(lengths))):
                key = tokens[offsets[i]:offsets[i + 1]].tobytes()
                if key not in seen:
                    seen.add(key)
                    keep_walk[i] = True
        seqs = [tokens[offsets[i]:offsets[i + 1]] for i in np.flatnonzero(keep_walk)]
        lengths = np.array([len(s) for s in seqs], dtype=np.int64)
        tokens = np.concatenate(seqs) if seqs else np.empty(0, dtype=np.int64)
        offsets = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    return tokens, offsets


def bfs_walks(off, tgt, prd, roots, depth: int, cap: int | None = None):
    """walks.py:207-310 (sequential restatement) -> (tokens, offsets, path rows (src,dst,wid))."""
    seqs, rows = [], []
    for root in np.asarray(roots, dtype=np.int64).tolist():
        parent, ppred, order = {root: -1}, {root: -1}, [root]
        frontier = [root]
        for _ in range(depth):
            nxt = []
            for u in frontier:
                for e in range(off[u], off[u + 1]):
                    v = int(tgt[e])
                    if v not in parent:
                        parent[v], ppred[v] = u, int(prd[e])
                        order.append(v)
                        nxt.append(v)
            if not nxt:
                break
            frontier = nxt
        parents = set(parent.values())
        leaves = [v for v in order if v not in parents] or [root]
        if cap:
            leaves = leaves[:cap]
        for leaf in leaves:
            chain, v = [], leaf
            while v != root:
                chain.append(v)
                rows.append((parent[v], v, len(seqs)))
                v = parent[v]
            chain.append(root)
            chain.reverse()
            tok = [chain[0]]
            for v in chain[1:]:
                tok += [ppred[v], v]
            seqs.append(tok)
    lengths = np.array([len(s) for s in seqs], dtype=np.int64)
    tokens = np.array([t for s in seqs for t in s], dtype=np.int64)
    offsets = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    return tokens, offsets, rows


def project(tokens, offsets, projection: str):
    """walks.py:323-341."""
    pos = np.arange(len(tokens)) - np.repeat(offsets[:-1], np.diff(offsets))
    keep = (pos % 2 == 0) if projection == "entity" else ((pos == 0) | (pos % 2 == 1))
    walk = np.repeat(np.arange(len(offsets) - 1), np.diff(offsets))
    counts = np.bincount(walk[keep], minlength=len(offsets) - 1)
    return tokens[keep], np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
