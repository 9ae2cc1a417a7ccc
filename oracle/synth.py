"""Synthetic-KG oracle -- TEST INFRASTRUCTURE ONLY (and the reference arm's input).

A numpy restatement of the device Barabasi-Albert generator
(paper_2508_01073_b200/csrc/synth.cu: ba_resolve, ba_chase, ba_dups,
wv_gen_barabasi) and of first-occurrence token encoding
(reference ingest.py:368-396 over benchgen.assign_predicates, :152-161).

The process is the reference's gen_barabasi (benchgen.py:78-109): vertex
v >= 1 draws min(m, v) distinct targets from the attachment bag, the list
[0] followed, per vertex u, by the block [t1, u, t2, u, ..., tk, u, u]; all of
v's draws see the bag as it was before v's block.  The device draws bag
positions from counter-based Philox4x32-10 (key = seed, counter = (edge,
attempt, tag)), so the graph is a pure function of (n, m, seed); this file
computes the same function with vectorised numpy -- the bit-exact parity
check of csrc/synth.cu (tests/test_gpu_synth.py) and a way for bench.py's
reference arm to build the cfg2 input without loading the product library.
"""

from __future__ import annotations

import numpy as np

MASK32 = np.uint64(0xFFFFFFFF)
_PH_M0, _PH_M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
BA_TAG = 0x42415247  # "BARG": the counter's fourth word in ba_draw


def philox4x32_10(c0, c1, c2, c3, k0: int, k1: int):
    """Philox4x32-10 on uint64 arrays holding 32-bit words (Salmon et al. 2011; common.cuh philox4x32_10)."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint64) & MASK32 for x in (c0, c1, c2, c3))
    for _ in range(10):
        p0 = _PH_M0 * c0
        p1 = _PH_M1 * c2
        n0 = (p1 >> np.uint64(32)) ^ c1 ^ np.uint64(k0)
        n2 = (p0 >> np.uint64(32)) ^ c3 ^ np.uint64(k1)
        c0, c1, c2, c3 = n0, p1 & MASK32, n2, p0 & MASK32
        k0 = (k0 + 0x9E3779B9) & 0xFFFFFFFF
        k1 = (k1 + 0xBB67AE85) & 0xFFFFFFFF
    return c0, c1, c2, c3


def mulhi64(a, b):
    """High 64 bits of the 128-bit product of uint64 arrays (schoolbook on 32-bit halves)."""
    a = np.asarray(a, dtype=np.uint64)
    b = np.asarray(b, dtype=np.uint64)
    s32 = np.uint64(32)
    ah, al = a >> s32, a & MASK32
    bh, bl = b >> s32, b & MASK32
    ll = al * bl
    lh = al * bh
    hl = ah * bl
    mid = (ll >> s32) + (lh & MASK32) + (hl & MASK32)
    return ah * bh + (lh >> s32) + (hl >> s32) + (mid >> s32)


def ba_edge_count(n: int, m: int) -> int:
    return int(sum(min(m, v) for v in range(1, min(n, m + 1))) + max(0, n - m - 1) * m)


class _Shape:
    def __init__(self, n, m):
        self.n, self.m = int(n), int(m)
        self.small_edges = self.m * (self.m + 1) // 2
        self.small_bag = (self.m + 1) ** 2

    def k(self, v):
        return np.minimum(v, self.m)

    def edge_base(self, v):
        v = np.asarray(v, dtype=np.int64)
        return np.where(v <= self.m + 1, (v - 1) * v // 2, self.small_edges + (v - 1 - self.m) * self.m)

    def bag_base(self, v):
        v = np.asarray(v, dtype=np.int64)
        return np.where(v <= self.m + 1, v * v, self.small_bag + (v - self.m - 1) * (2 * self.m + 1))

    def block_of(self, q):
        q = np.asarray(q, dtype=np.int64)
        u = np.floor(np.sqrt(q.astype(np.float64))).astype(np.int64)
        u -= (u * u > q)
        u += ((u + 1) * (u + 1) <= q)
        big = self.m + 1 + (q - self.small_bag) // (2 * self.m + 1)
        return np.where(q < self.small_bag, u, big)


def barabasi_edges(n: int, m: int, seed: int):
    """(src, dst) int64 arrays equal to wv_gen_barabasi(n, m, seed)'s output."""
    if n < 2 or m < 1:
        raise ValueError("n must be >= 2 and m >= 1")
    s = _Shape(n, m)
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    v = np.arange(1, n, dtype=np.int64)
    kv = s.k(v)
    src = np.repeat(v, kv)
    E = len(src)
    L = s.bag_base(src)  # v's draws use bag positions [0, bag_base(v))
    attempt = np.zeros(E, dtype=np.uint64)
    ptr = np.empty(E, dtype=np.int64)
    val = np.empty(E, dtype=np.int64)
    e_all = np.arange(E, dtype=np.uint64)
    todo = np.arange(E, dtype=np.int64)
    for _ in range(4096):
        # ba_resolve for the edges whose attempt changed (the rest draw what they drew before)
        e = e_all[todo]
        c0, c1, _, _ = philox4x32_10(e & MASK32, e >> np.uint64(32), attempt[todo], np.full(len(todo), BA_TAG,
                                                                                           np.uint64),
                                     seed & 0xFFFFFFFF, seed >> 32)
        r = (c1 << np.uint64(32)) | c0
        q = mulhi64(r, L[todo].astype(np.uint64)).astype(np.int64)
        u = s.block_of(q)
        off = q - s.bag_base(u)
        uu = np.maximum(u, 1)
        is_t = (u > 0) & (off < 2 * s.k(uu)) & (off % 2 == 0)
        ptr[todo] = np.where(is_t, s.edge_base(uu) + off // 2, -1)
        val[todo] = np.where(is_t, -1, u)
        # ba_chase: pointers strictly decrease, follow them to a value
        x = np.arange(E, dtype=np.int64)
        act = np.flatnonzero(ptr >= 0)
        x_act = ptr[act]
        while act.size:
            more = ptr[x_act] >= 0
            x[act[~more]] = x_act[~more]
            act, x_act = act[more], ptr[x_act[more]]
        dst = val[x]
        # ba_dups: a later slot equal to an earlier slot of the same vertex is redrawn
        dup = np.zeros(E, dtype=bool)
        for vv in range(1, min(n, m + 1)):  # vertices with fewer than m edges
            b = (vv - 1) * vv // 2
            for j in range(1, vv):
                dup[b + j] = bool((dst[b:b + j] == dst[b + j]).any())
        if n > m + 1:
            blk = dst[s.small_edges:].reshape(-1, m)
            dblk = dup[s.small_edges:].reshape(-1, m)
            for j in range(1, m):
                dblk[:, j] = (blk[:, :j] == blk[:, j:j + 1]).any(axis=1)
        if not dup.any():
            return src, dst
        todo = np.flatnonzero(dup)
        attempt[todo] += np.uint64(1)
    raise RuntimeError("barabasi generator did not converge")


def predicate_picks(n_edges: int, predicate_set_size: int, seed: int) -> np.ndarray:
    """benchgen.assign_predicates' stream (benchgen.py:152-161): SeedSequence([seed, 3]).integers."""
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), 3]))
    return rng.integers(0, predicate_set_size, size=n_edges)


def encode(src, picks, dst, n_entities: int):
    """build_vocabulary over the flattened (s, p, o) stream (ingest.py:368-396): token = rank of the
    key's first occurrence; entity keys are vertices, predicate keys n_entities + pick.
    -> (edges (E,3) int64, vocab size, sorted entity tokens, sorted predicate tokens)."""
    keys = np.stack([src, n_entities + np.asarray(picks, dtype=np.int64), dst], axis=1).ravel()
    uniq, first = np.unique(keys, return_index=True)
    order = np.argsort(first, kind="stable")
    token_of_uniq = np.empty(len(uniq), dtype=np.int64)
    token_of_uniq[order] = np.arange(len(uniq))
    edges = token_of_uniq[np.searchsorted(uniq, keys)].reshape(-1, 3)
    ent = np.sort(token_of_uniq[uniq < n_entities])
    prd = np.sort(token_of_uniq[uniq >= n_entities])
    return edges, len(uniq), ent, prd


def barabasi_kg(n: int, m: int, predicates: int, seed: int):
    """device_synthetic_kg("barabasi", n, m, predicates, seed) restated: (edges, V, entity tokens, predicate tokens)."""
    src, dst = barabasi_edges(n, m, seed)
    return encode(src, predicate_picks(len(src), predicates, seed), dst, n)
