"""SGNS oracle -- TEST INFRASTRUCTURE ONLY.

Restates /root/reference/pkg/src/walkvec/w2v.py in float64 numpy:
init (:123-131), min_count filter + shift-major pairs (:146-191), negatives
(:225-239, 500-504), SGNS loss/gradients (:247-299), coalescing (:407-416),
RowAdam (:364-404), batch sizing (:437-497), _train_single (:547-576) and
the reproducible multi-worker contract (:579-746).  Implementation choices
differ from the reference on purpose (matmul dots, sort + reduceat
coalescing) so agreement is evidence, not a copy.
"""

from __future__ import annotations

import numpy as np

B1, B2, EPS = 0.9, 0.999, 1e-8


def init(V: int, d: int, seed: int):
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), 1, 0]))
    b = 1.0 / d
    return rng.uniform(-b, b, size=(V, d)), rng.uniform(-b, b, size=(V, d))


def frequencies(tokens, V):
    return np.bincount(np.asarray(tokens, dtype=np.int64), minlength=V).astype(np.int64)


def filtered(tokens, offsets, keep):
    tok_keep = keep[tokens]
    walk = np.repeat(np.arange(len(offsets) - 1), np.diff(offsets))
    counts = np.bincount(walk[tok_keep], minlength=len(offsets) - 1)
    return tokens[tok_keep], np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)


def pairs(tokens, offsets, window: int):
    """shift-major (t[i], t[i+s]) block then (t[i+s], t[i]) block per shift."""
    walk = np.repeat(np.arange(len(offsets) - 1), np.diff(offsets))
    c, x = [], []
    for s in range(1, window + 1):
        if s >= len(tokens):
            break
        ok = walk[:-s] == walk[s:]
        a, b = tokens[:-s][ok], tokens[s:][ok]
        c += [a, b]
        x += [b, a]
    if not c or sum(len(v) for v in c) == 0:
        raise ValueError("empty training set")
    return np.stack([np.concatenate(c), np.concatenate(x)], axis=1)


def batch_size(N, d, k, budget=1 << 30, explicit=None, cap=0.9):
    per = (2 + k) * d * 8 + 16
    b = explicit if explicit is not None else max(1, min(budget // (4 * per), -(-N // 20)))
    while b > 1 and b * per > cap * budget:
        b //= 2
    return b


def sgns_step(inp, out, c, x, negs):
    """loss + (rows, grads) for both matrices (w2v.py:276-299), batch-mean."""
    B = len(c)
    u, v = inp[c], out[x]
    pos = (u * v).sum(axis=1)
    loss = np.logaddexp(0.0, -pos).sum()
    gpos = (1.0 / (1.0 + np.exp(-pos)) - 1.0) / B
    gu = gpos[:, None] * v
    orow, og = [x], [gpos[:, None] * u]
    if negs.size:
        n = out[negs]                                   # B,k,d
        neg = np.matmul(n, u[:, :, None])[:, :, 0]      # B,k
        loss += np.logaddexp(0.0, neg).sum()
        gneg = (1.0 / (1.0 + np.exp(-neg))) / B
        gu = gu + (gneg[:, :, None] * n).sum(axis=1)
        orow.append(negs.ravel())
        og.append((gneg[:, :, None] * u[:, None, :]).reshape(-1, inp.shape[1]))
    return loss / B, c, gu, np.concatenate(orow), np.vstack(og)


def coalesce(rows, grads):
    order = np.argsort(rows, kind="stable")
    r, g = rows[order], grads[order]
    heads = np.flatnonzero(np.concatenate([[True], r[1:] != r[:-1]]))
    return r[heads], np.add.reduceat(g, heads, axis=0)


class RowAdam:
    def __init__(self, shape, lr, sparse=True):
        self.lr, self.sparse = lr, sparse
        self.m, self.v = np.zeros(shape), np.zeros(shape)
        self.t = np.zeros(shape[0], dtype=np.int64)
        self.step = 0

    def update(self, P, rows, g):
        if self.sparse:
            self.t[rows] += 1
            t = self.t[rows].astype(np.float64)[:, None]
            self.m[rows] = B1 * self.m[rows] + (1 - B1) * g
            self.v[rows] = B2 * self.v[rows] + (1 - B2) * g * g
            P[rows] -= self.lr * (self.m[rows] / (1 - B1 ** t)) / (np.sqrt(self.v[rows] / (1 - B2 ** t)) + EPS)
        else:
            self.step += 1
            full = np.zeros_like(P)
            full[rows] = g
            self.m = B1 * self.m + (1 - B1) * full
            self.v = B2 * self.v + (1 - B2) * full * full
            P -= self.lr * (self.m / (1 - B1 ** self.step)) / (np.sqrt(self.v / (1 - B2 ** self.step)) + EPS)


def train(tokens, offsets, V, d, window, k, lr, min_count, epochs, seed, batch=None, budget=1 << 30,
          sparse=True, max_batches=None):
    """Single-worker SGNS (w2v.py:507-576) -> dict(inp, out, losses, touched_in, touched_out, keep)."""
    tokens = np.asarray(tokens, dtype=np.int64)
    offsets = np.asarray(offsets, dtype=np.int64)
    freq = frequencies(tokens, V)
    keep = freq >= min_count
    ft, fo = filtered(tokens, offsets, keep)
    if len(ft) == 0:
        raise ValueError("empty training set")
    pr = pairs(ft, fo, window)
    cand = np.flatnonzero(keep)
    inp, out = init(V, d, seed)
    B = batch_size(len(pr), d, k, budget, batch)
    sh = np.random.default_rng(np.random.SeedSequence([int(seed), 1, 1]))
    ng = np.random.default_rng(np.random.SeedSequence([int(seed), 1, 2, 0]))
    oi, oo = RowAdam(inp.shape, lr, sparse), RowAdam(out.shape, lr, sparse)
    ti, to = np.zeros(V, bool), np.zeros(V, bool)
    losses, nb = [], 0
    for epoch in range(epochs):
        order = sh.permutation(len(pr))
        tot, cnt = 0.0, 0
        for lo in range(0, len(pr), B):
            idx = order[lo:lo + B]
            negs = cand[ng.integers(0, len(cand), size=len(idx) * k)].reshape(len(idx), k) if k else \
                np.empty((len(idx), 0), dtype=np.int64)
            loss, ir, ig, orr, og = sgns_step(inp, out, pr[idx, 0], pr[idx, 1], negs)
            if not np.isfinite(loss):
                raise FloatingPointError(f"divergence at epoch {epoch}, batch {lo // B}")
            ur, ug = coalesce(ir, ig)
            oi.update(inp, ur, ug)
            ti[ur] = True
            ur, ug = coalesce(orr, og)
            oo.update(out, ur, ug)
            to[ur] = True
            tot += loss * len(idx)
            cnt += len(idx)
            nb += 1
            if max_batches is not None and nb >= max_batches:
                return dict(inp=inp, out=out, losses=losses + [tot / cnt], touched_in=ti, touched_out=to,
                            keep=keep, batch=B, pairs=pr)
        losses.append(tot / cnt)
    return dict(inp=inp, out=out, losses=losses, touched_in=ti, touched_out=to, keep=keep, batch=B, pairs=pr)


def scalar_loss(inp, out, c, x, negs):
    """Pure-scalar batch loss (the reference oracle's form, tests/oracles.py:168-199)."""
    import math

    def bce(z, y):
        if y == 1:
            return math.log1p(math.exp(-z)) if z > 0 else -z + math.log1p(math.exp(z))
        return math.log1p(math.exp(z)) if z < 0 else z + math.log1p(math.exp(-z))

    tot = 0.0
    for ci, xi, ns in zip(c, x, negs):
        u = inp[ci]
        tot += bce(float(sum(a * b for a, b in zip(u, out[xi]))), 1)
        for n in ns:
            tot += bce(float(sum(a * b for a, b in zip(u, out[n]))), 0)
    return tot / len(c)
