"""SGNS oracle -- TEST INFRASTRUCTURE ONLY.

Restates /root/reference/pkg/src/walkvec/w2v.py in float64 numpy:
init (:123-131), min_count filter + shift-major pairs (:146-191), negatives
(:225-239, 500-504), SGNS loss/gradients (:247-299), coalescing (:407-416),
RowAdam (:364-404), batch sizing (:437-497), _train_single (:547-576),
the reproducible multi-worker contract (:579-746) and CBOW (instances
:194-222, gradients :302-361, window_size negatives per instance :481-484).  Implementation choices
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


def cbow_instances(tokens, offsets, window: int):
    """(ctx [N, 2W] -1 padded, lengths, targets): one instance per token of every
    walk of length >= 2; column 2(s-1) is the token s to the left, 2(s-1)+1 to the right."""
    rows, tg = [], []
    for w in range(len(offsets) - 1):
        t = tokens[offsets[w]:offsets[w + 1]]
        L = len(t)
        if L < 2:
            continue
        for i in range(L):
            r = [-1] * (2 * window)
            for s_ in range(1, window + 1):
                if i - s_ >= 0:
                    r[2 * (s_ - 1)] = t[i - s_]
                if i + s_ < L:
                    r[2 * (s_ - 1) + 1] = t[i + s_]
            rows.append(r)
            tg.append(t[i])
    if not rows:
        raise ValueError("empty training set")
    ctx = np.array(rows, dtype=np.int64).reshape(-1, 2 * window)
    return ctx, (ctx >= 0).sum(axis=1).astype(np.int64), np.array(tg, dtype=np.int64)


def cbow_step(inp, out, ctx, lengths, targets, negs):
    """loss + (rows, grads): context mean c, positive/negative logits against
    output rows, grad_c / len spread over the window (w2v.py:302-361)."""
    B, d = len(targets), inp.shape[1]
    mask = ctx >= 0
    c = np.zeros((B, d))
    for col in range(ctx.shape[1]):  # masked columns add nothing
        m = mask[:, col]
        c[m] += inp[ctx[m, col]]
    c /= lengths[:, None]
    t = out[targets]
    pos = np.matmul(c[:, None, :], t[:, :, None])[:, 0, 0]
    loss = np.logaddexp(0.0, -pos).sum()
    gpos = (1.0 / (1.0 + np.exp(-pos)) - 1.0) / B
    gc = gpos[:, None] * t
    orow, og = [targets], [gpos[:, None] * c]
    if negs.size:
        n = out[negs]
        neg = np.matmul(n, c[:, :, None])[:, :, 0]
        loss += np.logaddexp(0.0, neg).sum()
        gneg = (1.0 / (1.0 + np.exp(-neg))) / B
        gc = gc + (gneg[:, :, None] * n).sum(axis=1)
        orow.append(negs.ravel())
        og.append((gneg[:, :, None] * c[:, None, :]).reshape(-1, d))
    per = gc / lengths[:, None]
    b_of, col_of = np.nonzero(mask)  # row-major: the reference's contexts[mask] order
    return loss / B, ctx[b_of, col_of], per[b_of], np.concatenate(orow), np.vstack(og)


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
          sparse=True, max_batches=None, model="skipgram"):
    """Single-worker SGNS or CBOW (w2v.py:507-576) -> dict(inp, out, losses, touched_in, touched_out, keep).

    CBOW draws ``window`` negatives per instance (``k`` is ignored, w2v.py:481-484)."""
    tokens = np.asarray(tokens, dtype=np.int64)
    offsets = np.asarray(offsets, dtype=np.int64)
    freq = frequencies(tokens, V)
    keep = freq >= min_count
    ft, fo = filtered(tokens, offsets, keep)
    if len(ft) == 0:
        raise ValueError("empty training set")
    cbow = model == "cbow"
    if cbow:
        ctx, lens, tg = cbow_instances(ft, fo, window)
        k = window
        n_items = len(tg)
        per = (2 * window + 1 + window) * d * 8 + 16  # estimate_per_sample_bytes (w2v.py:437-448)
        B = batch if batch is not None else max(1, min(budget // (4 * per), -(-n_items // 20)))
        while B > 1 and B * per > 0.9 * budget:
            B //= 2
        pr = None
    else:
        pr = pairs(ft, fo, window)
        n_items = len(pr)
        B = batch_size(len(pr), d, k, budget, batch)
    cand = np.flatnonzero(keep)
    inp, out = init(V, d, seed)
    sh = np.random.default_rng(np.random.SeedSequence([int(seed), 1, 1]))
    ng = np.random.default_rng(np.random.SeedSequence([int(seed), 1, 2, 0]))
    oi, oo = RowAdam(inp.shape, lr, sparse), RowAdam(out.shape, lr, sparse)
    ti, to = np.zeros(V, bool), np.zeros(V, bool)
    losses, nb = [], 0
    for epoch in range(epochs):
        order = sh.permutation(n_items)
        tot, cnt = 0.0, 0
        for lo in range(0, n_items, B):
            idx = order[lo:lo + B]
            negs = cand[ng.integers(0, len(cand), size=len(idx) * k)].reshape(len(idx), k) if k else \
                np.empty((len(idx), 0), dtype=np.int64)
            if cbow:
                loss, ir, ig, orr, og = cbow_step(inp, out, ctx[idx], lens[idx], tg[idx], negs)
            else:
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
