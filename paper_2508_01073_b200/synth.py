"""Synthetic knowledge graphs of the benchmark shapes (vectorised, host numpy).

Reference generators: pkg/src/walkvec/benchgen.py:78-161.
  * gen_barabasi (:78-109): each new vertex v adds min(m, v) distinct edges
    v -> t, t drawn from the attachment bag (every vertex once per unit of
    degree + 1), so in-degree is power-law and out-degree is m.  The
    reference is a sequential Python loop (35 s at 1M vertices); here the bag
    draw is restated as position sampling + pointer jumping: a draw at bag
    position q of an earlier edge's target slot takes that edge's target.
    Same process, not the same numpy stream (stated in DESIGN.md).
  * gen_erdos_renyi (:112-127): blocked Bernoulli matrix -- already vectorised
    in the reference; the same stream consumption gives the same graph.
  * assign_predicates (:152-161): i.i.d. uniform predicate per edge from
    SeedSequence([seed, 3]) -- identical stream.
Token encoding is ingest.encode_integer_triples (first occurrence order).
"""

from __future__ import annotations

import numpy as np

from .ingest import encode_integer_triples


def _gen_rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([int(seed), 2]))


def barabasi_edges(n: int, m: int, seed: int = 0) -> np.ndarray:
    """(E,2) int64 (src, dst) preferential-attachment edges, vectorised."""
    if n < 2:
        raise ValueError("n must be >= 2")
    rng = _gen_rng(seed)
    v = np.arange(1, n, dtype=np.int64)
    k = np.minimum(m, v)                       # edges of vertex v
    e_off = np.zeros(n, dtype=np.int64)        # first edge index of vertex v (v>=1 at e_off[v])
    np.cumsum(k, out=e_off[1:])
    E = int(e_off[-1])
    src = np.repeat(v, k)
    j = np.arange(E, dtype=np.int64) - e_off[src - 1]  # slot within the vertex
    # bag length before vertex v: 1 + sum_{u<v} (2 k_u + 1)
    bag_before = np.ones(n, dtype=np.int64)
    bag_before[1:] += np.cumsum(2 * k + 1) - (2 * k + 1)
    # bag position of vertex u's block start (u >= 1): bag_before[u]
    L = bag_before[src]                        # draws of vertex v use positions [0, L)

    def resolve(q):
        # map bag position -> (kind, index): position 0 = vertex 0 self slot;
        # block of u>=1 at bag_before[u]: [t1, u, t2, u, ..., tk, u, u]
        u = np.searchsorted(bag_before, q, side="right") - 1
        off = q - bag_before[u]
        is_self0 = u == 0
        in_pairs = (~is_self0) & (off < 2 * k[np.maximum(u, 1) - 1])
        is_target = in_pairs & (off % 2 == 0)
        edge = np.where(is_target, e_off[np.maximum(u, 1) - 1] + off // 2, -1)
        return u, is_target, edge

    q = (rng.random(E) * L).astype(np.int64)
    tgt = np.full(E, -1, dtype=np.int64)
    for _ in range(64):
        u, is_t, edge = resolve(q)
        val = np.where(is_t, -1, u)
        ptr = edge.copy()
        unresolved = is_t.copy()
        # pointer jumping over target slots: value of edge e = value of the slot it drew
        cur_val = val
        cur_ptr = ptr
        for _ in range(64):
            if not unresolved.any():
                break
            nxt = cur_ptr[unresolved]
            nv = cur_val[nxt]
            np_ = cur_ptr[nxt]
            idx = np.flatnonzero(unresolved)
            cur_val = cur_val.copy()
            cur_ptr = cur_ptr.copy()
            cur_val[idx] = nv
            cur_ptr[idx] = np_
            unresolved = cur_val < 0
        tgt = cur_val
        # duplicate targets within a vertex are redrawn (the reference rejects them)
        key = src * n + tgt
        order = np.argsort(key, kind="stable")
        dup_sorted = np.zeros(E, dtype=bool)
        dup_sorted[1:] = key[order][1:] == key[order][:-1]
        dup = np.zeros(E, dtype=bool)
        dup[order] = dup_sorted
        if not dup.any():
            break
        q[dup] = (rng.random(int(dup.sum())) * L[dup]).astype(np.int64)
    del j
    return np.column_stack([src, tgt])


def erdos_renyi_edges(n: int, p: float, seed: int = 0) -> np.ndarray:
    """Ordered pairs (u, v), u != v, each present with probability p (benchgen.py:112-127)."""
    if not 0 < p < 1:
        raise ValueError("p must be in (0, 1)")
    rng = _gen_rng(seed)
    rows_per_block = max(1, (1 << 24) // n)
    chunks = []
    for lo in range(0, n, rows_per_block):
        hi = min(lo + rows_per_block, n)
        rr, cc = np.nonzero(rng.random((hi - lo, n)) < p)
        rr = rr + lo
        keep = rr != cc
        chunks.append(np.column_stack([rr[keep], cc[keep]]))
    return np.vstack(chunks).astype(np.int64)


def predicate_picks(n_edges: int, predicate_set_size: int, seed: int = 0) -> np.ndarray:
    """assign_predicates' stream (benchgen.py:152-161): one uniform pick per edge."""
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), 3]))
    return rng.integers(0, predicate_set_size, size=n_edges)


def synthetic_kg(model: str, n: int, m: int = 10, p: float = 0.001, predicates: int = 10, seed: int = 7):
    """Token-encoded synthetic KG: (edges (E,3) int64, vocab_size, entity_tokens, predicate_tokens)."""
    if model == "barabasi":
        e2 = barabasi_edges(n, m, seed)
    elif model == "erdos_renyi":
        e2 = erdos_renyi_edges(n, p, seed)
    else:
        raise ValueError(f"unknown model {model!r}")
    picks = predicate_picks(len(e2), predicates, seed)
    return encode_integer_triples(e2[:, 0], picks, e2[:, 1], n)


# ------------------------------------------------------------------ device --
def device_barabasi_edges(n: int, m: int, seed: int = 7, device=None):
    """(src, dst) int64 device tensors of a preferential-attachment graph (csrc/synth.cu)."""
    from . import _lib

    torch = _lib.require_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if n < 2:
        raise ValueError("n must be >= 2")
    if m < 1:
        raise ValueError("m must be >= 1")
    E = _lib.query("wv_barabasi_edge_count", n, m)
    src = torch.empty(E, dtype=torch.int64, device=dev)
    dst = torch.empty(E, dtype=torch.int64, device=dev)
    ws = torch.empty(_lib.query("wv_barabasi_workspace_bytes", n, m), dtype=torch.uint8, device=dev)
    _lib.call("wv_gen_barabasi", n, m, int(seed) & 0xFFFFFFFFFFFFFFFF, _lib.ptr(src), _lib.ptr(dst), _lib.ptr(ws),
              ws.numel(), _lib.stream_ptr())
    return src, dst


def _device_rows(fn: str, n: int, arg, seed: int, device=None):
    from . import _lib

    torch = _lib.require_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    ws = torch.empty(_lib.query("wv_gen_rows_workspace_bytes", n), dtype=torch.uint8, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    s = int(seed) & 0xFFFFFFFFFFFFFFFF
    _lib.call(fn, n, arg, s, None, None, _lib.ptr(cnt), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    E = int(cnt.item())
    src = torch.empty(max(E, 1), dtype=torch.int64, device=dev)
    dst = torch.empty(max(E, 1), dtype=torch.int64, device=dev)
    _lib.call(fn, n, arg, s, _lib.ptr(src), _lib.ptr(dst), _lib.ptr(cnt), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    return src[:E], dst[:E]


def device_erdos_renyi_edges(n: int, p: float, seed: int = 7, device=None):
    """(src, dst) device tensors: gen_erdos_renyi semantics (benchgen.py:112-127), counter-based draws."""
    if not 0 < p < 1:
        raise ValueError("p must be in (0, 1)")
    return _device_rows("wv_gen_erdos_renyi", int(n), float(p), seed, device)


def device_uniform_attachment_edges(n: int, m: int = 10, seed: int = 7, device=None):
    """(src, dst) device tensors: gen_uniform_attachment semantics (benchgen.py:130-149)."""
    if n < 2:
        raise ValueError("n must be >= 2")
    if not 1 <= m <= 64:
        raise ValueError("m must be in [1, 64]")
    return _device_rows("wv_gen_uniform_attachment", int(n), int(m), seed, device)


def device_encode(src, preds, dst, n_entities: int, n_predicates: int):
    """First-occurrence encoding on the device -> (edges (E,3), vocab_size, entity_tokens, predicate_tokens).

    Token arrays are sorted int64 device tensors (ingest.py:282-284).
    """
    from . import _lib

    torch = _lib.require_cuda()
    dev = src.device
    E = int(src.numel())
    n_keys = int(n_entities) + int(n_predicates)
    edges = torch.empty((max(E, 1), 3), dtype=torch.int64, device=dev)
    tok_of_key = torch.empty(n_keys, dtype=torch.int64, device=dev)
    key_of_tok = torch.empty(n_keys, dtype=torch.int64, device=dev)
    vocab = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = torch.empty(_lib.query("wv_encode_workspace_bytes", E, n_keys), dtype=torch.uint8, device=dev)
    _lib.call("wv_encode_triples", _lib.ptr(src), _lib.ptr(preds), _lib.ptr(dst), E, int(n_entities),
              int(n_predicates), _lib.ptr(edges), _lib.ptr(tok_of_key), _lib.ptr(key_of_tok), _lib.ptr(vocab),
              _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    V = int(vocab.item())
    kot = key_of_tok[:V]
    ent = torch.nonzero(kot < int(n_entities)).flatten()
    prd = torch.nonzero(kot >= int(n_entities)).flatten()
    return edges[:E], V, ent, prd


def device_synthetic_kg(model: str, n: int, m: int = 10, predicates: int = 10, seed: int = 7, p: float = 0.001,
                        device=None):
    """synthetic_kg with the edge generator and the token encoding on the device.

    Predicates are drawn from the reference's own stream (assign_predicates,
    SeedSequence([seed, 3]).integers) on the host.  Returns
    (edges (E,3) device int64, vocab_size, entity_tokens, predicate_tokens).
    """
    from . import _lib

    torch = _lib.require_cuda()
    if model == "barabasi":
        src, dst = device_barabasi_edges(n, m, seed, device)
    elif model == "erdos_renyi":
        src, dst = device_erdos_renyi_edges(n, p, seed, device)
    elif model == "uniform_attachment":
        src, dst = device_uniform_attachment_edges(n, m, seed, device)
    else:
        raise ValueError(f"unknown model {model!r}")
    picks = torch.from_numpy(predicate_picks(int(src.numel()), predicates, seed)).to(src.device)
    return device_encode(src, picks, dst, n, predicates)
