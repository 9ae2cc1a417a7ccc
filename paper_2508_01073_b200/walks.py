"""Walk-corpus extraction on the device (drop-in for walkvec.walks).

Reference: pkg/src/walkvec/walks.py.  ``random_walks`` (:144-204) replicates
the roots ``walk_number`` times, cuts 8192-walk shards with one numpy stream
per shard and draws one double per (hop, row).  The device kernel gives each
walker its own lane and addresses draw ``k = hop * n_shard + row`` of the
shard's stream directly (PCG64 jump-ahead, or Philox counters), so the corpus
is byte-identical to the reference for any launch split.  ``bfs_walks``
(:261-310) runs one CTA per root.  Corpora stay on the device as int32 tokens
plus int64 offsets; ``tokens`` / ``offsets`` materialise int64 numpy arrays
on first access for reference-shaped callers.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .graph import as_device_graph
from .seeding import entropy_words, words_array

RANDOM = "random"
BFS = "bfs"
FULL = "full"
ENTITY = "entity"
PROPERTY = "property"
SHARD_SIZE = 8192  # walks.py:34
PAD = -1

_RNG_KINDS = {"pcg64": _lib.RNG_PCG64, "philox": _lib.RNG_PHILOX}


@dataclass(frozen=True)
class Walk:
    walk_id: int
    tokens: np.ndarray


@dataclass
class PathTable:
    """Per-walk (source, target, walk_id) rows of BFS leaf-to-root paths (walks.py:87-103)."""

    sources: np.ndarray = field(default_factory=lambda: np.empty(0, dtype=np.int64))
    targets: np.ndarray = field(default_factory=lambda: np.empty(0, dtype=np.int64))
    walk_ids: np.ndarray = field(default_factory=lambda: np.empty(0, dtype=np.int64))

    def __len__(self) -> int:
        return len(self.sources)

    def rows(self) -> list[tuple[int, int, int]]:
        return list(zip(self.sources.tolist(), self.targets.tolist(), self.walk_ids.tolist()))


class WalkCorpus:
    """Flat walk storage; device-resident (int32 tokens, int64 offsets).

    Construct from host arrays (``WalkCorpus(tokens, offsets, strategy)``,
    reference signature) or from device tensors via ``from_device``.
    """

    def __init__(self, tokens=None, offsets=None, strategy: str = RANDOM, projection: str = FULL):
        self.strategy = strategy
        self.projection = projection
        self._h_tokens = None if tokens is None else np.asarray(tokens, dtype=np.int64)
        self._h_offsets = None if offsets is None else np.asarray(offsets, dtype=np.int64)
        self.d_tokens = None
        self.d_offsets = None
        self._n = None if offsets is None else len(self._h_offsets) - 1
        self._total = None if tokens is None else len(self._h_tokens)

    @classmethod
    def from_device(cls, d_tokens, d_offsets, n_walks: int, n_tokens: int, strategy=RANDOM, projection=FULL):
        c = cls(None, None, strategy, projection)
        c.d_tokens = d_tokens
        c.d_offsets = d_offsets
        c._n = int(n_walks)
        c._total = int(n_tokens)
        return c

    # -- device side ------------------------------------------------------
    def device_arrays(self, device=None):
        """(int32 tokens, int64 offsets) on the device, uploading host data once."""
        if self.d_tokens is None:
            torch = _lib.require_cuda()
            dev = device or torch.device("cuda", torch.cuda.current_device())
            tok = self._h_tokens if self._h_tokens is not None else np.empty(0, dtype=np.int64)
            if tok.size and (tok.min() < 0 or tok.max() >= 2**31):
                raise ValueError("token out of int32 range")
            self.d_tokens = torch.from_numpy(tok.astype(np.int32)).to(dev)
            self.d_offsets = torch.from_numpy(np.ascontiguousarray(self._h_offsets)).to(dev)
        return self.d_tokens, self.d_offsets

    # -- reference-compatible host views -----------------------------------
    @property
    def tokens(self) -> np.ndarray:
        if self._h_tokens is None:
            self._h_tokens = self.d_tokens[: self._total].cpu().numpy().astype(np.int64)
        return self._h_tokens

    @tokens.setter
    def tokens(self, value):
        self._h_tokens = np.asarray(value, dtype=np.int64)
        self._total = len(self._h_tokens)
        self.d_tokens = None

    @property
    def offsets(self) -> np.ndarray:
        if self._h_offsets is None:
            self._h_offsets = self.d_offsets[: self._n + 1].cpu().numpy()
        return self._h_offsets

    @offsets.setter
    def offsets(self, value):
        self._h_offsets = np.asarray(value, dtype=np.int64)
        self._n = len(self._h_offsets) - 1
        self.d_offsets = None

    def __len__(self) -> int:
        return int(self._n)

    @property
    def total_tokens(self) -> int:
        return int(self._total)

    def walk_tokens(self, i: int) -> np.ndarray:
        off = self.offsets
        return self.tokens[off[i]: off[i + 1]]

    def __iter__(self):
        for i in range(len(self)):
            yield Walk(i, self.walk_tokens(i))

    def sequences(self) -> list[np.ndarray]:
        return [self.walk_tokens(i) for i in range(len(self))]

    @classmethod
    def from_sequences(cls, sequences, strategy: str = RANDOM, projection: str = FULL) -> "WalkCorpus":
        lengths = np.fromiter((len(s) for s in sequences), dtype=np.int64, count=len(sequences))
        offsets = np.zeros(len(sequences) + 1, dtype=np.int64)
        np.cumsum(lengths, out=offsets[1:])
        tokens = np.concatenate([np.asarray(s, dtype=np.int64) for s in sequences]) if len(sequences) else \
            np.empty(0, dtype=np.int64)
        return cls(tokens, offsets, strategy, projection)


def _resolve_roots(graph, start_vertices) -> np.ndarray:
    """walks.py:106-114 semantics."""
    if start_vertices is None:
        return np.arange(graph.vertex_count, dtype=np.int64)
    roots = np.asarray(list(start_vertices) if not isinstance(start_vertices, np.ndarray) else start_vertices,
                       dtype=np.int64)
    if roots.size == 0:
        raise ValueError("start_vertices must be non-empty")
    if roots.min() < 0 or roots.max() >= graph.vertex_count:
        raise ValueError("start vertex out of range")
    return roots


def _ws(torch, nbytes, dev):
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=dev)


def _compact(torch, dev, corpus, lengths, n_walks, width, strategy, projection=FULL):
    offsets = torch.empty(n_walks + 1, dtype=torch.int64, device=dev)
    ws = _ws(torch, _lib.query("wv_compact_workspace_bytes", n_walks), dev)
    # total tokens = sum(lengths) is needed to size the flat buffer
    total = int(lengths[:n_walks].sum()) if n_walks else 0
    tokens = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    _lib.call("wv_corpus_compact", _lib.ptr(corpus), _lib.ptr(lengths), n_walks, width, _lib.ptr(offsets),
              _lib.ptr(tokens), 4, _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    return WalkCorpus.from_device(tokens, offsets, n_walks, total, strategy, projection)


def random_walks_fixed(graph, roots, walk_depth: int, walk_number: int, rng_seed: int, rng: str = "pcg64",
                       work_begin: int = 0, work_count: int | None = None):
    """Raw kernel call: fixed-width int32 rows [work_count, 2*depth+1] (-1 padded) + lengths.

    ``roots`` is a device int64 tensor; the walkers are the slice
    ``[work_begin, work_begin + work_count)`` of repeat(roots, walk_number).
    """
    torch = _lib.require_cuda()
    g = as_device_graph(graph)
    dev = g.device
    n_roots = int(roots.numel())
    total = n_roots * int(walk_number)
    if work_count is None:
        work_count = total - work_begin
    width = 2 * int(walk_depth) + 1
    corpus = torch.empty(max(work_count, 1) * width, dtype=torch.int32, device=dev)
    lengths = torch.empty(max(work_count, 1), dtype=torch.int32, device=dev)
    words, n = words_array(entropy_words([rng_seed, 0]))
    adj = g.walk_adjacency()
    ws = _ws(torch, _lib.query("wv_random_walks_workspace_bytes", int(work_begin), int(work_count)), dev)
    _lib.call("wv_random_walks", _lib.ptr(g.d_row_offsets), _lib.ptr(g.d_edges), _lib.ptr(adj), g.vertex_count,
              _lib.ptr(roots), n_roots, int(walk_number), int(walk_depth), int(work_begin), int(work_count), words, n,
              _RNG_KINDS[rng], _lib.ptr(corpus), _lib.ptr(lengths), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    return corpus, lengths, width


def random_walks(graph, start_vertices=None, walk_depth: int = 5, walk_number: int = 1, rng_seed: int = 0,
                 duplicate_free: bool = False, workers: int = 1, *, rng: str = "pcg64") -> WalkCorpus:
    """Fixed-depth uniform random walks over out-edges (walks.py:144-204).

    ``workers`` is accepted for signature compatibility (the corpus never
    depends on it).  ``rng="pcg64"`` reproduces the unmodified reference
    bit-for-bit; ``rng="philox"`` reproduces the reference driven by
    ``Generator(Philox(SeedSequence(...)))``.
    """
    if walk_depth < 1:
        raise ValueError("walk_depth must be >= 1")
    if walk_number < 1:
        raise ValueError("walk_number must be >= 1")
    if rng not in _RNG_KINDS:
        raise ValueError(f"unknown rng {rng!r}")
    torch = _lib.require_cuda()
    g = as_device_graph(graph)
    dev = g.device
    roots_np = _resolve_roots(g, start_vertices)
    roots = torch.from_numpy(roots_np).to(dev)
    corpus, lengths, width = random_walks_fixed(g, roots, walk_depth, walk_number, rng_seed, rng)
    n_walks = len(roots_np) * int(walk_number)
    if duplicate_free:
        out_c = torch.empty_like(corpus)
        out_l = torch.empty_like(lengths)
        n_kept = torch.zeros(1, dtype=torch.int64, device=dev)
        ws = _ws(torch, _lib.query("wv_dedup_workspace_bytes", n_walks), dev)
        _lib.call("wv_duplicate_free", _lib.ptr(corpus), _lib.ptr(lengths), n_walks, width, int(walk_number),
                  _lib.ptr(out_c), _lib.ptr(out_l), _lib.ptr(n_kept), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
        corpus, lengths, n_walks = out_c, out_l, int(n_kept.item())
    return _compact(torch, dev, corpus, lengths, n_walks, width, RANDOM)


def bfs_walks(graph, start_vertices=None, walk_depth: int = 5, *, max_walks_per_root: int | None = None,
              with_table: bool = True):
    """BFS predecessor-tree walks (walks.py:261-310) -> (WalkCorpus, PathTable).

    ``max_walks_per_root`` (not in the reference; None = uncapped) keeps the
    first walks of each root in the reference's leaf-discovery order.
    """
    if walk_depth < 1:
        raise ValueError("walk_depth must be >= 1")
    torch = _lib.require_cuda()
    g = as_device_graph(graph)
    dev = g.device
    roots_np = _resolve_roots(g, start_vertices)
    roots = torch.from_numpy(roots_np).to(dev)
    R = len(roots_np)
    cap = int(max_walks_per_root) if max_walks_per_root else 0
    counts = torch.empty(R, dtype=torch.int64, device=dev)
    ws = _ws(torch, _lib.query("wv_bfs_workspace_bytes", g.vertex_count, R), dev)
    st = _lib.stream_ptr()
    _lib.call("wv_bfs_count", _lib.ptr(g.d_row_offsets), _lib.ptr(g.d_edges), g.vertex_count, _lib.ptr(roots), R,
              int(walk_depth), cap, _lib.ptr(counts), _lib.ptr(ws), ws.numel(), st)
    if bool((counts < 0).any()):
        raise RuntimeError("BFS tree exceeded the fallback capacity")
    base = torch.zeros(R + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=base[1:])
    n_walks = int(base[R])
    width = 2 * int(walk_depth) + 1
    corpus = torch.empty(max(n_walks, 1) * width, dtype=torch.int32, device=dev)
    lengths = torch.empty(max(n_walks, 1), dtype=torch.int32, device=dev)
    _lib.call("wv_bfs_emit", _lib.ptr(g.d_row_offsets), _lib.ptr(g.d_edges), g.vertex_count, _lib.ptr(roots), R,
              int(walk_depth), cap, _lib.ptr(base), _lib.ptr(corpus), _lib.ptr(lengths), _lib.ptr(ws), ws.numel(), st)
    corpus_obj = _compact(torch, dev, corpus, lengths, n_walks, width, BFS)
    if not with_table:
        return corpus_obj, None
    rows = (corpus_obj.total_tokens - n_walks) // 2
    src = torch.empty(max(rows, 1), dtype=torch.int64, device=dev)
    dst = torch.empty(max(rows, 1), dtype=torch.int64, device=dev)
    wid = torch.empty(max(rows, 1), dtype=torch.int64, device=dev)
    _lib.call("wv_path_table", _lib.ptr(corpus_obj.d_tokens), _lib.ptr(corpus_obj.d_offsets), n_walks, _lib.ptr(src),
              _lib.ptr(dst), _lib.ptr(wid), st)
    table = PathTable(src[:rows].cpu().numpy(), dst[:rows].cpu().numpy(), wid[:rows].cpu().numpy())
    return corpus_obj, table


def project_entity(walk: Walk) -> Walk:
    return Walk(walk.walk_id, walk.tokens[0::2])


def project_property(walk: Walk) -> Walk:
    return Walk(walk.walk_id, np.concatenate([walk.tokens[:1], walk.tokens[1::2]]))


def project_corpus(corpus: WalkCorpus, projection: str) -> WalkCorpus:
    """Entity / property projection of a full corpus (walks.py:323-341), on the device."""
    if projection == FULL:
        return corpus
    if getattr(corpus, "projection", FULL) != FULL:
        raise ValueError("corpus is already projected")
    if projection not in (ENTITY, PROPERTY):
        raise ValueError(f"unknown projection: {projection!r}")
    torch = _lib.require_cuda()
    if not isinstance(corpus, WalkCorpus):
        corpus = WalkCorpus(corpus.tokens, corpus.offsets, getattr(corpus, "strategy", RANDOM))
    tok, off = corpus.device_arrays()
    dev = tok.device
    n = len(corpus)
    mode = _lib.KEEP_ENTITY if projection == ENTITY else _lib.KEEP_PROPERTY
    new_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    new_tok = torch.empty(max(corpus.total_tokens, 1), dtype=torch.int32, device=dev)
    ws = _ws(torch, _lib.query("wv_filter_workspace_bytes", n), dev)
    _lib.call("wv_corpus_filter", _lib.ptr(tok), _lib.ptr(off), n, mode, None, _lib.ptr(new_off), _lib.ptr(new_tok),
              _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    total = int(new_off[n]) if n else 0
    return WalkCorpus.from_device(new_tok, new_off, n, total, corpus.strategy, projection)
