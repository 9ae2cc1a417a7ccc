"""SGNS training on the device (drop-in for walkvec.w2v.train, model="skipgram").

Reference: pkg/src/walkvec/w2v.py.  Semantics kept exactly:
  * frequencies over the raw corpus, tokens below min_count dropped before
    windowing (:146-191); candidates = flatnonzero(freq >= min_count) (:525-526)
  * U(-1/d, 1/d) init from SeedSequence([seed,1,0]) (:123-131), bit-exact
  * batch size = explicit or min(budget // (4*per_sample), ceil(N/20)),
    halved while over cap*budget with a ``batch_halved`` event (:437-497)
  * per epoch: a permutation of all pairs, contiguous batches, fresh uniform
    negatives per batch, batch-mean BCE loss, non-finite loss ->
    TrainingDiverged(epoch, batch) (:547-576)
  * duplicate rows summed in slot order, per-row Adam with per-row step
    counts (sparse) or one global step (dense) (:364-434)
  * multi-worker: contiguous spans of the permutation per worker, local
    replicas with their own Adam, averaged deltas every sync round (:579-746)

Two pair sources:
  * ``pairs="device"`` (default): the permutation is a keyed Feistel bijection
    over [0, N) and negatives come from Philox, all on the device; pairs are
    decoded on the fly from the corpus (never materialised).
  * ``pairs="numpy"``: replay of the reference's own numpy streams (the
    permutation from SeedSequence([seed,1,1]) and the negatives from
    [seed,1,2,worker]) through the same kernels -- matches ``train()`` of the
    reference to fp64 rounding (precision="fp64") on the same inputs.
"""

from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from .seeding import entropy_words, words_array

SKIPGRAM = "skipgram"
CBOW = "cbow"
DEFAULT_MEMORY_BUDGET = 1 << 30
MEMORY_BUDGET_ENV = "WALKVEC_MEMORY_BUDGET"
REPRODUCIBLE_SYNC_BATCHES = 64
# device timestamps per profiled batch (WvSgnsBatch.timer): start, decode end,
# gather end, join, owner end, sort start, sort end
STAMPS_PER_BATCH = 7
# (start, end) stamp pairs of the profiled phases: decode, gather, grouping (side stream), owner, whole batch
_PHASE_SLOTS = ((0, 1), (1, 2), (5, 6), (3, 4), (0, 4))
PHASE_NAMES = ("decode", "gather", "group", "owner", "batch")


class TrainingDiverged(RuntimeError):
    """Raised when a batch loss goes non-finite (w2v.py:46-52)."""

    def __init__(self, epoch: int, batch: int):
        super().__init__(f"divergence at epoch {epoch}, batch {batch}")
        self.epoch = epoch
        self.batch = batch


@dataclass
class TrainConfig:
    """Training hyperparameters (field-for-field the reference TrainConfig, w2v.py:55-90)."""

    model: str = SKIPGRAM
    epochs: int = 5
    window_size: int = 5
    negative_samples: int = 5
    learning_rate: float = 0.01
    min_count: int = 10
    vector_size: int = 100
    batch_size: int | None = None
    sync_interval_ms: int = 500
    memory_budget_bytes: int | None = None
    memory_cap_fraction: float = 0.9
    use_sparse: bool = True
    workers: int = 1
    reproducible: bool = False

    def __post_init__(self):
        if self.model not in (SKIPGRAM, CBOW):
            raise ValueError(f"unknown model: {self.model!r}")
        checks = (("epochs", 1), ("window_size", 1), ("negative_samples", 0), ("min_count", 0),
                  ("vector_size", 1), ("workers", 1))
        for name, lo in checks:
            if getattr(self, name) < lo:
                raise ValueError(f"{name} must be >= {lo}")
        if not 0 < self.memory_cap_fraction <= 1:
            raise ValueError("memory_cap_fraction must be in (0, 1]")
        if self.batch_size is not None and self.batch_size < 1:
            raise ValueError("batch_size must be >= 1 or None")


def estimate_per_sample_bytes(model_kind: str, d: int, negative_samples: int, window_size: int) -> int:
    """float64 rows one sample touches (w2v.py:437-443)."""
    rows = 2 + negative_samples if model_kind == SKIPGRAM else 2 * window_size + 1 + window_size
    return rows * d * 8 + 16


def suggest_batch_size(per_sample_bytes: int, memory_budget_bytes: int, corpus_pair_count: int) -> int:
    """min(budget // (4 * per_sample), ceil(N / 20)), at least 1 (w2v.py:446-456)."""
    if per_sample_bytes <= 0:
        raise ValueError("per_sample_bytes must be positive")
    by_memory = int(memory_budget_bytes) // (4 * int(per_sample_bytes))
    by_corpus = -(-int(corpus_pair_count) // 20)
    return max(1, min(by_memory, by_corpus))


def resolve_memory_budget(config: TrainConfig) -> int:
    """env WALKVEC_MEMORY_BUDGET > config > 1 GiB (w2v.py:459-465)."""
    env = os.environ.get(MEMORY_BUDGET_ENV)
    if env:
        return int(env)
    if config.memory_budget_bytes is not None:
        return int(config.memory_budget_bytes)
    return DEFAULT_MEMORY_BUDGET


def _clamped_batch_size(batch_size, per_sample, budget, cap, events):
    while batch_size > 1 and batch_size * per_sample > cap * budget:
        batch_size //= 2
        events("batch_halved", batch_size=batch_size)
    return batch_size


# ------------------------------------------------------------------ model --
class EmbeddingModel:
    """Paired |V| x d matrices (w2v.py:93-112), resident on the device.

    ``input_matrix`` / ``output_matrix`` are float64 numpy arrays materialised
    on first access: rows the optimizer never changed are regenerated
    bit-exactly from the init stream, the rest are the stored values.
    """

    def __init__(self, params, dim: int, trained_mask: np.ndarray):
        self._p = params  # _Params
        self.dim = int(dim)
        self.trained_mask = trained_mask
        self._cache = {}
        self._touched = {}

    @property
    def vocab_size(self) -> int:
        return self._p.V

    def _export(self, which: int) -> np.ndarray:
        if which not in self._cache:
            self._cache[which] = self._p.export(which)
        return self._cache[which]

    @property
    def input_matrix(self) -> np.ndarray:
        return self._export(0)

    @property
    def output_matrix(self) -> np.ndarray:
        return self._export(1)

    @property
    def touched_input(self) -> np.ndarray:
        if "in" not in self._touched:
            self._touched["in"] = self._p.touched_in.cpu().numpy().astype(bool)
        return self._touched["in"]

    @property
    def touched_output(self) -> np.ndarray:
        if "out" not in self._touched:
            self._touched["out"] = self._p.touched_out.cpu().numpy().astype(bool)
        return self._touched["out"]

    # device views (no copies) for GPU consumers
    @property
    def device_input(self):
        return self._p.inp

    @property
    def device_output(self):
        return self._p.out


class _Params:
    """Device parameter store + optimizer state of one replica."""

    def __init__(self, torch, dev, V: int, d: int, seed: int, precision: str, sparse: bool, lr: float,
                 shard: tuple[int, int] | None = None):
        """``shard=(nshard, rank)``: hold only the rows r with r % nshard == rank (row-sharded mode)."""
        self.torch = torch
        self.dev = dev
        self.V_global = int(V)
        self.shard = shard
        if shard is not None:
            V = -(-int(V) // shard[0])
        self.V, self.d = int(V), int(d)
        self.seed = int(seed)
        self.precision = _lib.FP64 if precision == "fp64" else _lib.FP32
        dt = torch.float64 if self.precision == _lib.FP64 else torch.float32
        self.dtype = dt
        self.sparse = bool(sparse)
        self.lr = float(lr)
        n = self.V * self.d
        self.inp = torch.empty(n, dtype=dt, device=dev)
        self.out = torch.empty(n, dtype=dt, device=dev)
        self.m_in = torch.zeros(n, dtype=dt, device=dev)
        self.v_in = torch.zeros(n, dtype=dt, device=dev)
        self.m_out = torch.zeros(n, dtype=dt, device=dev)
        self.v_out = torch.zeros(n, dtype=dt, device=dev)
        self.steps_in = torch.zeros(self.V, dtype=torch.int32, device=dev)
        self.steps_out = torch.zeros(self.V, dtype=torch.int32, device=dev)
        self.touched_in = torch.zeros(self.V, dtype=torch.uint8, device=dev)
        self.touched_out = torch.zeros(self.V, dtype=torch.uint8, device=dev)
        self.modified_in = torch.zeros(self.V, dtype=torch.uint8, device=dev)
        self.modified_out = torch.zeros(self.V, dtype=torch.uint8, device=dev)
        if self.sparse:
            self.dg_in = self.dg_out = None
        else:
            self.dg_in = torch.zeros(n, dtype=dt, device=dev)
            self.dg_out = torch.zeros(n, dtype=dt, device=dev)
        init = _lib.WvSgnsDevState()
        init.diverged_epoch = -1
        init.diverged_batch = -1
        host = torch.frombuffer(bytearray(bytes(init)), dtype=torch.uint8)
        self.state = host.to(dev)
        words, nw = words_array(entropy_words([seed, 1, 0]))
        self._init_words = (words, nw)
        if shard is None:
            _lib.call("wv_sgns_init", self.V, self.d, words, nw, self.precision, _lib.ptr(self.inp),
                      _lib.ptr(self.out), _lib.stream_ptr())
        else:
            _lib.call("wv_shard_init", self.V_global, self.d, words, nw, self.precision, int(shard[0]),
                      int(shard[1]), _lib.ptr(self.inp), _lib.ptr(self.out), _lib.stream_ptr())
        self.struct = _lib.WvSgnsModel(
            vocab_size=self.V, vector_size=self.d, precision=self.precision, sparse=int(self.sparse), pad=0,
            learning_rate=self.lr, input=_lib.ptr(self.inp), output=_lib.ptr(self.out), m_in=_lib.ptr(self.m_in),
            v_in=_lib.ptr(self.v_in), m_out=_lib.ptr(self.m_out), v_out=_lib.ptr(self.v_out),
            steps_in=_lib.ptr(self.steps_in), steps_out=_lib.ptr(self.steps_out),
            touched_in=_lib.ptr(self.touched_in), touched_out=_lib.ptr(self.touched_out),
            modified_in=_lib.ptr(self.modified_in), modified_out=_lib.ptr(self.modified_out),
            dense_g_in=_lib.ptr(self.dg_in), dense_g_out=_lib.ptr(self.dg_out), state=_lib.ptr(self.state))

    def read_state(self) -> _lib.WvSgnsDevState:
        raw = bytes(self.state.cpu().numpy().tobytes())
        return _lib.WvSgnsDevState.from_buffer_copy(raw)

    def export(self, which: int) -> np.ndarray:
        torch = self.torch
        out64 = torch.empty(self.V * self.d, dtype=torch.float64, device=self.dev)
        params = self.inp if which == 0 else self.out
        modified = self.modified_in if which == 0 else self.modified_out
        words, nw = self._init_words
        _lib.call("wv_sgns_export", self.V, self.d, words, nw, self.precision, which, _lib.ptr(params),
                  _lib.ptr(modified), _lib.ptr(out64), _lib.stream_ptr())
        return out64.cpu().numpy().reshape(self.V, self.d)


def init_embeddings(vocab_size: int, d: int, rng_seed: int, precision: str = "fp64") -> EmbeddingModel:
    """U(-1/d, 1/d) init on the device, bit-exact with w2v.init_embeddings (:123-131)."""
    if d < 1:
        raise ValueError("embedding dimension must be >= 1")
    torch = _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    p = _Params(torch, dev, vocab_size, d, rng_seed, precision, True, 0.0)
    # an untrained model: every row is its init; export straight from the store
    p.modified_in.fill_(1)
    p.modified_out.fill_(1)
    return EmbeddingModel(p, d, np.zeros(vocab_size, dtype=bool))


# ----------------------------------------------------------------- corpus --
class _DeviceCorpus:
    """Flat corpus on the device plus its frequency table and pair index."""

    def __init__(self, torch, dev, corpus, vocab_size: int, window: int, min_count: int):
        self.torch = torch
        self.dev = dev
        tok, off, n_walks, n_tok = _corpus_device_arrays(torch, dev, corpus)
        V = int(vocab_size)
        if n_tok:
            lo, hi = torch.aminmax(tok[:n_tok])
            if int(lo) < 0 or int(hi) >= V:
                raise ValueError("corpus token out of range for vocab_size")
        self.freq = torch.zeros(V, dtype=torch.int64, device=dev)
        st = _lib.stream_ptr()
        _lib.call("wv_token_histogram", _lib.ptr(tok), n_tok, V, _lib.ptr(self.freq), 0, st)
        self.keep = torch.empty(V, dtype=torch.uint8, device=dev)
        self.candidates = torch.empty(max(V, 1), dtype=torch.int32, device=dev)
        n_cand = torch.zeros(1, dtype=torch.int64, device=dev)
        ws = torch.empty(_lib.query("wv_candidates_workspace_bytes", V), dtype=torch.uint8, device=dev)
        _lib.call("wv_candidates", _lib.ptr(self.freq), V, int(min_count), _lib.ptr(self.keep),
                  _lib.ptr(self.candidates), _lib.ptr(n_cand), _lib.ptr(ws), ws.numel(), st)
        self.n_candidates = int(n_cand.item())
        # drop below-min_count tokens before windowing (windows close over gaps)
        dropped = bool(((self.freq > 0) & (self.keep == 0)).any()) if n_tok else False
        if dropped:
            new_off = torch.empty(n_walks + 1, dtype=torch.int64, device=dev)
            new_tok = torch.empty(max(n_tok, 1), dtype=torch.int32, device=dev)
            ws = torch.empty(_lib.query("wv_filter_workspace_bytes", n_walks), dtype=torch.uint8, device=dev)
            _lib.call("wv_corpus_filter", _lib.ptr(tok), _lib.ptr(off), n_walks, _lib.KEEP_TOKENS,
                      _lib.ptr(self.keep), _lib.ptr(new_off), _lib.ptr(new_tok), _lib.ptr(ws), ws.numel(), st)
            tok, off = new_tok, new_off
            n_tok = int(off[n_walks]) if n_walks else 0
        self.tokens, self.offsets, self.n_walks, self.n_tokens = tok, off, n_walks, n_tok
        self.window = int(window)
        if n_tok == 0:
            raise ValueError("empty training set")
        # length-class pair index (the native pair decode)
        W = n_walks
        self.walks_by_class = torch.empty(W, dtype=torch.int32, device=dev)
        self.class_len = torch.empty(W + 1, dtype=torch.int64, device=dev)
        self.class_walk_start = torch.empty(W + 1, dtype=torch.int64, device=dev)
        self.class_pair_start = torch.empty(W + 1, dtype=torch.int64, device=dev)
        nc = torch.zeros(1, dtype=torch.int64, device=dev)
        npairs = torch.zeros(1, dtype=torch.int64, device=dev)
        ws = torch.empty(_lib.query("wv_pair_index_workspace_bytes", W), dtype=torch.uint8, device=dev)
        _lib.call("wv_pair_index_build", _lib.ptr(off), W, self.window, _lib.ptr(self.walks_by_class),
                  _lib.ptr(self.class_len), _lib.ptr(self.class_walk_start), _lib.ptr(self.class_pair_start),
                  _lib.ptr(nc), _lib.ptr(npairs), _lib.ptr(ws), ws.numel(), st)
        self.n_classes = int(nc.item())
        self.n_pairs = int(npairs.item())
        if self.n_pairs == 0:
            raise ValueError("empty training set")

    def cbow_instances(self):
        """CBOW instance table [N, 2W+1] int32 in the reference's order (w2v.py:194-222)."""
        torch = self.torch
        n = torch.zeros(1, dtype=torch.int64, device=self.dev)
        ws = torch.empty(_lib.query("wv_cbow_instances_workspace_bytes", self.n_walks), dtype=torch.uint8,
                         device=self.dev)
        st = _lib.stream_ptr()
        _lib.call("wv_cbow_instances", _lib.ptr(self.tokens), _lib.ptr(self.offsets), self.n_walks, self.window, None,
                  _lib.ptr(n), _lib.ptr(ws), ws.numel(), st)
        self.n_instances = int(n.item())
        if self.n_instances == 0:
            raise ValueError("empty training set")
        inst = torch.empty(self.n_instances * (2 * self.window + 1), dtype=torch.int32, device=self.dev)
        _lib.call("wv_cbow_instances", _lib.ptr(self.tokens), _lib.ptr(self.offsets), self.n_walks, self.window,
                  _lib.ptr(inst), _lib.ptr(n), _lib.ptr(ws), ws.numel(), st)
        return inst

    def reference_pairs(self):
        """(N,2) int32 pair table in the reference's shift-major order (w2v.py:177-190)."""
        torch = self.torch
        pairs = torch.empty(2 * self.n_pairs, dtype=torch.int32, device=self.dev)
        n_out = C.c_int64(0)
        ws = torch.empty(_lib.query("wv_pairs_workspace_bytes", self.n_walks), dtype=torch.uint8, device=self.dev)
        _lib.call("wv_generate_pairs", _lib.ptr(self.tokens), _lib.ptr(self.offsets), self.n_walks, self.window,
                  _lib.ptr(pairs), C.byref(n_out), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
        assert n_out.value == self.n_pairs, (n_out.value, self.n_pairs)
        return pairs


def _corpus_device_arrays(torch, dev, corpus):
    """Accept our WalkCorpus, any object with tokens/offsets, or an iterable of sequences (w2v.py:134-143)."""
    from .walks import WalkCorpus

    if isinstance(corpus, WalkCorpus):
        tok, off = corpus.device_arrays(dev)
        return tok, off, len(corpus), corpus.total_tokens
    if hasattr(corpus, "tokens") and hasattr(corpus, "offsets"):
        tokens = np.asarray(corpus.tokens, dtype=np.int64)
        offsets = np.asarray(corpus.offsets, dtype=np.int64)
    else:
        seqs = [np.asarray(s, dtype=np.int64) for s in corpus]
        lengths = np.array([len(s) for s in seqs], dtype=np.int64)
        offsets = np.zeros(len(seqs) + 1, dtype=np.int64)
        np.cumsum(lengths, out=offsets[1:])
        tokens = np.concatenate(seqs) if seqs else np.empty(0, dtype=np.int64)
    if tokens.size and (tokens.min() < 0 or tokens.max() >= 2**31):
        raise ValueError("corpus token out of range")
    n = len(offsets) - 1
    tok = torch.from_numpy(tokens.astype(np.int32)).to(dev) if tokens.size else torch.zeros(1, dtype=torch.int32,
                                                                                            device=dev)
    return tok, torch.from_numpy(offsets).to(dev), n, int(tokens.size)


def generate_pairs(corpus, window_size: int, min_count: int, vocab_size: int | None = None):
    """(pairs int64 (N,2), frequency) in the reference order (w2v.py:161-191), computed on the device."""
    torch = _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    if vocab_size is None:
        tok, _, _, n_tok = _corpus_device_arrays(torch, dev, corpus)
        vocab_size = int(tok[:n_tok].max()) + 1 if n_tok else 0
    if vocab_size == 0:
        raise ValueError("empty training set")
    dc = _DeviceCorpus(torch, dev, corpus, vocab_size, window_size, min_count)
    pairs = dc.reference_pairs().view(-1, 2).cpu().numpy().astype(np.int64)
    return pairs, dc.freq.cpu().numpy()


def generate_cbow_instances(corpus, window_size: int, min_count: int, vocab_size: int | None = None):
    """(contexts (N, 2W) -1 padded, lengths, targets, frequency) like w2v.py:194-222, computed on the device."""
    torch = _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    if vocab_size is None:
        tok, _, _, n_tok = _corpus_device_arrays(torch, dev, corpus)
        vocab_size = int(tok[:n_tok].max()) + 1 if n_tok else 0
    if vocab_size == 0:
        raise ValueError("empty training set")
    dc = _DeviceCorpus(torch, dev, corpus, vocab_size, window_size, min_count)
    inst = dc.cbow_instances().view(-1, 2 * int(window_size) + 1).cpu().numpy().astype(np.int64)
    ctx = inst[:, :-1]
    return ctx, (ctx >= 0).sum(axis=1).astype(np.int64), inst[:, -1].copy(), dc.freq.cpu().numpy()


# ---------------------------------------------------------------- trainer --
class _Replica:
    """One worker: its parameter store, its batch workspace and launch closures.

    The captured CUDA graphs depend only on the parameter store, the workspace
    and the batch size: the corpus is read through the workspace's bound
    descriptor, so ``retarget`` onto a new corpus keeps them (no recapture).
    """

    def __init__(self, trainer, widx: int, params: _Params):
        self.t = trainer
        self.widx = widx
        self.p = params
        torch = trainer.torch
        self.k = trainer.k
        self.batch_size = trainer.batch_size
        self.cw = trainer.cbow_window
        self.ws = torch.empty(_lib.query("wv_sgns_batch_workspace_bytes", params.V, params.d, trainer.k,
                                         trainer.batch_size, params.precision, self.cw), dtype=torch.uint8,
                              device=trainer.dev)
        _lib.call("wv_sgns_workspace_init", _lib.ptr(self.ws), self.ws.numel(), params.V, params.d, trainer.k,
                  trainer.batch_size, params.precision, self.cw, _lib.stream_ptr())
        self.graphs = {}
        self.graph_launches = {}  # key -> kernels per replay
        self.profile_samples = []  # [(decode, gather, group, owner, batch) ms] of profiled batches
        self.bind()

    def compatible(self, trainer) -> bool:
        return trainer.k == self.k and trainer.batch_size <= self.batch_size and trainer.cbow_window == self.cw

    def retarget(self, trainer):
        """Train the same replica on another corpus (same batch geometry)."""
        self.t = trainer
        self.bind()

    def bind(self):
        bs = self.t.batch_struct
        bs.batch_rows = self.batch_size
        _lib.call("wv_sgns_bind", C.byref(bs), _lib.ptr(self.ws), self.ws.numel(), self.p.V, self.p.d,
                  self.p.precision, _lib.stream_ptr())

    def launch(self, rows: int, events=None):
        """One batch; ``events`` = (DeviceTimer, first slot): STAMPS_PER_BATCH device timestamps."""
        t = self.t
        bs = t.batch_struct
        bs.batch_rows = int(rows)
        if events is None:
            _lib.call("wv_sgns_batch", C.byref(self.p.struct), C.byref(bs), _lib.ptr(self.ws), self.ws.numel(),
                      _lib.stream_ptr())
            return
        timer, base = events
        bs.timer, bs.timer_base = timer.h, int(base)
        try:
            _lib.call("wv_sgns_batch", C.byref(self.p.struct), C.byref(bs), _lib.ptr(self.ws), self.ws.numel(),
                      _lib.stream_ptr())
        finally:
            bs.timer, bs.timer_base = None, 0

    def launch_many(self, rows: int, count: int):
        """``count`` consecutive batches, pipelined across the workspace halves."""
        bs = self.t.batch_struct
        bs.batch_rows = int(rows)
        _lib.call("wv_sgns_batches", C.byref(self.p.struct), C.byref(bs), _lib.ptr(self.ws), self.ws.numel(),
                  int(count), _lib.stream_ptr())

    def _profiled(self, count: int, rows: int, every: int = 16):
        """Eager batches; one in ``every`` bracketed by device timestamps (no graph nodes distort it)."""
        sampled = list(range(0, count, every))
        timer = _lib.DeviceTimer(STAMPS_PER_BATCH * max(len(sampled), 1))
        slot = {b: i for i, b in enumerate(sampled)}
        for b in range(count):
            i = slot.get(b)
            self.launch(rows, None if i is None else (timer, STAMPS_PER_BATCH * i))
        self.t.torch.cuda.current_stream().synchronize()
        for i in range(len(sampled)):
            o = STAMPS_PER_BATCH * i
            self.profile_samples.append(tuple(timer.elapsed(o + a, o + b) for a, b in _PHASE_SLOTS))

    def run(self, count: int, rows: int):
        """``count`` consecutive batches of ``rows`` pairs, CUDA-graph replayed."""
        torch = self.t.torch
        G = self.t.graph_batches
        if count <= 0:
            return
        if self.t.profile:
            self._profiled(count, rows)
            return
        if G <= 1 or count < 2:
            self.launch_many(rows, count)
            return
        key = (rows, min(G, count))
        reps, rem = divmod(count, key[1])
        if key not in self.graphs:
            g = torch.cuda.CUDAGraph()
            before = _lib.launch_count()
            # capture on a side stream without torch.cuda.graph's gc.collect()/empty_cache()
            cur = torch.cuda.current_stream()
            cap = torch.cuda.Stream(device=self.t.dev)
            cap.wait_stream(cur)
            with torch.cuda.stream(cap):
                g.capture_begin()
                try:
                    self.launch_many(rows, key[1])
                finally:
                    g.capture_end()
            cur.wait_stream(cap)
            self.graphs[key] = g
            self.graph_launches[key] = _lib.launch_count() - before
            _lib.note_graph_replay(-self.graph_launches[key])  # the capture itself runs nothing
        g = self.graphs[key]
        for _ in range(reps):
            g.replay()
        _lib.note_graph_replay(reps * self.graph_launches[key])
        if rem:
            self.launch_many(rows, rem)


class _Trainer:
    def __init__(self, corpus, vocab_size, config: TrainConfig, rng_seed, events, precision, pairs, graph_batches,
                 device=None):
        torch = _lib.require_cuda()
        self.torch = torch
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.config = config
        self.seed = int(rng_seed)
        self.events = events
        # CBOW draws window_size negatives per instance (w2v.py:481-484)
        self.cbow_window = int(config.window_size) if config.model == CBOW else 0
        self.k = int(config.window_size) if config.model == CBOW else int(config.negative_samples)
        self.pairs_mode = pairs
        self.graph_batches = int(graph_batches)
        self.profile = False
        self.V = int(vocab_size)
        self.dc = _DeviceCorpus(torch, self.dev, corpus, vocab_size, config.window_size, config.min_count)
        self.instances = self.dc.cbow_instances() if self.cbow_window else None
        self.N = self.dc.n_instances if self.cbow_window else self.dc.n_pairs
        per_sample = estimate_per_sample_bytes(config.model, config.vector_size, config.negative_samples,
                                               config.window_size)
        budget = resolve_memory_budget(config)
        bsz = config.batch_size if config.batch_size is not None else suggest_batch_size(per_sample, budget, self.N)
        self.batch_size = _clamped_batch_size(bsz, per_sample, budget, config.memory_cap_fraction, events)
        self.precision = precision
        if pairs == "numpy":
            self.ref_pairs = None if self.cbow_window else self.dc.reference_pairs()
            self.perm = torch.empty(self.N, dtype=torch.int64, device=self.dev)
            self.neg_table = torch.empty(max(self.N * self.k, 1), dtype=torch.int32, device=self.dev)
            self.h_candidates = np.flatnonzero(self.dc.keep.cpu().numpy() != 0).astype(np.int64)
        else:
            self.ref_pairs = self.perm = self.neg_table = None
        dc = self.dc
        cand_identity = dc.n_candidates == self.V
        self.batch_struct = _lib.WvSgnsBatch(
            mode=_lib.PAIRS_EXPLICIT if pairs == "numpy" else _lib.PAIRS_NATIVE, negatives=self.k,
            window=int(config.window_size), model=_lib.MODEL_CBOW if self.cbow_window else _lib.MODEL_SKIPGRAM,
            batch_rows=self.batch_size, n_pairs=self.N,
            seed=self.seed & 0xFFFFFFFFFFFFFFFF, tokens=_lib.ptr(dc.tokens), offsets=_lib.ptr(dc.offsets),
            walks_by_class=_lib.ptr(dc.walks_by_class), class_len=_lib.ptr(dc.class_len),
            class_walk_start=_lib.ptr(dc.class_walk_start), class_pair_start=_lib.ptr(dc.class_pair_start),
            n_classes=dc.n_classes, candidates=None if cand_identity else _lib.ptr(dc.candidates),
            n_candidates=dc.n_candidates, pairs=_lib.ptr(self.ref_pairs), perm=_lib.ptr(self.perm),
            negative_table=_lib.ptr(self.neg_table), instances=_lib.ptr(self.instances))
        if self.k > 0 and dc.n_candidates == 0:
            raise ValueError("no negative-sample candidates")

    def decode(self, epoch: int, pos_begin: int = 0, n: int | None = None):
        """Rows [n, 2+k] (centre, context, negatives) and pair indices [n] of the epoch's
        permuted positions [pos_begin, pos_begin + n), decoded exactly as the batches
        decode them (wv_sgns_decode; skip-gram)."""
        torch = self.torch
        n = self.N - int(pos_begin) if n is None else int(n)
        rows = torch.empty((max(n, 1), 2 + self.k), dtype=torch.int32, device=self.dev)
        q = torch.empty(max(n, 1), dtype=torch.int64, device=self.dev)
        _lib.call("wv_sgns_decode", C.byref(self.batch_struct), int(epoch), int(pos_begin), n, _lib.ptr(rows),
                  _lib.ptr(q), _lib.stream_ptr())
        return rows[:n], q[:n]

    def new_params(self):
        c = self.config
        return _Params(self.torch, self.dev, self.V, c.vector_size, self.seed, self.precision, c.use_sparse,
                       c.learning_rate)

    # numpy replay of the reference streams -------------------------------
    def _upload_epoch_streams(self, order: np.ndarray, neg_rows: list[tuple[int, int, np.random.Generator]]):
        torch = self.torch
        self.perm.copy_(torch.from_numpy(order.astype(np.int64)))
        if self.k:
            negs = np.empty(self.N * self.k, dtype=np.int32)
            for lo, rows, rng in neg_rows:
                idx = rng.integers(0, len(self.h_candidates), size=rows * self.k)
                negs[lo * self.k:(lo + rows) * self.k] = self.h_candidates[idx]
            self.neg_table.copy_(torch.from_numpy(negs))

    def train_single(self):
        c = self.config
        p = self.new_params()
        rep = _Replica(self, 0, p)
        B, N = self.batch_size, self.N
        full, rem = divmod(N, B)
        losses = []
        if self.pairs_mode == "numpy":
            shuffle_rng = np.random.default_rng(np.random.SeedSequence([self.seed, 1, 1]))
            neg_rng = np.random.default_rng(np.random.SeedSequence([self.seed, 1, 2, 0]))
        for epoch in range(c.epochs):
            if self.pairs_mode == "numpy":
                order = shuffle_rng.permutation(N)
                sched = [(lo, min(B, N - lo), neg_rng) for lo in range(0, N, B)]
                self._upload_epoch_streams(order, sched)
            _lib.call("wv_sgns_epoch_begin", _lib.ptr(p.state), epoch, 0, _lib.stream_ptr())
            rep.run(full, B)
            if rem:
                rep.launch(rem)
            st = p.read_state()
            if st.diverged_batch >= 0:
                raise TrainingDiverged(int(st.diverged_epoch), int(st.diverged_batch))
            losses.append(st.epoch_loss_sum / st.epoch_count)
        return p, losses

    def train_multi(self, workers: int, exchange=None):
        """Local-replica data parallelism (w2v.py:662-746); ``exchange`` sums across ranks."""
        torch = self.torch
        c = self.config
        B, N = self.batch_size, self.N
        sync = REPRODUCIBLE_SYNC_BATCHES if c.reproducible else self._sync_batches_estimate()
        span = -(-N // workers)
        batches_per_worker = -(-span // B)
        rounds = max(1, -(-batches_per_worker // sync))
        local = exchange is None
        widxs = list(range(workers)) if local else [exchange.rank]
        reps = []
        touched_in = torch.zeros(self.V, dtype=torch.uint8, device=self.dev)
        touched_out = torch.zeros(self.V, dtype=torch.uint8, device=self.dev)
        for w in widxs:
            p = self.new_params()
            # kernels mark per-round touches; they are folded into p.touched_* each round
            p.struct.touched_in = _lib.ptr(touched_in)
            p.struct.touched_out = _lib.ptr(touched_out)
            reps.append(_Replica(self, w, p))
        n_el = self.V * c.vector_size
        snap_in = reps[0].p.inp.clone()
        snap_out = reps[0].p.out.clone()
        delta = torch.empty(n_el, dtype=reps[0].p.dtype, device=self.dev)
        delta_sum_in = torch.zeros_like(delta)
        delta_sum_out = torch.zeros_like(delta)
        cnt_in = torch.zeros(self.V, dtype=torch.float32, device=self.dev)
        cnt_out = torch.zeros(self.V, dtype=torch.float32, device=self.dev)
        if self.pairs_mode == "numpy":
            shuffle_rng = np.random.default_rng(np.random.SeedSequence([self.seed, 1, 1]))
            neg_rngs = {w: np.random.default_rng(np.random.SeedSequence([self.seed, 1, 2, w])) for w in
                        range(workers)}
        losses = []
        st = _lib.stream_ptr()
        for epoch in range(c.epochs):
            if self.pairs_mode == "numpy":
                order = shuffle_rng.permutation(N)
                sched = []
                for w in range(workers):
                    lo_w, hi_w = w * span, min((w + 1) * span, N)
                    sched += [(lo, min(B, hi_w - lo), neg_rngs[w]) for lo in range(lo_w, hi_w, B)]
                self._upload_epoch_streams(order, sched)
            for r in reps:
                _lib.call("wv_sgns_epoch_begin", _lib.ptr(r.p.state), epoch, min(r.widx * span, N), st)
            done = {r.widx: 0 for r in reps}
            for _ in range(rounds):
                delta_sum_in.zero_()
                delta_sum_out.zero_()
                cnt_in.zero_()
                cnt_out.zero_()
                for r in reps:
                    lo_w, hi_w = min(r.widx * span, N), min((r.widx + 1) * span, N)
                    mine = -(-(hi_w - lo_w) // B)
                    todo = min(sync, mine - done[r.widx])
                    if todo > 0:
                        last_lo = lo_w + (done[r.widx] + todo - 1) * B
                        last_rows = min(B, hi_w - last_lo)
                        r.run(todo - 1 if last_rows < B else todo, B)
                        if last_rows < B:
                            r.launch(last_rows)
                        done[r.widx] += todo
                    _lib.call("wv_replica_delta", _lib.ptr(r.p.inp), _lib.ptr(snap_in), n_el, r.p.precision,
                              _lib.ptr(delta), st)
                    delta_sum_in += delta
                    _lib.call("wv_replica_delta", _lib.ptr(r.p.out), _lib.ptr(snap_out), n_el, r.p.precision,
                              _lib.ptr(delta), st)
                    delta_sum_out += delta
                    cnt_in += touched_in.float()
                    cnt_out += touched_out.float()
                    r.p.touched_in |= touched_in
                    r.p.touched_out |= touched_out
                    touched_in.zero_()
                    touched_out.zero_()
                if exchange is not None:
                    self.last_merge = exchange.merge_deltas_((delta_sum_in, delta_sum_out), (cnt_in, cnt_out),
                                                             c.vector_size)
                # every replica applies the same merge -> identical union rows
                for i, r in enumerate(reps):
                    last = i == len(reps) - 1
                    s_in = snap_in if last else snap_in.clone()
                    s_out = snap_out if last else snap_out.clone()
                    _lib.call("wv_replica_apply", _lib.ptr(r.p.inp), _lib.ptr(s_in), _lib.ptr(delta_sum_in),
                              _lib.ptr(cnt_in), self.V, c.vector_size, r.p.precision, st)
                    _lib.call("wv_replica_apply", _lib.ptr(r.p.out), _lib.ptr(s_out), _lib.ptr(delta_sum_out),
                              _lib.ptr(cnt_out), self.V, c.vector_size, r.p.precision, st)
            loss_sum, count, div = 0.0, 0, None
            for r in reps:
                s = r.p.read_state()
                loss_sum += s.epoch_loss_sum
                count += s.epoch_count
                if s.diverged_batch >= 0 and div is None:
                    div = (int(s.diverged_epoch), int(s.diverged_batch))
            if exchange is not None:
                loss_sum, count, div = exchange.reduce_epoch(loss_sum, count, div)
            if div is not None:
                raise TrainingDiverged(*div)
            losses.append(float(loss_sum / count) if count else float("nan"))
        p0 = reps[0].p
        for r in reps[1:]:
            p0.modified_in |= r.p.modified_in
            p0.modified_out |= r.p.modified_out
            p0.touched_in |= r.p.touched_in
            p0.touched_out |= r.p.touched_out
        if exchange is not None:
            exchange.or_flags_(p0.modified_in, p0.modified_out, p0.touched_in, p0.touched_out)
        return p0, losses

    def _sync_batches_estimate(self) -> int:
        """Batches per sync_interval_ms (w2v.py:628-639), from the HBM bytes one batch moves."""
        c = self.config
        es = 8 if self.precision == "fp64" else 4
        rows = self.batch_size * ((2 * self.cbow_window + 1 + self.k) if self.cbow_window else (2 + self.k))
        batch_bytes = rows * c.vector_size * es * 2 + min(rows, 2 * self.V) * c.vector_size * es * 8
        est_ms = max(batch_bytes / 3.0e12 * 1e3, 0.02)
        return max(1, min(int(round(c.sync_interval_ms / est_ms)), 1 << 14))


class SkipGramSession:
    """Persistent SGNS state trained over a sequence of corpora (streaming ``train``).

    One parameter store and its RowAdam state stay resident in HBM while
    corpora arrive -- e.g. the walks of successive root blocks of a graph too
    large to walk in one piece.  Each ``fit`` runs ``epochs`` passes over that
    corpus's pairs with train()'s batch rule, kernels and numerics
    (w2v.py:547-576).  Negatives are drawn uniformly over the whole
    vocabulary: min_count filtering needs global frequencies, which one block
    does not have (with walk_number >= min_count every root token passes
    anyway).  Epoch streams (Feistel permutation key, Philox
    negatives) advance with a session-wide epoch counter.
    """

    def __init__(self, vocab_size: int, config: TrainConfig, rng_seed: int, *, precision: str = "fp32",
                 graph_batches: int = 64, device=None, on_event=None):
        if config.model != SKIPGRAM:
            raise NotImplementedError("the B200 backend implements model='skipgram'")
        if precision not in ("fp32", "fp64"):
            raise ValueError("precision must be 'fp32' or 'fp64'")
        torch = _lib.require_cuda()
        self.torch = torch
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.config = config
        self.V = int(vocab_size)
        self.seed = int(rng_seed)
        self.precision = precision
        self.graph_batches = int(graph_batches)
        self.events = on_event or (lambda kind, **info: None)
        self.params = _Params(torch, self.dev, self.V, config.vector_size, self.seed, precision, config.use_sparse,
                              config.learning_rate)
        self.epochs_done = 0
        self.pairs_done = 0
        self.batches_done = 0
        self.last_batch_size = 0
        self.last_replica = None
        self.exchange = None

    def attach_exchange(self, exchange):
        """Join a data-parallel group: sync() then averages per-row deltas across ranks
        (_merge_bundles semantics, w2v.py:642-659) every time it is called."""
        torch, p = self.torch, self.params
        self.exchange = exchange
        self._round_in = torch.zeros(self.V, dtype=torch.uint8, device=self.dev)
        self._round_out = torch.zeros(self.V, dtype=torch.uint8, device=self.dev)
        p.struct.touched_in = _lib.ptr(self._round_in)
        p.struct.touched_out = _lib.ptr(self._round_out)
        self._snap_in = p.inp.clone()
        self._snap_out = p.out.clone()
        self._delta_in = torch.empty_like(p.inp)
        self._delta_out = torch.empty_like(p.out)
        self._cnt_in = torch.empty(self.V, dtype=torch.float32, device=self.dev)
        self._cnt_out = torch.empty(self.V, dtype=torch.float32, device=self.dev)

    def sync(self):
        """One replica-averaging round over the attached exchange (one all-reduce of deltas + counts)."""
        if self.exchange is None:
            return
        p, st = self.params, _lib.stream_ptr()
        n_el = self.V * self.config.vector_size
        _lib.call("wv_replica_delta", _lib.ptr(p.inp), _lib.ptr(self._snap_in), n_el, p.precision,
                  _lib.ptr(self._delta_in), st)
        _lib.call("wv_replica_delta", _lib.ptr(p.out), _lib.ptr(self._snap_out), n_el, p.precision,
                  _lib.ptr(self._delta_out), st)
        self._cnt_in.copy_(self._round_in)
        self._cnt_out.copy_(self._round_out)
        p.touched_in |= self._round_in
        p.touched_out |= self._round_out
        self._round_in.zero_()
        self._round_out.zero_()
        self.last_merge = self.exchange.merge_deltas_((self._delta_in, self._delta_out),
                                                      (self._cnt_in, self._cnt_out), self.config.vector_size)
        _lib.call("wv_replica_apply", _lib.ptr(p.inp), _lib.ptr(self._snap_in), _lib.ptr(self._delta_in),
                  _lib.ptr(self._cnt_in), self.V, self.config.vector_size, p.precision, st)
        _lib.call("wv_replica_apply", _lib.ptr(p.out), _lib.ptr(self._snap_out), _lib.ptr(self._delta_out),
                  _lib.ptr(self._cnt_out), self.V, self.config.vector_size, p.precision, st)

    def fit(self, corpus, epochs: int = 1, *, profile: bool = False) -> list[float]:
        """Train ``epochs`` passes over ``corpus``; returns the per-epoch mean losses."""
        from dataclasses import replace

        cfg = replace(self.config, min_count=0, epochs=int(epochs), workers=1)
        tr = _Trainer(corpus, self.V, cfg, self.seed, self.events, self.precision, "device", self.graph_batches,
                      device=self.dev)
        tr.profile = profile
        rep = self.last_replica
        if rep is not None and rep.compatible(tr):
            rep.retarget(tr)
        else:
            rep = _Replica(tr, 0, self.params)
        self.last_replica = rep
        B, N = tr.batch_size, tr.N
        full, rem = divmod(N, B)
        p = self.params
        losses = []
        for _ in range(int(epochs)):
            _lib.call("wv_sgns_epoch_begin", _lib.ptr(p.state), self.epochs_done, 0, _lib.stream_ptr())
            rep.run(full, B)
            if rem:
                rep.launch(rem)
            st = p.read_state()
            if st.diverged_batch >= 0:
                raise TrainingDiverged(int(st.diverged_epoch), int(st.diverged_batch))
            losses.append(st.epoch_loss_sum / st.epoch_count)
            self.epochs_done += 1
            self.pairs_done += N
            self.batches_done += full + (1 if rem else 0)
        self.last_batch_size = B
        self.last_pairs = N
        return losses

    def rows_updated(self) -> int:
        """Cumulative unique (row, matrix) Adam updates (telemetry for the roofline)."""
        return int(self.params.read_state().rows_updated)

    @property
    def model(self) -> EmbeddingModel:
        return EmbeddingModel(self.params, self.config.vector_size, np.ones(self.V, dtype=bool))


def train(corpus, vocab_size: int, config: TrainConfig, rng_seed: int, on_event=None, *, precision: str = "fp32",
          pairs: str = "device", graph_batches: int = 64, exchange=None):
    """Run SGNS over the corpus on the device; returns (EmbeddingModel, per-epoch losses).

    Signature-compatible with walkvec.w2v.train (w2v.py:507-544) plus:
      precision      "fp32" (default) or "fp64" parameter store
      pairs          "device" (Feistel/Philox on the device) or "numpy"
                     (replay the reference's own numpy streams)
      graph_batches  batches captured per CUDA graph
      exchange       a dist.RankExchange for multi-GPU data parallelism
    """
    if precision not in ("fp32", "fp64"):
        raise ValueError("precision must be 'fp32' or 'fp64'")
    if pairs not in ("device", "numpy"):
        raise ValueError("pairs must be 'device' or 'numpy'")
    events = on_event or (lambda kind, **info: None)
    tr = _Trainer(corpus, vocab_size, config, rng_seed, events, precision, pairs, graph_batches)
    if exchange is not None:
        params, losses = tr.train_multi(exchange.world_size, exchange)
    elif config.workers == 1:
        params, losses = tr.train_single()
    else:
        params, losses = tr.train_multi(config.workers)
    keep = tr.dc.keep.cpu().numpy().astype(bool)
    model = EmbeddingModel(params, config.vector_size, keep.copy())
    model.n_pairs = tr.N
    model.batch_size = tr.batch_size
    return model, losses
