"""Pipeline boundary (drop-in for walkvec.pipeline.extract_walks / fit_transform).

Reference: pkg/src/walkvec/pipeline.py:39-219.  Stage order, error wrapping
(PipelineError(stage)) and timings are the reference's; the stages run on
the device.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import walks as walks_mod
from .graph import build_graph
from .w2v import CBOW, SKIPGRAM, TrainConfig, train
from .walks import BFS, ENTITY, FULL, PROPERTY, RANDOM, WalkCorpus


class PipelineError(RuntimeError):
    """A stage failure; ``stage`` names the stage that raised (pipeline.py:30-36)."""

    def __init__(self, stage: str, cause: BaseException):
        super().__init__(f"{stage}: {cause}")
        self.stage = stage
        self.cause = cause


@dataclass
class PipelineConfig:
    """All pipeline hyperparameters with the reference defaults (pipeline.py:39-104)."""

    walk_strategy: str = RANDOM
    walk_depth: int = 5
    walk_number: int = 100
    embedding_model: str = SKIPGRAM
    epochs: int = 5
    batch_size: int | None = None
    vector_size: int = 100
    window_size: int = 5
    min_count: int = 10
    learning_rate: float = 0.01
    negative_samples: int = 5
    random_state: int = 42
    reproducible: bool = False
    workers: int = 1
    generate_artifact: bool = False
    projection: str = FULL
    duplicate_free: bool = False
    include_literals: bool = False
    strict: bool = False
    sync_interval_ms: int = 500
    memory_budget_bytes: int | None = None
    memory_cap_fraction: float = 0.9
    use_sparse: bool = True

    def __post_init__(self):
        if self.walk_strategy not in (RANDOM, BFS):
            raise ValueError(f"walk_strategy must be 'random' or 'bfs', got {self.walk_strategy!r}")
        if self.embedding_model not in (SKIPGRAM, CBOW):
            raise ValueError(f"embedding_model must be 'skipgram' or 'cbow', got {self.embedding_model!r}")
        if self.projection not in (FULL, ENTITY, PROPERTY):
            raise ValueError(f"projection must be full/entity/property, got {self.projection!r}")
        for name in ("walk_depth", "walk_number", "epochs", "vector_size", "window_size", "workers"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1")
        if self.min_count < 0:
            raise ValueError("min_count must be >= 0")
        if self.negative_samples < 0:
            raise ValueError("negative_samples must be >= 0")
        if self.random_state < 0:
            raise ValueError("random_state must be >= 0")
        if self.batch_size is not None and self.batch_size < 1:
            raise ValueError("batch_size must be >= 1 or None")

    def train_config(self) -> TrainConfig:
        return TrainConfig(model=self.embedding_model, epochs=self.epochs, window_size=self.window_size,
                           negative_samples=self.negative_samples, learning_rate=self.learning_rate,
                           min_count=self.min_count, vector_size=self.vector_size, batch_size=self.batch_size,
                           sync_interval_ms=self.sync_interval_ms, memory_budget_bytes=self.memory_budget_bytes,
                           memory_cap_fraction=self.memory_cap_fraction, use_sparse=self.use_sparse,
                           workers=self.workers, reproducible=self.reproducible)


class EmbeddingTable:
    """|vocab| x d rows keyed by lexical token (pipeline.py:140-161)."""

    def __init__(self, vocab, vectors, trained_mask, losses, timings=None, model=None):
        self.vocab = vocab
        self._vectors = vectors
        self._model = model
        self.trained_mask = trained_mask
        self.losses = losses
        self.timings = timings or {}

    @property
    def vectors(self) -> np.ndarray:
        if self._vectors is None:
            self._vectors = self._model.input_matrix
        return self._vectors

    def __len__(self) -> int:
        return self.vectors.shape[0]

    def __contains__(self, lexical: str) -> bool:
        return lexical in self.vocab.token_of

    def __getitem__(self, lexical: str) -> np.ndarray:
        return self.vectors[self.vocab.token_of[lexical]]

    def as_dict(self) -> dict:
        return {lex: self.vectors[tok] for lex, tok in self.vocab.token_of.items()}


_FORMATS = ("nt", "csv", "tsv", "txt")
_UNSUPPORTED = {".parquet": "parquet", ".orc": "orc"}


def detect_format(path) -> str:
    """File format from the extension (pipeline.py:107-114)."""
    from pathlib import Path

    suffix = Path(path).suffix.lower()
    if suffix in _UNSUPPORTED:
        raise ValueError(f"format unsupported: {_UNSUPPORTED[suffix]}")
    mapped = {".nt": "nt", ".csv": "csv", ".tsv": "tsv", ".txt": "txt"}.get(suffix)
    if mapped is None:
        raise ValueError(f"cannot infer format from {suffix!r}; pass format explicitly")
    return mapped


def load_data(path, format: str | None = None, include_literals: bool = False, strict: bool = False,
              has_header: bool = False, error_sink: list | None = None):
    """Parse and tokenize an input file on the GPU: (vocabulary, edges) (pipeline.py:117-135).

    The file's bytes go to the device once; lines are parsed and keys interned
    by first occurrence there (``ingest.load_triples_device``).  Errors are the
    reference's: ValueError for formats, ParseError / ValueError from parsing,
    wrapped as ``PipelineError("ingest", ...)``.
    """
    from .ingest import load_triples_device

    if format is None:
        format = detect_format(path)
    if format not in _FORMATS:
        if format in _UNSUPPORTED.values():
            raise ValueError(f"format unsupported: {format}")
        raise ValueError(f"unknown format: {format!r}")
    try:
        return load_triples_device(path, format, strict=strict, error_sink=error_sink,
                                   include_literals=include_literals, has_header=has_header)
    except (ValueError, OSError) as err:
        raise PipelineError("ingest", err) from err


def extract_walks(graph, roots, config: PipelineConfig, *, rng: str = "pcg64",
                  max_walks_per_root: int | None = None) -> WalkCorpus:
    """Configured walk strategy + projection (pipeline.py:164-179)."""
    if config.walk_strategy == RANDOM:
        corpus = walks_mod.random_walks(graph, start_vertices=roots, walk_depth=config.walk_depth,
                                        walk_number=config.walk_number, rng_seed=config.random_state,
                                        duplicate_free=config.duplicate_free, workers=config.workers, rng=rng)
    else:
        corpus, _ = walks_mod.bfs_walks(graph, start_vertices=roots, walk_depth=config.walk_depth,
                                        max_walks_per_root=max_walks_per_root, with_table=False)
    return walks_mod.project_corpus(corpus, config.projection)


def _sync():
    torch = _lib.require_cuda()
    torch.cuda.synchronize()


def fit_transform(edges, vocab, config: PipelineConfig, walk_vertices=None, on_event=None, *,
                  rng: str = "pcg64", precision: str = "fp32", pairs: str = "device",
                  max_walks_per_root: int | None = None) -> EmbeddingTable:
    """Graph build, walk extraction and training in one call (pipeline.py:182-219)."""
    if len(edges) == 0:
        raise PipelineError("graph", ValueError("no edges to embed"))
    timings: dict[str, float] = {}
    try:
        start = time.perf_counter()
        graph = build_graph(edges, len(vocab))
        _sync()
        timings["graph_s"] = time.perf_counter() - start
    except ValueError as err:
        raise PipelineError("graph", err) from err
    try:
        roots = vocab.entity_tokens() if walk_vertices is None else walk_vertices
        start = time.perf_counter()
        corpus = extract_walks(graph, roots, config, rng=rng, max_walks_per_root=max_walks_per_root)
        _sync()
        timings["walks_s"] = time.perf_counter() - start
    except ValueError as err:
        raise PipelineError("walks", err) from err
    try:
        start = time.perf_counter()
        model, losses = train(corpus, len(vocab), config.train_config(), config.random_state, on_event=on_event,
                              precision=precision, pairs=pairs)
        _sync()
        timings["train_s"] = time.perf_counter() - start
    except (ValueError, RuntimeError) as err:
        raise PipelineError("train", err) from err
    torch = _lib.require_cuda()
    tok, _ = corpus.device_arrays()
    freq = torch.zeros(len(vocab), dtype=torch.int64, device=tok.device)
    _lib.call("wv_token_histogram", _lib.ptr(tok), corpus.total_tokens, len(vocab), _lib.ptr(freq), 0,
              _lib.stream_ptr())
    vocab.frequency = freq.cpu().numpy()
    return EmbeddingTable(vocab, None, model.trained_mask, losses, timings, model=model)
