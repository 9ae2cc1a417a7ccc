"""paper_2508_01073_b200: B200-native (sm_100a) RDF2vec hot path.

Drop-in for the reference walkvec package's hot path (random / BFS walk
extraction, SGNS training, and the graph / pipeline calls around them).
Compute runs in libwalkvec_b200.so (hand-written CUDA behind a C ABI,
include/walkvec_b200.h); there is no CPU fallback.

    from paper_2508_01073_b200 import PipelineConfig, fit_transform
    table = fit_transform(edges, vocab, PipelineConfig(walk_depth=4, walk_number=25))

``install()`` re-points a loaded reference ``walkvec`` package at this
backend (random_walks, bfs_walks, train, build_graph, extract_walks).
"""

from ._lib import BackendUnavailable
from . import formats
from .graph import Graph, build_graph
from .ingest import PAD, ParseError, Vocabulary, build_vocabulary, encode_integer_triples, load_triples_device
from .install import install, uninstall
from .pipeline import (EmbeddingTable, PipelineConfig, PipelineError, detect_format, extract_walks, fit_transform,
                       load_data)
from .w2v import (
    CBOW,
    SKIPGRAM,
    EmbeddingModel,
    SkipGramSession,
    TrainConfig,
    TrainingDiverged,
    estimate_per_sample_bytes,
    generate_cbow_instances,
    generate_pairs,
    init_embeddings,
    resolve_memory_budget,
    suggest_batch_size,
    train,
)
from .walks import (
    BFS,
    ENTITY,
    FULL,
    PROPERTY,
    RANDOM,
    SHARD_SIZE,
    PathTable,
    Walk,
    WalkCorpus,
    bfs_walks,
    project_corpus,
    project_entity,
    project_property,
    random_walks,
)

__version__ = "0.1.0"

__all__ = [
    "BFS", "CBOW", "ENTITY", "FULL", "PAD", "PROPERTY", "RANDOM", "SHARD_SIZE", "SKIPGRAM",
    "BackendUnavailable", "EmbeddingModel", "EmbeddingTable", "Graph", "PathTable", "PipelineConfig",
    "PipelineError", "SkipGramSession", "TrainConfig", "TrainingDiverged", "Vocabulary", "Walk", "WalkCorpus",
    "ParseError", "bfs_walks", "build_graph", "build_vocabulary", "detect_format", "load_data", "load_triples_device", "encode_integer_triples", "estimate_per_sample_bytes",
    "extract_walks", "fit_transform", "generate_cbow_instances", "generate_pairs", "init_embeddings", "install", "project_corpus",
    "project_entity", "project_property", "random_walks", "resolve_memory_budget", "suggest_batch_size",
    "train", "uninstall",
]
