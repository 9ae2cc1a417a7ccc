"""Re-point a loaded reference ``walkvec`` package at the B200 backend.

The reference has no plugin registry: its call sites reach the
hot path through module attributes -- pipeline.extract_walks ->
walks_mod.random_walks / bfs_walks (pipeline.py:20, 167, 178), and
``train`` imported by name into pipeline (pipeline.py:23, 211), cli
(cli.py:21, 169) and re-exported from the package.  install() swaps exactly
those attributes, plus ``load_data`` (pipeline.py:117, cli.py:103; GPU ingest)
and the artifact writers save_embeddings_text / _tsv and save_corpus_binary
(device-formatted, byte-identical files) and load_corpus_binary (device parse);
uninstall() restores them.
"""

from __future__ import annotations

import importlib

_saved: dict = {}
_saved_methods: dict = {}


def _wrap_train(train_fn, precision: str, pairs: str, package: str):
    def train(corpus, vocab_size, config, rng_seed, on_event=None):
        from .w2v import TrainConfig, TrainingDiverged

        cfg = TrainConfig(**{f: getattr(config, f) for f in TrainConfig.__dataclass_fields__})
        try:
            model, losses = train_fn(corpus, vocab_size, cfg, rng_seed, on_event=on_event, precision=precision,
                                     pairs=pairs)
        except TrainingDiverged as err:
            # the caller catches the reference's own type (w2v.py:46-52; pipeline.py wraps it in PipelineError)
            ref_type = importlib.import_module(f"{package}.w2v").TrainingDiverged
            raise ref_type(err.epoch, err.batch) from err
        return model, losses

    train.__doc__ = f"walkvec.w2v.train on the B200 backend (precision={precision!r}, pairs={pairs!r})"
    return train


def _wrap_load_data(load_fn, pkg_name: str):
    """Device ingest, returning the reference's own Vocabulary type (save_tsv etc.)."""

    def load_data(path, format=None, include_literals=False, strict=False, has_header=False, error_sink=None):
        ref_ingest = importlib.import_module(f"{pkg_name}.ingest")
        ref_pipe = importlib.import_module(f"{pkg_name}.pipeline")
        from .pipeline import PipelineError

        try:
            vocab, edges = load_fn(path, format=format, include_literals=include_literals, strict=strict,
                                   has_header=has_header, error_sink=error_sink)
        except PipelineError as err:
            raise ref_pipe.PipelineError("ingest", err.__cause__ or err) from err
        ref = ref_ingest.Vocabulary()
        ref.lexical_of = list(vocab.lexical_of)
        ref.token_of = {s_: i for i, s_ in enumerate(ref.lexical_of)}
        ref._entity_tokens = set(vocab.entity_tokens().tolist())
        ref._predicate_tokens = set(vocab._predicate_tokens)
        return ref, edges

    return load_data


def install(package: str = "walkvec", *, precision: str = "fp64", pairs: str = "device"):
    """Swap the reference's hot-path functions for the device implementations.

    ``precision`` is the parameter store of the swapped ``train``: "fp64" (the
    default: the reference's own arithmetic, w2v.py:127-130, 379-380) or "fp32"
    (half the HBM bytes, tolerance-checked).  ``pairs`` is its pair/negative
    source: "device" (Feistel permutation + Philox negatives, nothing
    materialised on the host) or "numpy" (replays the reference's own numpy
    streams: the same pairs, order and negatives as the reference's train()).
    """
    if precision not in ("fp64", "fp32"):
        raise ValueError("precision must be 'fp64' or 'fp32'")
    if pairs not in ("device", "numpy"):
        raise ValueError("pairs must be 'device' or 'numpy'")
    from . import formats as dev_formats
    from . import walks as dev_walks
    from .pipeline import load_data as dev_load_data
    from .w2v import train as dev_train

    pkg = importlib.import_module(package)
    walks_mod = importlib.import_module(f"{package}.walks")
    w2v_mod = importlib.import_module(f"{package}.w2v")
    pipe_mod = importlib.import_module(f"{package}.pipeline")
    targets = [
        (walks_mod, "random_walks", dev_walks.random_walks),
        (walks_mod, "bfs_walks", dev_walks.bfs_walks),
        (pkg, "random_walks", dev_walks.random_walks),
        (pkg, "bfs_walks", dev_walks.bfs_walks),
        (w2v_mod, "train", _wrap_train(dev_train, precision, pairs, package)),
        (pipe_mod, "train", _wrap_train(dev_train, precision, pairs, package)),
        (pkg, "train", _wrap_train(dev_train, precision, pairs, package)),
        (pipe_mod, "load_data", _wrap_load_data(dev_load_data, package)),
        (pipe_mod, "save_embeddings_text", dev_formats.save_embeddings_text),
        (pipe_mod, "save_embeddings_tsv", dev_formats.save_embeddings_tsv),
        (walks_mod, "save_corpus_binary", dev_formats.save_corpus_binary),
        (walks_mod, "load_corpus_binary", dev_formats.load_corpus_binary),
        (pkg, "save_corpus_binary", dev_formats.save_corpus_binary),
        (pkg, "load_corpus_binary", dev_formats.load_corpus_binary),
        (pkg, "load_data", _wrap_load_data(dev_load_data, package)),
    ]
    try:
        cli_mod = importlib.import_module(f"{package}.cli")
        targets.append((cli_mod, "train", _wrap_train(dev_train, precision, pairs, package)))
    except ImportError:
        pass
    for mod, name, fn in targets:
        _saved.setdefault((mod.__name__, name), getattr(mod, name))
        setattr(mod, name, fn)
    # Vocabulary.save_tsv is a method (cli.py:116, pipeline.py:302): swap it on the class
    ingest_mod = importlib.import_module(f"{package}.ingest")
    _saved_methods.setdefault((ingest_mod.__name__, "Vocabulary", "save_tsv"), ingest_mod.Vocabulary.save_tsv)
    ingest_mod.Vocabulary.save_tsv = lambda self, path: dev_formats.save_vocabulary_tsv(self, path)


def uninstall():
    for (modname, name), fn in list(_saved.items()):
        setattr(importlib.import_module(modname), name, fn)
    _saved.clear()
    for (modname, cls, name), fn in list(_saved_methods.items()):
        setattr(getattr(importlib.import_module(modname), cls), name, fn)
    _saved_methods.clear()
