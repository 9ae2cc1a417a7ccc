"""Re-point a loaded reference ``walkvec`` package at the B200 backend.

The reference has no plugin registry: its call sites reach the
hot path through module attributes -- pipeline.extract_walks ->
walks_mod.random_walks / bfs_walks (pipeline.py:20, 167, 178), and
``train`` imported by name into pipeline (pipeline.py:23, 211), cli
(cli.py:21, 169) and re-exported from the package.  install() swaps exactly
those attributes; uninstall() restores them.
"""

from __future__ import annotations

import importlib

_saved: dict = {}


def _wrap_train(train_fn):
    def train(corpus, vocab_size, config, rng_seed, on_event=None):
        from .w2v import TrainConfig

        cfg = TrainConfig(**{f: getattr(config, f) for f in TrainConfig.__dataclass_fields__})
        model, losses = train_fn(corpus, vocab_size, cfg, rng_seed, on_event=on_event)
        return model, losses

    return train


def install(package: str = "walkvec"):
    """Swap the reference's hot-path functions for the device implementations."""
    from . import walks as dev_walks
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
        (w2v_mod, "train", _wrap_train(dev_train)),
        (pipe_mod, "train", _wrap_train(dev_train)),
        (pkg, "train", _wrap_train(dev_train)),
    ]
    try:
        cli_mod = importlib.import_module(f"{package}.cli")
        targets.append((cli_mod, "train", _wrap_train(dev_train)))
    except ImportError:
        pass
    for mod, name, fn in targets:
        _saved.setdefault((mod.__name__, name), getattr(mod, name))
        setattr(mod, name, fn)


def uninstall():
    for (modname, name), fn in list(_saved.items()):
        setattr(importlib.import_module(modname), name, fn)
    _saved.clear()
