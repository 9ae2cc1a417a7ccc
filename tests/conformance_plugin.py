"""pytest plugin: the reference's own test-suite against the B200 backend.

Loaded with ``-p conformance_plugin`` by tests/test_gpu_conformance.py around
the UNMODIFIED reference tests in baseline/_ref/walkvec_tests.  Before any test
module is imported it puts baseline/_ref first on sys.path, imports the
reference package ``walkvec`` and calls ``install()``, which re-points the
reference's hot-path attributes (walks.random_walks / bfs_walks, w2v.train and
its imports in pipeline / cli / the package, load_data, the writers) at the
device implementations.  Every swapped function is wrapped with a call counter,
written as JSON to $WV_CONFORMANCE_CALLS at exit, so the caller can prove the
backend -- not the reference -- ran.  $WV_CONFORMANCE = "<precision>:<pairs>".
"""

from __future__ import annotations

import functools
import importlib
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"
CALLS: dict[str, int] = {}


def _counted(fn, key):
    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        CALLS[key] = CALLS.get(key, 0) + 1
        return fn(*args, **kwargs)

    return wrapper


def pytest_configure(config):
    for p in (str(ROOT), str(REF)):
        if p not in sys.path:
            sys.path.insert(0, p)
    import walkvec  # noqa: F401  (the reference, from baseline/_ref)

    install = importlib.import_module("paper_2508_01073_b200.install")

    precision, pairs = os.environ.get("WV_CONFORMANCE", "fp64:device").split(":")
    install.install("walkvec", precision=precision, pairs=pairs)
    for modname, name in list(install._saved):
        mod = importlib.import_module(modname)
        setattr(mod, name, _counted(getattr(mod, name), f"{modname}.{name}"))


def pytest_unconfigure(config):
    out = os.environ.get("WV_CONFORMANCE_CALLS")
    if out:
        Path(out).write_text(json.dumps(CALLS, indent=1, sort_keys=True))
