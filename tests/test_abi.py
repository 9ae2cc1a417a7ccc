"""C-ABI library: loads without a GPU, exports every declared symbol, host-side RNG helpers."""

import ctypes as C
import json
import re

import numpy as np

from conftest import ROOT
from paper_2508_01073_b200 import _lib
from paper_2508_01073_b200.seeding import entropy_words, words_array

HEADER = ROOT / "include" / "walkvec_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(wv_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)
    assert lib.wv_abi_version() == _lib.ABI_VERSION


def test_struct_layouts_match_header():
    lib = _lib.load()
    for i, st in enumerate((_lib.WvSgnsDevState, _lib.WvSgnsModel, _lib.WvSgnsBatch)):
        assert lib.wv_struct_size(i) == C.sizeof(st), st
    for st in (_lib.WvSgnsDevState, _lib.WvSgnsModel, _lib.WvSgnsBatch):
        assert C.sizeof(st) % 8 == 0


def test_host_seedseq_matches_numpy(golden):
    g = golden("seedseq.npz")
    for i, e in enumerate(json.loads(str(g["entropies"]))):
        words = entropy_words(e[:-1])
        arr, n = words_array(words)
        out = (C.c_uint64 * 4)()
        _lib.call("wv_seedseq_generate", arr, n, e[-1], 4, out)
        assert list(out) == [int(x) for x in g[f"state4_{i}"]]


def test_host_stream_elements_match_numpy(golden):
    g = golden("seedseq.npz")
    for i, e in enumerate(json.loads(str(g["entropies"]))):
        arr, n = words_array(entropy_words(e[:-1]))
        for kind, tag, ks in ((_lib.RNG_PCG64, "pcg", [0, 1, 2, 3, 999, 1000, 1099]),
                              (_lib.RNG_PHILOX, "philox", [0, 1, 2, 3, 4, 5, 999, 1000, 1099])):
            for k, want in zip(ks, g[f"{tag}_{i}"]):
                out = C.c_uint64()
                _lib.call("wv_stream_u64", arr, n, e[-1], kind, k, C.byref(out))
                assert out.value == int(want)


def test_error_path_sets_message():
    out = C.c_uint64()
    arr, n = words_array([1])
    try:
        _lib.call("wv_stream_u64", arr, n, 0, 7, 0, C.byref(out))
    except ValueError as err:
        assert "unknown rng kind" in str(err)
    else:
        raise AssertionError("expected ValueError")


def test_compute_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        return
    from paper_2508_01073_b200 import BackendUnavailable, build_graph

    try:
        build_graph(np.array([[0, 1, 2]]), 3)
    except BackendUnavailable:
        pass
    else:
        raise AssertionError("expected BackendUnavailable without a GPU")
