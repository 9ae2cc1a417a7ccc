"""ctypes binding of libwalkvec_b200.so (the C ABI declared in include/walkvec_b200.h).

The library is the only compute path: there is no CPU fallback.  Loading it
needs no GPU (the CPU test-suite checks the exported symbols); any compute
call without a CUDA device raises ``BackendUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

_PKG = Path(__file__).resolve().parent
# WV_LIB overrides the in-tree library (A/B builds of kernel variants)
LIB_PATH = Path(os.environ["WV_LIB"]) if os.environ.get("WV_LIB") else _PKG / "libwalkvec_b200.so"

RNG_PCG64 = 0
RNG_PHILOX = 1
KEEP_ENTITY = 0
KEEP_PROPERTY = 1
KEEP_TOKENS = 2
FP32 = 0
FP64 = 1
PAIRS_NATIVE = 0
PAIRS_EXPLICIT = 1
MODEL_SKIPGRAM, MODEL_CBOW = 0, 1
PHASE_PAIRS, PHASE_GROUP, PHASE_UPDATE, PHASE_ALL = 1, 2, 4, 7
ABI_VERSION = 1


class BackendUnavailable(RuntimeError):
    """The sm_100a library or a CUDA device is missing (no silent fallback)."""


class WvError(RuntimeError):
    """A non-zero status from the C ABI."""


class WvSgnsDevState(C.Structure):
    _fields_ = [
        ("lo", C.c_int64),
        ("epoch", C.c_int64),
        ("batch", C.c_int64),
        ("step", C.c_int64),
        ("epoch_loss_sum", C.c_double),
        ("epoch_count", C.c_int64),
        ("diverged_epoch", C.c_int64),
        ("diverged_batch", C.c_int64),
        ("last_batch_loss", C.c_double),
        ("block_counter", C.c_uint32),
        ("pad", C.c_uint32),
        ("rows_updated", C.c_int64),
    ]


class WvSgnsModel(C.Structure):
    _fields_ = [
        ("vocab_size", C.c_int64),
        ("vector_size", C.c_int),
        ("precision", C.c_int),
        ("sparse", C.c_int),
        ("pad", C.c_int),
        ("learning_rate", C.c_double),
        ("input", C.c_void_p),
        ("output", C.c_void_p),
        ("m_in", C.c_void_p),
        ("v_in", C.c_void_p),
        ("m_out", C.c_void_p),
        ("v_out", C.c_void_p),
        ("steps_in", C.c_void_p),
        ("steps_out", C.c_void_p),
        ("touched_in", C.c_void_p),
        ("touched_out", C.c_void_p),
        ("modified_in", C.c_void_p),
        ("modified_out", C.c_void_p),
        ("dense_g_in", C.c_void_p),
        ("dense_g_out", C.c_void_p),
        ("state", C.c_void_p),
    ]


class WvSgnsBatch(C.Structure):
    _fields_ = [
        ("mode", C.c_int),
        ("negatives", C.c_int),
        ("window", C.c_int),
        ("model", C.c_int),
        ("batch_rows", C.c_int64),
        ("n_pairs", C.c_int64),
        ("seed", C.c_uint64),
        ("tokens", C.c_void_p),
        ("offsets", C.c_void_p),
        ("walks_by_class", C.c_void_p),
        ("class_len", C.c_void_p),
        ("class_walk_start", C.c_void_p),
        ("class_pair_start", C.c_void_p),
        ("n_classes", C.c_int64),
        ("candidates", C.c_void_p),
        ("n_candidates", C.c_int64),
        ("pairs", C.c_void_p),
        ("perm", C.c_void_p),
        ("negative_table", C.c_void_p),
        ("timer", C.c_void_p),
        ("timer_base", C.c_int64),
        ("instances", C.c_void_p),
    ]


P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int
U64 = C.c_uint64

# name -> (restype, argtypes); must mirror include/walkvec_b200.h exactly
SIGNATURES = {
    "wv_last_error": (C.c_char_p, []),
    "wv_abi_version": (I32, []),
    "wv_struct_size": (I64, [I32]),
    "wv_stream_sync": (I32, [P]),
    "wv_launch_count": (I64, []),
    "wv_timer_create": (P, [I32]),
    "wv_timer_record": (I32, [P, I32, P]),
    "wv_timer_elapsed": (I32, [P, I32, I32, P]),
    "wv_timer_destroy": (I32, [P]),
    "wv_seedseq_generate": (I32, [P, I32, U64, I32, P]),
    "wv_stream_u64": (I32, [P, I32, U64, I32, U64, P]),
    "wv_csr_workspace_bytes": (I64, [I64, I64]),
    "wv_csr_build": (I32, [P, I64, I64, P, P, P, I64, P]),
    "wv_csr_unpack": (I32, [P, I64, P, P, P]),
    "wv_walk_adjacency_build": (I32, [P, P, I64, I64, P, P]),
    "wv_random_walks_workspace_bytes": (I64, [I64, I64]),
    "wv_random_walks": (I32, [P, P, P, I64, P, I64, I64, I32, I64, I64, P, I32, I32, P, P, P, I64, P]),
    "wv_compact_workspace_bytes": (I64, [I64]),
    "wv_corpus_compact": (I32, [P, P, I64, I32, P, P, I32, P, I64, P]),
    "wv_dedup_workspace_bytes": (I64, [I64]),
    "wv_duplicate_free": (I32, [P, P, I64, I32, I64, P, P, P, P, I64, P]),
    "wv_filter_workspace_bytes": (I64, [I64]),
    "wv_corpus_filter": (I32, [P, P, I64, I32, P, P, P, P, I64, P]),
    "wv_token_histogram": (I32, [P, I64, I64, P, I32, P]),
    "wv_bfs_workspace_bytes": (I64, [I64, I64]),
    "wv_bfs_count": (I32, [P, P, I64, P, I64, I32, I64, P, P, I64, P]),
    "wv_bfs_emit": (I32, [P, P, I64, P, I64, I32, I64, P, P, P, P, I64, P]),
    "wv_path_table": (I32, [P, P, I64, P, P, P, P]),
    "wv_sgns_init": (I32, [I64, I32, P, I32, I32, P, P, P]),
    "wv_sgns_export": (I32, [I64, I32, P, I32, I32, I32, P, P, P, P]),
    "wv_pair_index_workspace_bytes": (I64, [I64]),
    "wv_pair_index_build": (I32, [P, I64, I32, P, P, P, P, P, P, P, I64, P]),
    "wv_pairs_workspace_bytes": (I64, [I64]),
    "wv_generate_pairs": (I32, [P, P, I64, I32, P, P, P, I64, P]),
    "wv_candidates_workspace_bytes": (I64, [I64]),
    "wv_candidates": (I32, [P, I64, I64, P, P, P, P, I64, P]),
    "wv_sgns_epoch_begin": (I32, [P, I64, I64, P]),
    "wv_sgns_decode": (I32, [P, I64, I64, I64, P, P, P]),
    "wv_wvc1_read_workspace_bytes": (I64, [I64]),
    "wv_vocab_tsv_workspace_bytes": (I64, [I64]),
    "wv_vocab_tsv": (I32, [P, P, I64, P, P, P, P, P, I64, P]),
    "wv_wvc1_read": (I32, [P, I64, I64, P, P, P, P, I64, P]),
    "wv_shard_count_requests": (I32, [P, I64, I64, I64, I32, P, P, P]),
    "wv_sgns_batch_workspace_bytes": (I64, [I64, I32, I32, I64, I32, I32]),
    "wv_sgns_workspace_init": (I32, [P, I64, I64, I32, I32, I64, I32, I32, P]),
    "wv_cbow_instances_workspace_bytes": (I64, [I64]),
    "wv_cbow_instances": (I32, [P, P, I64, I32, P, P, P, I64, P]),
    "wv_sgns_bind": (I32, [P, P, I64, I64, I32, I32, P]),
    "wv_sgns_batch": (I32, [P, P, P, I64, P]),
    "wv_sgns_batch_phases": (I32, [P, P, P, I64, I32, P]),
    "wv_sgns_batches": (I32, [P, P, P, I64, I64, P]),
    "wv_gen_rows_workspace_bytes": (I64, [I64]),
    "wv_gen_erdos_renyi": (I32, [I64, C.c_double, U64, P, P, P, P, I64, P]),
    "wv_gen_uniform_attachment": (I32, [I64, I32, U64, P, P, P, P, I64, P]),
    "wv_format_workspace_bytes": (I64, [I64, I32]),
    "wv_format_plan": (I32, [P, I32, I64, I32, P, P, P, P, I64, P]),
    "wv_format_emit": (I32, [P, P, I64, I32, C.c_char, P, P, I64, P]),
    "wv_wvc1_pack": (I32, [P, P, I64, P, P]),
    "wv_ingest_lines_workspace_bytes": (I64, [I64]),
    "wv_ingest_lines": (I32, [P, I64, P, P, P, I64, P]),
    "wv_ingest_workspace_bytes": (I64, [I64]),
    "wv_ingest_records_workspace_bytes": (I64, [I64]),
    "wv_ingest_records": (I32, [P, I64, I32, P, P, P, P, P, I64, P]),
    "wv_ingest_parse": (I32, [P, I64, P, I64, I32, P, C.c_uint64, I32, I32, I32, P, P, P, P, P, P, P, P, P, I64, P]),
    "wv_shard_init": (I32, [I64, I32, P, I32, I32, I32, I32, P, P, P]),
    "wv_shard_decode_group": (I32, [P, P, P, I64, I64, I32, I32, P]),
    "wv_shard_requests": (I32, [P, P, P, I64, I64, I32, I32, I64, I64, P, P, P, P, P, P]),
    "wv_shard_serve": (I32, [P, P, I64, I64, I32, P, P]),
    "wv_shard_place": (I32, [P, P, I64, I32, I32, P, P]),
    "wv_shard_gather": (I32, [P, P, P, I64, I64, I32, I32, P, P, I64, P, P, P, P]),
    "wv_shard_update": (I32, [P, P, P, I64, I64, I32, I32, P, P, P, P]),
    "wv_replica_delta": (I32, [P, P, I64, I32, P, P]),
    "wv_replica_apply": (I32, [P, P, P, P, I64, I32, I32, P]),
    "wv_barabasi_edge_count": (I64, [I64, I32]),
    "wv_barabasi_workspace_bytes": (I64, [I64, I32]),
    "wv_gen_barabasi": (I32, [I64, I32, U64, P, P, P, I64, P]),
    "wv_encode_workspace_bytes": (I64, [I64, I64]),
    "wv_encode_triples": (I32, [P, P, P, I64, I64, I64, P, P, P, P, P, I64, P]),
}

_lock = threading.Lock()
_lib: C.CDLL | None = None


def load(build_if_missing: bool = True) -> C.CDLL:
    """Load (building first if needed) the shared library; no GPU required."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists() and build_if_missing:
            from . import _build

            _build.build()
        if not LIB_PATH.exists():
            raise BackendUnavailable(f"{LIB_PATH} is missing; run paper_2508_01073_b200/_build.py")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("WV_LIB") and not hasattr(lib, name):
                continue  # A/B builds of older revisions: bind what they export
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.wv_abi_version() != ABI_VERSION:
            raise BackendUnavailable("libwalkvec_b200.so ABI version mismatch; rebuild")
        _lib = lib
        return lib


def call(name: str, *args):
    """Invoke a status-returning ABI function; raise WvError on failure."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.wv_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(msg)
        raise WvError(f"{name}: {msg}")
    return rc


_graph_replayed_launches = 0


def note_graph_replay(launches: int):
    """Count the kernels a CUDA-graph replay re-issues (the C side sees only the capture)."""
    global _graph_replayed_launches
    _graph_replayed_launches += int(launches)


def launch_count() -> int:
    """Kernels of this library enqueued so far: direct launches + graph replays."""
    return int(load().wv_launch_count()) + _graph_replayed_launches


class DeviceTimer:
    """``n`` CUDA events that also timestamp inside captured CUDA graphs (external records)."""

    def __init__(self, n: int):
        self.n = int(n)
        self.h = load().wv_timer_create(self.n)
        if not self.h:
            raise WvError(load().wv_last_error().decode())

    def record(self, i: int, stream=None):
        call("wv_timer_record", self.h, int(i), stream_ptr(stream))

    def elapsed(self, i: int, j: int) -> float:
        ms = C.c_float(0.0)
        call("wv_timer_elapsed", self.h, int(i), int(j), C.byref(ms))
        return float(ms.value)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.wv_timer_destroy(self.h)
            self.h = None


def query(name: str, *args) -> int:
    return int(getattr(load(), name)(*args))


def require_cuda():
    """The compute path needs a CUDA device; fail loudly instead of falling back."""
    import torch

    if not torch.cuda.is_available():
        raise BackendUnavailable("walkvec_b200 needs a CUDA (sm_100a) device; no CPU fallback exists")
    load()
    return torch


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
