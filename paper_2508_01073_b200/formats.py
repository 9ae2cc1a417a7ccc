"""On-disk formats of the path's outputs, written from the device.

* ``save_embeddings_text`` / ``save_embeddings_tsv`` (pipeline.py:236-251):
  word2vec text ("<count> <dim>" header, "<lexical> <d floats>" lines) and
  the TSV export, with Python's correctly rounded ``%.8g`` computed on the
  device (csrc/formats.cu) and the file written in one piece.
* ``save_corpus_binary`` (walks.py:344-364): the WVC1 corpus, body packed on
  the device.  Files are byte-identical to the reference's writers, so the
  reference's readers (``load_embeddings_text``, ``load_corpus_binary``) load them.
"""

from __future__ import annotations

import struct

import numpy as np

from . import _lib

_CORPUS_MAGIC = b"WVC1"


def _escape_lexical_tsv(value: str) -> str:
    return value.replace("\\", "\\\\").replace("\t", "\\t").replace("\n", "\\n")


def _format_rows(vectors, lexicals: list[str], sep: str) -> bytes:
    torch = _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    vec = vectors if isinstance(vectors, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(vectors))
    if vec.dtype not in (torch.float32, torch.float64):
        vec = vec.double()
    vec = vec.to(dev).contiguous()
    rows, d = int(vec.shape[0]), int(vec.shape[1])
    enc = [s.encode("utf-8", "surrogatepass") for s in lexicals]
    lens = np.fromiter((len(b) for b in enc), dtype=np.int64, count=rows)
    lex_off = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(lens, out=lex_off[1:])
    lex = torch.frombuffer(bytearray(b"".join(enc) or b"\0"), dtype=torch.uint8).to(dev)
    off = torch.from_numpy(lex_off).to(dev)
    total = torch.zeros(1, dtype=torch.int64, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = torch.empty(_lib.query("wv_format_workspace_bytes", rows, d), dtype=torch.uint8, device=dev)
    prec = _lib.FP32 if vec.dtype == torch.float32 else _lib.FP64
    st = _lib.stream_ptr()
    _lib.call("wv_format_plan", _lib.ptr(vec), prec, rows, d, _lib.ptr(off), _lib.ptr(total), _lib.ptr(bad),
              _lib.ptr(ws), ws.numel(), st)
    if int(bad.item()):
        raise ValueError("a value lies outside the device %.8g formatter's range (1e-30 <= |x| < 1e16)")
    out = torch.empty(max(int(total.item()), 1), dtype=torch.uint8, device=dev)
    _lib.call("wv_format_emit", _lib.ptr(lex), _lib.ptr(off), rows, d, sep.encode(), _lib.ptr(out), _lib.ptr(ws),
              ws.numel(), st)
    return out[: int(total.item())].cpu().numpy().tobytes()


def _lexicals(vocab, rows: int) -> list[str]:
    return [vocab.lexical(t) for t in range(rows)]


def save_embeddings_text(vectors, vocab, path):
    """word2vec text format (pipeline.py:236-243)."""
    rows, d = int(vectors.shape[0]), int(vectors.shape[1])
    body = _format_rows(vectors, _lexicals(vocab, rows), " ")
    with open(path, "wb") as fh:
        fh.write(f"{rows} {d}\n".encode())
        fh.write(body)


def save_embeddings_tsv(vectors, vocab, path):
    """Tab-separated export: escaped lexical, then the d components (pipeline.py:246-251)."""
    rows = int(vectors.shape[0])
    body = _format_rows(vectors, [_escape_lexical_tsv(s) for s in _lexicals(vocab, rows)], "\t")
    with open(path, "wb") as fh:
        fh.write(body)


def save_corpus_binary(corpus, path):
    """WVC1 walk corpus (walks.py:344-364), body packed on the device."""
    from .walks import BFS, ENTITY, FULL, PROPERTY, RANDOM

    torch = _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    if hasattr(corpus, "device_arrays"):
        tok, off = corpus.device_arrays(dev)
    else:  # the reference's WalkCorpus (host int64 arrays)
        t64 = np.asarray(corpus.tokens, dtype=np.int64)
        if t64.size and (t64.min() < 0 or t64.max() >= 2**31):
            raise ValueError("token does not fit in u32")
        tok = torch.from_numpy(t64.astype(np.int32) if t64.size else np.zeros(1, np.int32)).to(dev)
        off = torch.from_numpy(np.asarray(corpus.offsets, dtype=np.int64)).to(dev)
    n, total = len(corpus), int(np.asarray(corpus.offsets)[-1]) if not hasattr(corpus, "total_tokens") \
        else corpus.total_tokens
    if total and int(tok[:total].max()) < 0:
        raise ValueError("token does not fit in u32")
    strategies = {RANDOM: 0, BFS: 1}
    projections = {FULL: 0, ENTITY: 1, PROPERTY: 2}
    body = torch.empty(max(n + total, 1), dtype=torch.int32, device=dev)
    _lib.call("wv_wvc1_pack", _lib.ptr(tok), _lib.ptr(off), n, _lib.ptr(body), _lib.stream_ptr())
    with open(path, "wb") as fh:
        fh.write(_CORPUS_MAGIC)
        fh.write(struct.pack("<BBHI", strategies[corpus.strategy], projections[corpus.projection], 0, n))
        fh.write(body[: n + total].cpu().numpy().astype("<u4").tobytes())


def load_corpus_binary(path):
    """Read a WVC1 walk corpus (walks.py:368-389) into a device WalkCorpus.

    The file is read once; record boundaries (a chain of u32 length headers)
    are found on the device by speculative chunk parsing (csrc/formats.cu).
    Errors follow the reference: ValueError for a bad magic or a corrupt body,
    IndexError when the body ends before the header's walk count.
    """
    from .walks import BFS, ENTITY, FULL, PROPERTY, RANDOM, WalkCorpus

    torch = _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    raw = open(path, "rb").read()
    if raw[:4] != _CORPUS_MAGIC:
        raise ValueError("not a walk corpus file")
    strategy_b, projection_b, _, count = struct.unpack("<BBHI", raw[4:12])
    strategies = {0: RANDOM, 1: BFS}
    projections = {0: FULL, 1: ENTITY, 2: PROPERTY}
    if (len(raw) - 12) % 4:
        raise ValueError("buffer size must be a multiple of element size")
    n = (len(raw) - 12) // 4
    body = torch.frombuffer(bytearray(raw[12:]), dtype=torch.int32).to(dev) if n else \
        torch.zeros(1, dtype=torch.int32, device=dev)
    n_tok = max(n - count, 0)
    offsets = torch.empty(count + 1, dtype=torch.int64, device=dev)
    tokens = torch.empty(max(n_tok, 1), dtype=torch.int32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = torch.empty(_lib.query("wv_wvc1_read_workspace_bytes", n), dtype=torch.uint8, device=dev)
    _lib.call("wv_wvc1_read", _lib.ptr(body), n, count, _lib.ptr(offsets), _lib.ptr(tokens), _lib.ptr(status),
              _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    st = int(status.item())
    if st == 3:
        raise IndexError(f"index {n} is out of bounds for axis 0 with size {n}")
    if st != 0 or (count == 0 and n != 0):
        raise ValueError("corrupt walk corpus file")
    if n_tok and int(tokens[:n_tok].min()) < 0:
        raise ValueError("token out of int32 range")
    return WalkCorpus.from_device(tokens, offsets, count, n_tok, strategies[strategy_b], projections[projection_b])


def save_vocabulary_tsv(vocab, path):
    """Vocabulary.save_tsv (ingest.py:307-323) with the lines formatted on the device:
    token, escaped lexical (_escape_field, ingest.py:345-346), roles, frequency."""
    torch = _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    lexicals = list(vocab.lexical_of)
    rows = len(lexicals)
    enc = [s_.encode("utf-8", "surrogatepass") for s_ in lexicals]
    lex_off = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(np.fromiter((len(b) for b in enc), dtype=np.int64, count=rows), out=lex_off[1:])
    ents, preds = vocab._entity_tokens, vocab._predicate_tokens
    roles = np.fromiter(((1 if t in ents else 0) | (2 if t in preds else 0) for t in range(rows)), dtype=np.uint8,
                        count=rows)
    freq = vocab.frequency
    counts = np.zeros(rows, dtype=np.int64) if freq is None else np.asarray(freq, dtype=np.int64)[:rows]
    d_lex = torch.frombuffer(bytearray(b"".join(enc) or b"\0"), dtype=torch.uint8).to(dev)
    d_off = torch.from_numpy(lex_off).to(dev)
    d_roles = torch.from_numpy(roles if rows else np.zeros(1, np.uint8)).to(dev)
    d_counts = torch.from_numpy(counts if rows else np.zeros(1, np.int64)).to(dev)
    total = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = torch.empty(_lib.query("wv_vocab_tsv_workspace_bytes", rows), dtype=torch.uint8, device=dev)
    st = _lib.stream_ptr()
    args = (_lib.ptr(d_lex), _lib.ptr(d_off), rows, _lib.ptr(d_roles), _lib.ptr(d_counts))
    _lib.call("wv_vocab_tsv", *args, None, _lib.ptr(total), _lib.ptr(ws), ws.numel(), st)
    n = int(total.item())
    out = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    _lib.call("wv_vocab_tsv", *args, _lib.ptr(out), _lib.ptr(total), _lib.ptr(ws), ws.numel(), st)
    with open(path, "wb") as fh:
        fh.write(out[:n].cpu().numpy().tobytes())
