"""Token space for the path: Vocabulary + integer ID encoding.

Reference: pkg/src/walkvec/ingest.py:251-305 (Vocabulary) and :368-396
(build_vocabulary).  Tokens are assigned in first-occurrence order over the
flattened (subject, predicate, object) stream; entities and predicates share
one space.  String inputs (N-Triples / tables / Triple streams) are parsed
and interned on the GPU (``load_triples_device``, csrc/ingest.cu); this
module also provides the Vocabulary type the pipeline returns and a
vectorised encoder for integer-keyed triples (the synthetic graphs), equal
to build_vocabulary(assign_predicates(...)) on the same edges.
"""

from __future__ import annotations

import numpy as np

PAD = -1


class Vocabulary:
    """Bijection between lexical keys and contiguous tokens (ingest.py:251-305)."""

    def __init__(self):
        self.token_of: dict[str, int] = {}
        self.lexical_of: list[str] = []
        self._entity_tokens: set[int] = set()
        self._predicate_tokens: set[int] = set()
        self.frequency: np.ndarray | None = None
        self._entity_array: np.ndarray | None = None

    def __len__(self) -> int:
        return len(self.lexical_of)

    def __contains__(self, lexical: str) -> bool:
        return lexical in self.token_of

    @property
    def entity_count(self) -> int:
        return len(self.entity_tokens())

    @property
    def predicate_count(self) -> int:
        return len(self._predicate_tokens)

    def entity_tokens(self) -> np.ndarray:
        if self._entity_array is not None:
            return self._entity_array
        return np.array(sorted(self._entity_tokens), dtype=np.int64)

    def intern(self, lexical: str) -> int:
        token = self.token_of.get(lexical)
        if token is None:
            token = len(self.lexical_of)
            self.token_of[lexical] = token
            self.lexical_of.append(lexical)
        return token

    def lexical(self, token: int) -> str:
        return self.lexical_of[token]

    @classmethod
    def from_integer_encoding(cls, lexicals: list[str], entity_tokens: np.ndarray, predicate_tokens: np.ndarray):
        v = cls()
        v.lexical_of = list(lexicals)
        v.token_of = {s: i for i, s in enumerate(v.lexical_of)}
        v._entity_array = np.asarray(entity_tokens, dtype=np.int64)
        v._entity_tokens = set(v._entity_array.tolist())
        v._predicate_tokens = set(np.asarray(predicate_tokens, dtype=np.int64).tolist())
        return v


def _nt_escape(key: str, literal: bool) -> str:
    key = key.replace("\\", "\\\\").replace("\n", "\\n").replace("\r", "\\r")
    return key.replace('"', '\\"') if literal else key.replace(">", "\\u003E")


def build_vocabulary(triples, include_literals: bool = False):
    """Tokenise a Triple stream into (Vocabulary, (E,3) int64 edges) (ingest.py:368-396) on the GPU.

    The triples are serialised once as escaped N-Triples (keys as IRIs, literal
    objects as literals; escapes round-trip every key exactly) and tokenised by
    the device ingest, so token numbering, roles and edges are the reference's.
    """
    lines = []
    for t in triples:
        lit = getattr(t, "object_kind", "resource") == "literal"
        o = f'"{_nt_escape(t.object, True)}"' if lit else f"<{_nt_escape(t.object, False)}>"
        lines.append(f"<{_nt_escape(t.subject, False)}> <{_nt_escape(t.predicate, False)}> {o} .\n")
    if not lines:
        raise ValueError("empty graph")
    return load_triples_device("".join(lines).encode("utf-8", "surrogatepass"), "nt", strict=True,
                               include_literals=include_literals)


def encode_integer_triples(src: np.ndarray, pred: np.ndarray, dst: np.ndarray, n_entities: int,
                           with_lexicals: bool = False):
    """First-occurrence token encoding of integer triples, vectorised.

    Entities are keys ``0..n_entities-1`` ("v{u}"), predicates keys
    ``n_entities + k`` ("P{k}").  Returns (edges (E,3) int64, vocab_size,
    entity_tokens sorted, predicate_tokens sorted[, lexicals]).  Equal to the
    reference's build_vocabulary over assign_predicates' triples.
    """
    src = np.asarray(src, dtype=np.int64)
    pred = np.asarray(pred, dtype=np.int64) + int(n_entities)
    dst = np.asarray(dst, dtype=np.int64)
    stream = np.empty(3 * len(src), dtype=np.int64)
    stream[0::3], stream[1::3], stream[2::3] = src, pred, dst
    keys, first = np.unique(stream, return_index=True)
    order = np.argsort(first, kind="stable")
    token_of_key = np.empty(len(keys), dtype=np.int64)
    token_of_key[order] = np.arange(len(keys), dtype=np.int64)
    tok = token_of_key[np.searchsorted(keys, stream)]
    edges = tok.reshape(-1, 3)
    is_entity = keys < n_entities
    entity_tokens = np.sort(token_of_key[is_entity])
    predicate_tokens = np.sort(token_of_key[~is_entity])
    out = (edges, len(keys), entity_tokens, predicate_tokens)
    if with_lexicals:
        lex = np.empty(len(keys), dtype=object)
        for kk, t in zip(keys.tolist(), token_of_key.tolist()):
            lex[t] = f"v{kk}" if kk < n_entities else f"P{kk - n_entities}"
        out = out + (list(lex),)
    return out


# ------------------------------------------------------------ GPU ingest --
class ParseError(ValueError):
    """A malformed statement line or table row, with its 1-based position (ingest.py:26-32)."""

    def __init__(self, message: str, line: int):
        super().__init__(f"line {line}: {message}")
        self.line = line
        self.reason = message


_MODES = {"nt": 0, "txt": 1, "csv": 2, "tsv": 2}
_DELIM = {"csv": ord(","), "tsv": ord("\t"), "nt": 0, "txt": 0}
_MESSAGES = {
    1: "dangling escape at end of string", 5: "unexpected end of statement", 6: "unterminated IRI",
    7: "empty blank node label", 8: "unterminated literal", 9: "expected datatype IRI after ^^",
    10: "unterminated datatype IRI", 11: "empty language tag", 13: "literal not allowed as subject",
    14: "predicate must be an IRI", 15: "expected terminating '.'", 16: "trailing content after '.'",
}
_STRING_ESCAPES = {"t": "\t", "b": "\b", "n": "\n", "r": "\r", "f": "\f", '"': '"', "'": "'", "\\": "\\"}


def _csv_unquote(raw: str) -> str:
    """A csv.reader quoted field's value from its raw text: the opening quote dropped, "" -> ",
    text after the closing quote kept (excel dialect, strict=False)."""
    out, i, inside = [], 1, True
    while i < len(raw):
        c = raw[i]
        if inside and c == '"':
            if i + 1 < len(raw) and raw[i + 1] == '"':
                out.append('"')
                i += 2
                continue
            inside = False
            i += 1
            continue
        out.append(c)
        i += 1
    return "".join(out)


def _unescape_key(raw: str) -> str:
    """Decode a key span the device already validated (ingest.py:72-101)."""
    if "\\" not in raw:
        return raw
    out, i = [], 0
    while i < len(raw):
        c = raw[i]
        if c != "\\":
            out.append(c)
            i += 1
            continue
        e = raw[i + 1]
        if e in _STRING_ESCAPES:
            out.append(_STRING_ESCAPES[e])
            i += 2
        else:
            w = 4 if e == "u" else 8
            out.append(chr(int(raw[i + 2:i + 2 + w], 16)))
            i += 2 + w
    return "".join(out)


def _message(code: int, raw: bytes, at: int) -> str:
    if code < 0:
        return f"expected 3 columns, got {-code}"
    if code in _MESSAGES:
        return _MESSAGES[code]
    if code in (2, 3, 4):  # escapes: raw[at] == '\\'
        e = chr(raw[at + 1])
        if code == 4:
            return f"unknown escape \\{e}"
        w = 4 if e == "u" else 8
        if code == 2:
            return f"truncated \\{e} escape"
        return f"bad \\{e} escape: {raw[at + 2:at + 2 + w].decode('utf-8', 'replace')!r}"
    if code == 12:
        ch = raw[at:at + 4].decode("utf-8", "ignore")[:1] or chr(raw[at])
        return f"unexpected character {ch!r}"
    return f"parse error {code}"


def _read_bytes(source) -> bytes:
    if isinstance(source, (bytes, bytearray, memoryview)):
        return bytes(source)
    if isinstance(source, str) or hasattr(source, "__fspath__"):
        with open(source, "rb") as fh:
            return fh.read()
    data = source.read()
    return data.encode("utf-8") if isinstance(data, str) else data


_HASH_ATTEMPTS = 4


def load_triples_device(source, format: str = "nt", *, strict: bool = False, error_sink: list | None = None,
                        include_literals: bool = False, has_header: bool = False, device=None):
    """Parse + tokenize on the GPU: (Vocabulary, (E,3) int64 edges).

    Equals ``build_vocabulary(parse_ntriples(source, strict, error_sink), include_literals)``
    (format "nt") or ``build_vocabulary(parse_edge_table(path, format, has_header))``
    (ingest.py:188-257, 368-396): same tokens, lexical keys, roles, edges and
    errors (ParseError with the reference's message and line; non-strict
    N-Triples lines go to ``error_sink``).  Input is UTF-8 bytes; csv/tsv with
    quoted fields (delimiters and line breaks inside quotes) follow csv.reader.
    """
    from . import _lib

    if format not in _MODES:
        raise ValueError(f"unknown edge table format: {format!r}")
    torch = _lib.require_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    raw = _read_bytes(source)
    if not raw:
        raise ValueError("empty graph")
    host = torch.frombuffer(bytearray(raw), dtype=torch.uint8).pin_memory()
    text = host.to(dev, non_blocking=True)
    n = len(raw)
    st = _lib.stream_ptr()
    line_end = torch.empty(n + 1, dtype=torch.int64, device=dev)
    n_terms = torch.zeros(1, dtype=torch.int64, device=dev)
    mode = _MODES[format]
    line_no = None
    if format in ("csv", "tsv") and b'"' in raw:
        # quoted fields (csv.reader, ingest.py:241) may hold delimiters and line breaks:
        # records located by the quoting state machine, numbered by csv.reader's line_num
        mode = 3
        line_no = torch.empty(n + 1, dtype=torch.int64, device=dev)
        n_phys = torch.zeros(1, dtype=torch.int64, device=dev)
        ws = torch.empty(_lib.query("wv_ingest_records_workspace_bytes", n), dtype=torch.uint8, device=dev)
        _lib.call("wv_ingest_records", _lib.ptr(text), n, _DELIM[format], _lib.ptr(line_end), _lib.ptr(line_no),
                  _lib.ptr(n_terms), _lib.ptr(n_phys), _lib.ptr(ws), ws.numel(), st)
        n_lines = int(n_terms.item())
        if n_lines == 0 or int(line_end[n_lines - 1]) != n - 1:  # an unterminated last record
            line_end[n_lines] = n
            line_no[n_lines] = int(n_phys.item()) + 1
            n_lines += 1
    else:
        ws = torch.empty(_lib.query("wv_ingest_lines_workspace_bytes", n), dtype=torch.uint8, device=dev)
        _lib.call("wv_ingest_lines", _lib.ptr(text), n, _lib.ptr(line_end), _lib.ptr(n_terms), _lib.ptr(ws),
                  ws.numel(), st)
        n_lines = int(n_terms.item())
        if raw[-1] not in (10, 13):  # unterminated last line ends at the end of the text
            line_end[n_lines] = n
            n_lines += 1
    status = torch.empty(n_lines, dtype=torch.uint8, device=dev)
    err = torch.empty(n_lines, dtype=torch.int32, device=dev)
    err_at = torch.empty(n_lines, dtype=torch.int64, device=dev)
    bad = torch.empty(2, dtype=torch.int64, device=dev)
    n_out = torch.zeros(4, dtype=torch.int64, device=dev)
    edges = torch.empty(max(3 * n_lines, 3), dtype=torch.int64, device=dev)
    roles = torch.empty(max(3 * n_lines, 1), dtype=torch.int32, device=dev)
    tok_span = torch.empty(max(9 * n_lines, 3), dtype=torch.int64, device=dev)
    ws = torch.empty(_lib.query("wv_ingest_workspace_bytes", n_lines), dtype=torch.uint8, device=dev)
    for hash_seed in range(_HASH_ATTEMPTS):
        # a 64-bit key-hash collision (distinct keys, equal hashes) is detected, never merged:
        # re-intern with an independently seeded hash
        n_out.zero_()
        _lib.call("wv_ingest_parse", _lib.ptr(text), n, _lib.ptr(line_end), n_lines, mode, _lib.ptr(line_no),
                  hash_seed,
                  _DELIM[format], int(has_header), int(include_literals), _lib.ptr(status), _lib.ptr(err),
                  _lib.ptr(err_at), _lib.ptr(bad), _lib.ptr(n_out), _lib.ptr(edges), _lib.ptr(roles),
                  _lib.ptr(tok_span), _lib.ptr(ws), ws.numel(), st)
        n_stmt, n_edges, n_tok, collision = (int(x) for x in n_out.cpu().tolist())
        if not collision:
            break
    first_bad, first_value = (int(x) for x in bad.cpu().tolist())
    big = (1 << 63) - 1
    if first_bad != big or first_value != big:
        codes = err.cpu().numpy()
        ats = err_at.cpu().numpy()
        stat = status.cpu().numpy()
        if format != "nt" or strict:
            if stat[first_bad] == 3:
                raise ValueError("subject and predicate must be non-empty")
            row = int(line_no[first_bad]) if line_no is not None else first_bad + 1
            raise ParseError(_message(int(codes[first_bad]), raw, int(ats[first_bad])), row)
        stop = first_value if first_value != big else n_lines
        if error_sink is not None:
            for L in np.flatnonzero(stat[:stop] == 2).tolist():
                error_sink.append(ParseError(_message(int(codes[L]), raw, int(ats[L])), L + 1))
        if first_value != big:
            raise ValueError("subject and predicate must be non-empty")
    if collision:
        raise RuntimeError(f"64-bit key hash collisions under {_HASH_ATTEMPTS} independent hash seeds")
    if n_stmt == 0:
        raise ValueError("empty graph")
    spans = tok_span[: 3 * n_tok].view(-1, 3).cpu().numpy()
    lexicals = []
    for s, t, fl in spans.tolist():
        key = raw[s:t].decode("utf-8", "surrogatepass")
        esc = fl & 3
        lexicals.append(_unescape_key(key) if esc == 1 else (_csv_unquote(key) if esc == 2 else key))
    r = roles[:n_tok].cpu().numpy()
    vocab = Vocabulary.from_integer_encoding(lexicals, np.flatnonzero(r & 1), np.flatnonzero(r & 2))
    return vocab, edges[: 3 * n_edges].view(-1, 3).cpu().numpy()
