"""Token space for the path: Vocabulary + integer ID encoding.

Reference: pkg/src/walkvec/ingest.py:251-305 (Vocabulary) and :368-396
(build_vocabulary).  Tokens are assigned in first-occurrence order over the
flattened (subject, predicate, object) stream; entities and predicates share
one space.  String parsing (N-Triples / CSV) precedes the hot path and stays
with the reference; this module provides the Vocabulary type the pipeline
returns and a vectorised encoder for integer-keyed triples (the synthetic
graphs), equal to build_vocabulary(assign_predicates(...)) on the same edges.
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


def build_vocabulary(triples, include_literals: bool = False):
    """Tokenise a Triple stream into (Vocabulary, (E,3) int64 edges) (ingest.py:368-396)."""
    vocab = Vocabulary()
    src, pred, dst = [], [], []
    seen_any = False
    for t in triples:
        seen_any = True
        s = vocab.intern(t.subject)
        vocab._entity_tokens.add(s)
        p = vocab.intern(t.predicate)
        vocab._predicate_tokens.add(p)
        if getattr(t, "object_kind", "resource") == "literal" and not include_literals:
            continue
        o = vocab.intern(t.object)
        vocab._entity_tokens.add(o)
        src.append(s)
        pred.append(p)
        dst.append(o)
    if not seen_any:
        raise ValueError("empty graph")
    edges = np.empty((len(src), 3), dtype=np.int64)
    edges[:, 0] = src
    edges[:, 1] = pred
    edges[:, 2] = dst
    return vocab, edges


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
