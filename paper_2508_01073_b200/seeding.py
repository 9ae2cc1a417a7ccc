"""numpy SeedSequence entropy encoding shared by every stream on the path.

The reference seeds one generator per unit of work from integer lists:
walks ``[seed, 0, shard]`` (walks.py:172), embeddings ``[seed, 1, 0]``
(w2v.py:127), shuffle ``[seed, 1, 1]`` and negatives ``[seed, 1, 2, worker]``
(w2v.py:548-549, 687).  numpy turns each integer into its little-endian u32
words (at least one word) and concatenates them; the device kernels hash the
same words, so the host only has to produce them.
"""

from __future__ import annotations

import ctypes as C


def int_words(n: int) -> list[int]:
    n = int(n)
    if n < 0:
        raise ValueError("seed entropy must be non-negative")
    if n == 0:
        return [0]
    out = []
    while n:
        out.append(n & 0xFFFFFFFF)
        n >>= 32
    return out


def entropy_words(values) -> list[int]:
    words: list[int] = []
    for v in values:
        words.extend(int_words(v))
    return words


def words_array(words: list[int]):
    if len(words) > 13:
        raise ValueError("seed entropy too long for the device SeedSequence (max 13 words)")
    arr = (C.c_uint32 * max(1, len(words)))(*words)
    return arr, len(words)
