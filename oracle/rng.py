"""Pure-integer restatement of numpy's SeedSequence, PCG64 and Philox4x64-10.

numpy is the reference's only dependency (pkg/pyproject.toml:10); every
stream on the path comes from these generators (walks.py:172, w2v.py:127,
548-549).  Restated from numpy's published algorithms (bit_generator.pyx
SeedSequence; pcg64.h XSL-RR 128/64; philox.h) and checked against numpy
itself in tests/test_oracle.py.  TEST INFRASTRUCTURE ONLY.
"""

from __future__ import annotations

M32 = 0xFFFFFFFF
M64 = 0xFFFFFFFFFFFFFFFF
M128 = (1 << 128) - 1
INIT_A, MULT_A = 0x43B0D7E5, 0x931E8875
INIT_B, MULT_B = 0x8B51F9DD, 0x58F38DED
MIX_L, MIX_R = 0xCA01F9DD, 0x4973F715
PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645


def entropy_words(values) -> list[int]:
    out = []
    for v in values:
        v = int(v)
        if v == 0:
            out.append(0)
        while v:
            out.append(v & M32)
            v >>= 32
    return out


def seedseq_pool(values) -> list[int]:
    ent = entropy_words(values)
    hc = INIT_A

    def hashmix(x):
        nonlocal hc
        x = (x ^ hc) & M32
        hc = (hc * MULT_A) & M32
        x = (x * hc) & M32
        return x ^ (x >> 16)

    def mix(x, y):
        r = (MIX_L * x - MIX_R * y) & M32
        return r ^ (r >> 16)

    pool = [hashmix(ent[i] if i < len(ent) else 0) for i in range(4)]
    for s in range(4):
        for d in range(4):
            if s != d:
                pool[d] = mix(pool[d], hashmix(pool[s]))
    for s in range(4, len(ent)):
        for d in range(4):
            pool[d] = mix(pool[d], hashmix(ent[s]))
    return pool


def generate_state_u64(values, n64: int) -> list[int]:
    pool = seedseq_pool(values)
    hc = INIT_B
    words = []
    for i in range(2 * n64):
        x = (pool[i % 4] ^ hc) & M32
        hc = (hc * MULT_B) & M32
        x = (x * hc) & M32
        words.append(x ^ (x >> 16))
    return [words[2 * i] | (words[2 * i + 1] << 32) for i in range(n64)]


class PCG64:
    """numpy PCG64 seeded from SeedSequence(values), with O(log k) jump-ahead."""

    def __init__(self, values):
        g = generate_state_u64(values, 4)
        initstate = (g[0] << 64) | g[1]
        initseq = (g[2] << 64) | g[3]
        self.inc = ((initseq << 1) | 1) & M128
        self.state = 0
        self._step()
        self.state = (self.state + initstate) & M128
        self._step()

    def _step(self):
        self.state = (self.state * PCG_MULT + self.inc) & M128

    @staticmethod
    def output(state: int) -> int:
        hi, lo = state >> 64, state & M64
        v, rot = hi ^ lo, state >> 122
        return ((v >> rot) | (v << ((64 - rot) & 63))) & M64

    def state_after(self, n: int) -> int:
        """state after n more steps (affine jump: x -> A x + C)."""
        A, Cc = 1, 0
        a, c = PCG_MULT, self.inc
        while n:
            if n & 1:
                A, Cc = (A * a) & M128, (Cc * a + c) & M128
            a, c = (a * a) & M128, (c * (a + 1)) & M128
            n >>= 1
        return (A * self.state + Cc) & M128

    def u64_at(self, k: int) -> int:
        """stream element k (0-based) without consuming."""
        return self.output(self.state_after(k + 1))


PH_M0, PH_M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
PH_W0, PH_W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B


def philox4x64_10(ctr, key):
    c0, c1, c2, c3 = ctr
    k0, k1 = key
    for r in range(10):
        if r:
            k0, k1 = (k0 + PH_W0) & M64, (k1 + PH_W1) & M64
        p0, p1 = PH_M0 * c0, PH_M1 * c2
        c0, c1, c2, c3 = (p1 >> 64) ^ c1 ^ k0, p1 & M64, (p0 >> 64) ^ c3 ^ k1, p0 & M64
    return c0, c1, c2, c3


class Philox:
    """numpy Philox(SeedSequence(values)) stream, counter-addressed."""

    def __init__(self, values):
        self.key = tuple(generate_state_u64(values, 2))

    def u64_at(self, k: int) -> int:
        return philox4x64_10((1 + k // 4, 0, 0, 0), self.key)[k % 4]


def to_double(u: int) -> float:
    return (u >> 11) * (1.0 / 9007199254740992.0)
