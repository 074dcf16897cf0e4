"""Seeded input stream — restatement of the reference's ``snop::Rng``
(/root/reference/proj/core/include/snop/rng.hpp:17-49): ``std::mt19937_64`` engine, 53-bit
uniform, explicit Box-Muller with a cached spare. Streams are pinned bit-for-bit against the
reference header compiled under ``oracle/_ref`` (tests/golden/ref_infra.json).

Host-side input generation only (never on the device hot path).
"""
from __future__ import annotations

import math

import numpy as np

_N, _M = 312, 156
_MATRIX_A = np.uint64(0xB5026F5AA96619E9)
_UPPER = np.uint64(0xFFFFFFFF80000000)
_LOWER = np.uint64(0x7FFFFFFF)
_MASK64 = (1 << 64) - 1


def _twist(mt: np.ndarray) -> None:
    """In-place mt19937_64 state transition, vectorised in three dependency-free slices."""
    one = np.uint64(1)

    def gen(i0, i1, nxt, far):
        x = (mt[i0:i1] & _UPPER) | (nxt & _LOWER)
        xa = x >> one
        xa ^= np.where((x & one) == one, _MATRIX_A, np.uint64(0))
        mt[i0:i1] = far ^ xa

    gen(0, _N - _M, mt[1:_N - _M + 1].copy(), mt[_M:_N].copy())
    gen(_N - _M, _N - 1, mt[_N - _M + 1:_N].copy(), mt[0:_M - 1].copy())
    gen(_N - 1, _N, mt[0:1].copy(), mt[_M - 1:_M].copy())


def _temper(y: np.ndarray) -> np.ndarray:
    y = y ^ ((y >> np.uint64(29)) & np.uint64(0x5555555555555555))
    y = y ^ ((y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000))
    y = y ^ ((y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000))
    return y ^ (y >> np.uint64(43))


class Rng:
    """``snop::Rng`` (rng.hpp:17-49)."""

    def __init__(self, seed: int):
        mt = [0] * _N
        mt[0] = seed & _MASK64
        for i in range(1, _N):
            prev = mt[i - 1]
            mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & _MASK64
        self._mt = np.array(mt, dtype=np.uint64)
        self._buf = np.empty(0, dtype=np.uint64)
        self._pos = 0
        self._has_spare = False
        self._spare = 0.0

    def _refill(self) -> None:
        _twist(self._mt)
        self._buf = _temper(self._mt)
        self._pos = 0

    def next_u64(self) -> int:
        if self._pos >= self._buf.size:
            self._refill()
        v = int(self._buf[self._pos])
        self._pos += 1
        return v

    def next_u64_array(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        k = 0
        while k < n:
            if self._pos >= self._buf.size:
                self._refill()
            take = min(n - k, self._buf.size - self._pos)
            out[k:k + take] = self._buf[self._pos:self._pos + take]
            self._pos += take
            k += take
        return out

    def uniform(self, lo: float | None = None, hi: float | None = None) -> float:
        u = float(self.next_u64() >> 11) * 2.0 ** -53
        if lo is None:
            return u
        return lo + (hi - lo) * u

    def uniform_array(self, n: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
        u = (self.next_u64_array(n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        return lo + (hi - lo) * u

    def normal(self) -> float:
        if self._has_spare:
            self._has_spare = False
            return self._spare
        u1 = (float(self.next_u64() >> 11) + 1.0) * 2.0 ** -53
        u2 = self.uniform()
        r = math.sqrt(-2.0 * math.log(u1))
        a = 2.0 * math.pi * u2
        self._spare = r * math.sin(a)
        self._has_spare = True
        return r * math.cos(a)


def chunk_bounds(n_items: int, n_chunks: int) -> list[tuple[int, int]]:
    """The reference's fixed partition (parallel.hpp:17-48): independent of thread count."""
    if n_items == 0:
        return []
    if n_chunks == 0 or n_chunks > n_items:
        n_chunks = n_items
    base, extra = divmod(n_items, n_chunks)
    beg = [c * base + min(c, extra) for c in range(n_chunks + 1)]
    return [(beg[c], beg[c + 1]) for c in range(n_chunks)]
