"""Vectorised host port of tlr::Rng (util.hpp:24-53): std::mt19937_64 with the
standard seeding, uniform (0, 1] from the top 53 bits, and the Marsaglia polar
method with a one-value pair cache.

Host-side uses: the RandomBall3D point sampler (geometry.cpp:60-74) and the
oracle / tests.  The device draws the same streams in csrc/rng.cuh.
"""
from __future__ import annotations

import numpy as np

N, M = 312, 156
MATRIX_A = np.uint64(0xB5026F5AA96619E9)
UM = np.uint64(0xFFFFFFFF80000000)
LM = np.uint64(0x7FFFFFFF)


def _seed_state(seed: int) -> np.ndarray:
    mt = [seed & 0xFFFFFFFFFFFFFFFF]
    for i in range(1, N):
        p = mt[-1]
        mt.append((6364136223846793005 * (p ^ (p >> 62)) + i) & 0xFFFFFFFFFFFFFFFF)
    return np.array(mt, dtype=np.uint64)


def _twist(mt: np.ndarray):
    one = np.uint64(1)
    zero = np.uint64(0)
    y = (mt[0:N - M] & UM) | (mt[1:N - M + 1] & LM)
    mt[0:N - M] = mt[M:N] ^ (y >> one) ^ np.where((y & one) != 0, MATRIX_A, zero)
    y = (mt[N - M:N - 1] & UM) | (mt[N - M + 1:N] & LM)
    mt[N - M:N - 1] = mt[0:M - 1] ^ (y >> one) ^ np.where((y & one) != 0, MATRIX_A, zero)
    y = (mt[N - 1] & UM) | (mt[0] & LM)
    mt[N - 1] = mt[M - 1] ^ (y >> one) ^ (MATRIX_A if (int(y) & 1) else zero)


def _temper(y: np.ndarray) -> np.ndarray:
    y = y ^ ((y >> np.uint64(29)) & np.uint64(0x5555555555555555))
    y = y ^ ((y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000))
    y = y ^ ((y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000))
    return y ^ (y >> np.uint64(43))


class Mt64:
    def __init__(self, seed: int):
        self.mt = _seed_state(seed)
        self.idx = N
        self._g = np.zeros(0)  # produced-but-unconsumed gaussians (pair cache)

    def raw(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        o = 0
        while o < n:
            if self.idx >= N:
                _twist(self.mt)
                self.idx = 0
            take = min(n - o, N - self.idx)
            out[o:o + take] = _temper(self.mt[self.idx:self.idx + take])
            self.idx += take
            o += take
        return out

    def uniforms(self, n: int) -> np.ndarray:
        return ((self.raw(n) >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53

    def gaussians(self, n: int) -> np.ndarray:
        while len(self._g) < n:
            need = n - len(self._g)
            att = max(8, int(need * 0.65) + 8)  # ~pi/4 acceptance, 2 values per accept
            uv = self.uniforms(2 * att).reshape(-1, 2) * 2.0 - 1.0
            s = (uv * uv).sum(1)
            ok = (s < 1.0) & (s != 0.0)
            u, v, s = uv[ok, 0], uv[ok, 1], s[ok]
            f = np.sqrt(-2.0 * np.log(s) / s)
            g = np.empty(2 * len(s))
            g[0::2] = u * f
            g[1::2] = v * f
            self._g = np.concatenate([self._g, g])
        out, self._g = self._g[:n].copy(), self._g[n:]
        return out
