"""Synthetic inputs of the BASELINE.json configurations (host side).

Configs 1-4 are covariance matrices of the reference's point sets
(geometry.cpp:20-168; ``geometry.py``).  Config 5, the batched-ARA microbench,
is not a covariance: it is one TLR column of synthetic low-rank tiles, exactly
as SURVEY.md 8(d) defines it:

    tile t (t = 0..T-1) sits at (i, j) = (t + 1, 0) of an nb = T + 1 matrix,
    rank r_t = 8 + (mix64(777 ^ t) mod 121)  in [8, 128],
    A_t = Q1 diag(sigma) Q2^T,  sigma_p = 10^(-8 p / (r_t - 1)),
    Q1, Q2 = orthonormalised m x r_t gaussian blocks of the generator seeded by
    tile_seed(4242, 5, t, 0)  (numpy's PCG64 stream; Cholesky-QR, two passes),
    stored as U = Q1 diag(sigma), V = Q2.

The reference call it times is chol_ara_update(M, nullptr, 0, cfg, ws, Chol)
(ara.cpp:302-419) with bs = 32 and eps in {1e-2, 1e-4, 1e-6, 1e-8}.  Both bench
arms get the identical arrays from this module.
"""
from __future__ import annotations

import numpy as np

from .util import mix64, tile_seed


def _cholqr2(g):
    """Stacked Cholesky-QR, two passes: orthonormal columns of each g[a]."""
    for _ in range(2):
        r = np.linalg.cholesky(np.swapaxes(g, 1, 2) @ g)  # lower, = R^T
        g = np.swapaxes(np.linalg.solve(r, np.swapaxes(g, 1, 2)), 1, 2)
    return g


def cfg5_rank(t: int) -> int:
    return 8 + int(mix64(777 ^ t) % 121)


def cfg5_tile(t: int, m: int = 512):
    r = cfg5_rank(t)
    g = np.random.default_rng(tile_seed(4242, 5, t, 0)).standard_normal((1, m, 2 * r))
    q1, q2 = _cholqr2(g[:, :, :r])[0], _cholqr2(g[:, :, r:])[0]
    sigma = 10.0 ** (-8.0 * np.arange(r) / (r - 1))
    return q1 * sigma, q2


def cfg5_column(ntiles: int = 4096, m: int = 512):
    """(n, b, ranks[nb(nb-1)/2] int32, U flat, V flat) in the reference's flat
    layout (tile (i, j) at i(i-1)/2 + j, column-major payloads).  Tiles of equal
    rank are orthonormalised in one stacked QR (same result as cfg5_tile)."""
    nb = ntiles + 1
    ranks = np.zeros(nb * (nb - 1) // 2, np.int32)
    rk = np.array([cfg5_rank(t) for t in range(ntiles)])
    Ut, Vt = [None] * ntiles, [None] * ntiles
    for r in np.unique(rk):
        ts = np.nonzero(rk == r)[0]
        g = np.stack([np.random.default_rng(tile_seed(4242, 5, int(t), 0)).standard_normal((m, 2 * r))
                      for t in ts])
        q1, q2 = _cholqr2(g[:, :, :r]), _cholqr2(g[:, :, r:])
        sigma = 10.0 ** (-8.0 * np.arange(r) / (r - 1))
        for a, t in enumerate(ts):
            Ut[t] = (q1[a] * sigma).T.ravel()
            Vt[t] = q2[a].T.ravel()
    for t in range(ntiles):
        i = t + 1
        ranks[i * (i - 1) // 2] = rk[t]
    return nb * m, m, ranks, np.concatenate(Ut), np.concatenate(Vt)
