"""Shared problem builders for the parity tests (mirror the reference tests'
fixtures: test_ara.cpp:15-68, test_factor.cpp:13-49)."""
import numpy as np

from paper_2108_11932_b200 import geometry as G


def points(kind, n, tile, seed=42):
    return G.kd_order(G.generate_points(kind, n, seed), tile).matrix_order()


def covariance_ref(ref, n, b, eps, seed=42, kind=G.BALL3D, ell=0.2, nugget=0.0, bs=16,
                   kernel=0, compressor=0):
    """covariance_tlr (test_ara.cpp:15-23) built by the reference."""
    pts = points(kind, n, b, seed if kind == G.BALL3D else 0)
    return ref.build(pts, kernel, ell, nugget, b, eps, compressor, bs, seed)


def to_gpu(tg, A_ref):
    """The reference-built matrix uploaded unchanged (flat layout)."""
    diag, ranks, U, V = A_ref.to_flat()
    return tg.TlrMatrix.from_flat(A_ref.n, A_ref.b, A_ref.eps, diag, ranks, U, V)


def dblocks_np(nb, rows, seed):
    """Deterministic random D blocks (1x1 / 2x2) for LDL-mode sampling tests."""
    r = np.random.default_rng(seed)
    out = []
    for j in range(nb):
        n = rows[j]
        d, e, s2 = np.zeros(n), np.zeros(max(n - 1, 0)), np.zeros(n, np.uint8)
        k = 0
        while k < n:
            if k + 1 < n and r.uniform() < 0.3:
                d[k], d[k + 1], e[k] = r.normal(), r.normal(), r.normal()
                s2[k] = 1
                k += 2
            else:
                d[k] = r.normal() + 2.0
                k += 1
        out.append((d, e, s2))
    return out


def qbt(Q, B):
    return Q @ B.T
