"""Generate the golden fixtures from the UNMODIFIED reference (oracle/_ref).

Run in the build container (where /root/reference and oracle/_ref exist):
    python tests/golden/make_golden.py
The fixtures pin the oracle build (CPU tests re-derive them and must match)
and let the GPU tests check parity without loading the oracle at run time.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402
from paper_2108_11932_b200 import geometry as G  # noqa: E402

# problem: 2D exponential covariance (cfg1 family, small), tile 64
N, B, EPS, BS, SEED = 512, 64, 1e-6, 16, 5


def problem():
    pts = G.kd_order(G.generate_points(G.GRID2D, N, 0), B).matrix_order()
    return ref.build(pts, 0, 0.1, 0.0, B, EPS, 0, BS, SEED)


def main():
    out = {}
    # tlr::Rng draw streams (util.hpp:24-53)
    for s in (0, 12345):
        out[f"rng_{s}"] = ref.rng_gaussians(s, 512)
    # orthog (dense_kernels.cpp:379-420) on a fixed Q / Y
    r = np.random.default_rng(3)
    Q, _ = np.linalg.qr(r.normal(size=(64, 10)))
    Y = r.normal(size=(64, 8))
    Y[:, 3] = Q @ r.normal(size=10)  # a column inside range(Q): deficient
    Yo, R, cn, nm, nd = ref.orthog(Q, Y, 77)
    out["orthog_Q"], out["orthog_Y_in"] = Q, Y
    out["orthog_Y"], out["orthog_R"], out["orthog_cn"], out["orthog_nm"] = Yo, R, cn, nm
    out["orthog_next_draw"] = np.array([nd])
    # TLR Cholesky of the problem
    A = problem()
    d, rk, U, V = A.to_parts()
    out["A_diag"] = np.stack(d)
    out["A_ranks"] = np.asarray(rk, np.int32)
    out["A_U"] = np.concatenate([u.T.ravel() for u in U]) if U else np.zeros(0)
    out["A_V"] = np.concatenate([v.T.ravel() for v in V]) if V else np.zeros(0)
    F = ref.factor(A, 0, bs=BS, eps=EPS, seed=SEED)
    out["L_ranks"] = np.asarray(F.L_ranks(), np.int32)
    out["L_ara_rounds"] = np.asarray(F.stats().ara_rounds, np.int32)
    out["resid_2norm"] = np.array([ref.estimate_2norm_diff(A, F, 50, 17)])
    ld, _, lu, lv = F.L_parts()
    out["L_diag"] = np.stack(ld)
    np.savez_compressed(os.path.join(HERE, "tlr_small.npz"), **out)
    print("wrote", os.path.join(HERE, "tlr_small.npz"), {k: np.shape(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
