"""Dev tool: chol_ara_update on one column with the wide-basis recompression
on B (default) and with QR + Jacobi on R (TLRG_WIDE_B=0): per-tile difference
of the approximations Q B^T, in units of eps."""
import os, sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2108_11932_b200 as tg
from paper_2108_11932_b200 import geometry as G
from oracle import ref
from helpers import points, to_gpu
n, b, eps, bs = 8192, 512, 1e-4, 32
A_ref = ref.build(points(G.GRID3D, n, b, 0), 1, 0.2, 1e-4, b, eps, 0, bs, 12345)
A = to_gpu(tg, A_ref)
F = tg.tlr_ldlt(A.copy(), tg.AraConfig(block_samples=bs, eps=eps, seed=1))
A = F.L  # later columns of the factor carry the wide bases
D = F.D
for k in (3, 5, 8, 10):
    res = {}
    for mode in ("1", "0"):
        os.environ["TLRG_WIDE_B"] = mode
        res[mode] = tg.chol_ara_update(A, D, k, tg.AraConfig(block_samples=bs, eps=eps, seed=1))
    for a, c in zip(res["1"], res["0"]):
        Pa, Pc = a.Q @ a.B.T, c.Q @ c.B.T
        d = np.linalg.norm(Pa - Pc, 2)
        if a.Q.shape[1] > 60 or d > 0.05 * eps:
            print(k, a.i, "rank", a.Q.shape[1], c.Q.shape[1], "diff/eps %.3e" % (d / eps),
                  "orth %.1e" % np.abs(a.Q.T @ a.Q - np.eye(a.Q.shape[1])).max(), flush=True)
