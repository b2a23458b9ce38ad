"""Backward/forward solve error and Frobenius residual of the B200 factor and
the reference factor on the same reference-built A, over several ARA seeds
(cfg3 family by default): is a gap systematic or seed noise?"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2108_11932_b200 as tg  # noqa: E402
from helpers import points, to_gpu  # noqa: E402
from oracle import ref  # noqa: E402
from paper_2108_11932_b200 import geometry as G  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
seeds = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [12345, 1, 2, 3, 4, 5]
b, eps, bs = 512, 1e-4, 32
pts = points(G.GRID3D, n, b, 0)
A_ref = ref.build(pts, 1, 0.2, 1e-4, b, eps, 0, bs, 12345)
A = to_gpu(tg, A_ref)
rows = []
for sd in seeds:
    F_ref = ref.factor(A_ref, 1, bs=bs, eps=eps, seed=sd)
    ra = ref.accuracy(A_ref, F_ref)
    F = tg.tlr_ldlt(A.copy(), tg.AraConfig(block_samples=bs, eps=eps, seed=sd))
    oa = tg.tlr.accuracy(A, F)
    rows.append((sd, oa["backward_err"], ra["backward_err"], oa["forward_err"], ra["forward_err"],
                 oa["resid_frob_rel"], ra["resid_frob_rel"]))
    print("seed %6d  bwd ours %.3e ref %.3e | fwd ours %.3e ref %.3e | frob ours %.3e ref %.3e" %
          rows[-1], flush=True)
r = np.array(rows)[:, 1:]
gm = np.exp(np.log(r).mean(axis=0))
print("geomean bwd ours %.3e ref %.3e | fwd ours %.3e ref %.3e | frob ours %.3e ref %.3e" % tuple(gm))
