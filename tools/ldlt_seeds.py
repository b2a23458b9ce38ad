"""Dev tool: LDL^T solve errors over ARA seeds (cfg3 family) for A/B switches."""
import sys, os, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2108_11932_b200 as tg
from paper_2108_11932_b200 import geometry as G
from oracle import ref
from helpers import points, to_gpu
SEED = 12345
n, b, eps, bs = 8192, 512, 1e-4, 32
A_ref = ref.build(points(G.GRID3D, n, b, 0), 1, 0.2, 1e-4, b, eps, 0, bs, SEED)
A = to_gpu(tg, A_ref)
seeds = [int(x) for x in sys.argv[1:]] or [1, 2, 4, SEED, 7, 11]
for sd in seeds:
    F = tg.tlr_ldlt(A.copy(), tg.AraConfig(block_samples=bs, eps=eps, seed=sd))
    oa = tg.tlr.accuracy(A, F)
    ra = ref.accuracy(A_ref, ref.factor(A_ref, 1, bs=bs, eps=eps, seed=sd))
    print("ref %.3e %.3f" % (ra["backward_err"], ra["forward_err"]), "ours", sd, "%.3e %.3f" % (oa["backward_err"], oa["forward_err"]), "rankmean %.3f" % F.L.ranks().mean(), flush=True)
