"""Diagnose a solve-error gap: backward error of (our factor, our solve),
(our factor -> TLRF -> reference solve), (reference factor, reference solve)
on the same reference-built A (cfg3 family by default)."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2108_11932_b200 as tg  # noqa: E402
from helpers import points, to_gpu  # noqa: E402
from oracle import ref  # noqa: E402
from paper_2108_11932_b200 import geometry as G  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
b, eps, bs, SEED = 512, 1e-4, 32, 12345
pts = points(G.GRID3D, n, b, 0)
A_ref = ref.build(pts, 1, 0.2, 1e-4, b, eps, 0, bs, SEED)
F_ref = ref.factor(A_ref, 1, bs=bs, eps=eps, seed=SEED)
A = to_gpu(tg, A_ref)
F = tg.tlr_ldlt(A.copy(), tg.AraConfig(block_samples=bs, eps=eps, seed=SEED))
x = ref.rng_gaussians(7, n)
bb = A_ref.matvec(x)


def bwd(xs):
    return float(np.linalg.norm(A_ref.matvec(xs) - bb) / np.linalg.norm(bb))


print("ours/ours   ", bwd(tg.factor_solve(F, bb)))
F.write("/tmp/ours.tlrf")
st = C.c_int()
h = ref.lib().ref_factor_read(b"/tmp/ours.tlrf", C.byref(st))
Fo = ref.RefFactor(h)
print("ours/refslv ", bwd(Fo.solve(bb)))
print("ref/ref     ", bwd(F_ref.solve(bb)))
# the factors' 2-norm residuals against the same A
print("resid2 ours ", tg.estimate_2norm_diff(A, F, 50, 17), " ref ", ref.estimate_2norm_diff(A_ref, F_ref, 50, 17))
print("resid2 ours via ref ", ref.estimate_2norm_diff(A_ref, Fo, 50, 17))
# per-column D pivots: smallest |d|
dmin_o = min(np.min(np.abs(d.d)) for d in F.D)
dmin_r = min(np.min(np.abs(F_ref.dblock(k)[0])) for k in range(A.nb))
print("min|d| ours", dmin_o, "ref", dmin_r)
# per-column pivot trace (min |eigenvalue| of the D blocks)
pt_o = np.asarray(F.stats.pivot_trace)
pt_r = np.asarray(F_ref.stats().pivot_trace)
print("pivot_trace ours", np.array2string(pt_o, precision=3))
print("pivot_trace ref ", np.array2string(pt_r, precision=3))
# column 0 is exact input: our Bunch-Kaufman vs LAPACK dsytrf on the same tile
A00 = A_ref.diag(0)
Lo, Do, po, info = tg.tlr.dense_ldl(A00)
Lr, dr, er, s2r, pr = ref.dense_ldl(A00)
print("col0 perm equal", bool((po == pr).all()), "2x2 equal", bool((Do.start2x2 == s2r).all()),
      "min|d| ours", np.min(np.abs(Do.d)), "ref", np.min(np.abs(dr)),
      "max|dL|", np.max(np.abs(Lo - Lr)))
