"""Dev tool: hash of a factor's L (ranks, diagonal, U/V) for bitwise A/B of
kernel changes that must not change arithmetic: python tools/factor_hash.py cfg4 16384"""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2108_11932_b200 as tg
from paper_2108_11932_b200 import geometry as G
import bench
name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
kind, n, b, eps, bs, kern, ell, nug, mode = bench.CONFIGS[name]
n = int(sys.argv[2]) if len(sys.argv) > 2 else n
pts = bench.problem_points(name, n)
A = tg.tlr.build_tlr(pts, kern, ell, nug, b, eps, cfg=tg.AraConfig(block_samples=bs, seed=12345))
F = (tg.tlr_cholesky if mode == 0 else tg.tlr_ldlt)(A, tg.AraConfig(block_samples=bs, eps=eps, seed=12345))
h = hashlib.sha256()
for part in F.L.to_parts():
    if isinstance(part, (list, tuple)):
        for x in part:
            h.update(np.ascontiguousarray(x).tobytes())
    else:
        h.update(np.ascontiguousarray(part).tobytes())
print(name, n, "L hash", h.hexdigest()[:16], "mean rank %.4f" % F.L.ranks().mean())
