"""Probe: build + factor one config on the GPU and print phases (dev tool)."""
import sys, time, json, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2108_11932_b200 as tg
from paper_2108_11932_b200.tlr import build_tlr
import bench
cfgname = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
kind, n, b, eps, bs, kern, ell, nug, mode = bench.CONFIGS[cfgname]
pts = bench.problem_points(cfgname)
t = time.time()
A = build_tlr(pts, kern, ell, nug, b, eps, cfg=tg.AraConfig(block_samples=bs, seed=12345))
print("build", time.time() - t, "A ranks mean", A.ranks().mean(), flush=True)
cfg = tg.AraConfig(block_samples=bs, eps=eps, seed=12345)
for rep in range(2):
    t = time.time()
    F = (tg.tlr_cholesky if mode == 0 else tg.tlr_ldlt)(A.copy(), cfg)
    s = F.stats
    print("factor wall", time.time() - t, "dev", s.t_device, flush=True)
print({k: round(getattr(s, k), 4) for k in ["t_dense", "t_misc", "t_compensation", "t_sampling", "t_orthog", "t_projection", "t_recompress", "wall", "t_device"]})
print("flops exec", s.flops_exec / 1e9, "ref", s.flops_gemm_ref / 1e9, "launches", s.kernel_launches, "tile_rounds", s.tile_rounds_resident)
r = F.L.ranks(); print("L rank mean", r.mean(), "max", r.max())
print("resid", tg.estimate_2norm_diff(A, F, 30, 17))
