"""Dev tool: build one config on the device and factor it once (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_11932_b200 as tg
from paper_2108_11932_b200.tlr import build_tlr
import bench
cfgname = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
kind, n, b, eps, bs, kern, ell, nug, mode = bench.CONFIGS[cfgname]
A = build_tlr(bench.problem_points(cfgname), kern, ell, nug, b, eps,
              cfg=tg.AraConfig(block_samples=bs, seed=12345))
ctx = A.ctx
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1  # > 1: warm repeats (the last is profiled)
for rep in range(reps):
    if rep == reps - 1:
        ctx.lib.tlrg_profiler(1)
        print("=== profiled run", file=sys.stderr, flush=True)
    Ain = A.copy() if rep < reps - 1 else A
    F = (tg.tlr_cholesky if mode == 0 else tg.tlr_ldlt)(Ain, tg.AraConfig(block_samples=bs, eps=eps, seed=12345))
    print("t_device", F.stats.t_device, "launches", F.stats.kernel_launches, flush=True)
    del F
ctx.lib.tlrg_profiler(0)
