"""Dev tool: per-step device time of repeated factorizations (run-to-run spread)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_11932_b200 as tg
from paper_2108_11932_b200.tlr import build_tlr
import bench
cfgname = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
kind, n, b, eps, bs, kern, ell, nug, mode = bench.CONFIGS[cfgname]
A = build_tlr(bench.problem_points(cfgname), kern, ell, nug, b, eps,
              cfg=tg.AraConfig(block_samples=bs, seed=12345))
fac = tg.tlr_cholesky if mode == 0 else tg.tlr_ldlt
cfg = tg.AraConfig(block_samples=bs, eps=eps, seed=12345)
for r in range(reps):
    B = A.copy()
    t0 = time.perf_counter()
    F = fac(B, cfg)
    w = time.perf_counter() - t0
    s = F.stats
    print(f"rep {r}: dev {s.t_device:.4f} wall {w:.4f} fused {s.t_ara_kernel:.4f} comp {s.t_compensation:.4f} "
          f"rec {s.t_recompress:.4f} samp {s.t_sampling:.4f}", flush=True)
    del F, B
