import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2108_11932_b200 as tg
from helpers import covariance_ref, to_gpu
from oracle import ref
A_ref = covariance_ref(ref, 4096, 256, 1e-6, bs=32, seed=42)
A = to_gpu(tg, A_ref)
for rep in range(3):
    F = tg.tlr_cholesky(A.copy(), tg.AraConfig(block_samples=32, eps=1e-6, seed=5))
    s = F.stats
    print(rep, {k: round(getattr(s, k), 5) for k in ("t_sampling", "t_projection", "t_reduction", "t_dense", "t_orthog", "t_misc", "t_recompress", "t_compensation", "wall")}, flush=True)
