"""FactorStats phase split of one factorization (the reference's phase
accounting test case: ball3d 4096 / 256, eps 1e-6, bs 32) for ours and the
reference."""
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2108_11932_b200 as tg  # noqa: E402
from helpers import covariance_ref, to_gpu  # noqa: E402
from oracle import ref  # noqa: E402

n, b, eps, bs = int(sys.argv[1]) if len(sys.argv) > 1 else 4096, 256, 1e-6, 32
A_ref = covariance_ref(ref, n, b, eps, bs=bs, seed=42)
A = to_gpu(tg, A_ref)
for _ in range(2):
    F = tg.tlr_cholesky(A.copy(), tg.AraConfig(block_samples=bs, eps=eps, seed=5))
s = F.stats
print({k: round(getattr(s, k), 5) for k in ("t_sampling", "t_projection", "t_reduction", "t_dense",
                                             "t_orthog", "t_misc", "t_recompress",
                                             "t_compensation", "wall", "t_device")})
r = ref.factor(A_ref, 0, bs=bs, eps=eps, seed=5).stats()
print("ref", {k: round(getattr(r, k), 5) for k in ("t_sampling", "t_projection", "t_reduction",
                                                   "t_dense", "t_orthog", "t_misc", "wall")})
