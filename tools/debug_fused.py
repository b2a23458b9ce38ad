"""Dev tool: fused vs graph-loop ARA on the same column (per-tile ranks, rounds, QB^T)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2108_11932_b200 as tg
from oracle import ref
from helpers import covariance_ref, to_gpu
A_ref = covariance_ref(ref, 768, 128, 1e-6)
for k, eps, seed in [(1, 1e-5, 1234), (0, 1e-6, 88), (3, 1e-8, 5)]:
    A = to_gpu(tg, A_ref)
    cfg = tg.AraConfig(block_samples=16, eps=eps, seed=seed)
    os.environ["TLRG_NO_FUSED"] = "1"
    a = tg.chol_ara_update(A, None, k, cfg)
    os.environ["TLRG_NO_FUSED"] = "0"
    b = tg.chol_ara_update(A, None, k, cfg)
    w = ref.chol_ara_update(A_ref, k, bs=16, eps=eps, seed=seed, parallel_buffers=16, subset_capacity=2)
    for x, y, z in zip(a, b, w):
        d = np.abs(x.Q @ x.B.T - y.Q @ y.B.T).max() if x.Q.shape[1] and y.Q.shape[1] else -1
        print(k, x.i, "graph", x.Q.shape[1], x.rounds_resident, "fused", y.Q.shape[1], y.rounds_resident,
              "ref", z["Q"].shape[1], z["rounds"], "diff %.2e" % d)
