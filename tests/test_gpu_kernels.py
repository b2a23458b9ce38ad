"""GPU parity of the building blocks against the oracle (the unmodified
reference compiled under oracle/_ref) and numpy.  Mirrors test_dense.cpp /
test_ara.cpp cases."""
import numpy as np
import pytest

from helpers import covariance_ref, dblocks_np, to_gpu

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N,K,ta,tb", [(64, 32, 16, 0, 0), (100, 17, 33, 1, 0), (7, 129, 65, 0, 1),
                                         (130, 70, 1, 1, 1), (512, 16, 512, 1, 0), (3, 3, 0, 0, 0),
                                         # large-tile kernels (128 x 64 / 128 x 32, 3 stages)
                                         (512, 512, 300, 0, 1), (1024, 96, 257, 0, 0),
                                         (513, 64, 600, 1, 1), (2048, 32, 401, 0, 1),
                                         (1537, 30, 500, 0, 0)])
def test_grouped_dmma_gemm_matches_numpy(tg, M, N, K, ta, tb):
    r = np.random.default_rng(M * 1000 + N)
    A = r.normal(size=(K, M) if ta else (M, K))
    B = r.normal(size=(N, K) if tb else (K, N))
    C0 = r.normal(size=(M, N))
    want = 0.7 * ((A.T if ta else A) @ (B.T if tb else B)) - 0.3 * C0
    got = tg.tlr.gemm(0.7, A, ta, B, tb, -0.3, C0)
    assert np.abs(got - want).max() <= 1e-13 * max(1.0, np.abs(want).max()) * max(K, 1)


@pytest.mark.parametrize("seed", [0, 1, 12345, 2**63 + 5])
def test_device_rng_draw_for_draw(tg, ref, seed):
    n = 20001
    got = tg.tlr.rng_gaussians(seed, n)
    want = ref.rng_gaussians(seed, n)
    assert np.abs(got - want).max() <= 4e-15 * np.abs(want).max()


@pytest.mark.parametrize("rows,q,k,case", [(96, 0, 16, "plain"), (128, 20, 16, "plain"),
                                           (64, 8, 8, "dup"), (64, 0, 8, "zero"),
                                           (200, 40, 32, "lowrank")])
def test_orthog_matches_reference(tg, ref, rows, q, k, case):
    r = np.random.default_rng(rows + q + k)
    Q = np.linalg.qr(r.normal(size=(rows, q)))[0] if q else None
    if case == "plain":
        Y = r.normal(size=(rows, k))
    elif case == "dup":
        Y = r.normal(size=(rows, k))
        Y[:, 3] = Y[:, 1]
        Y[:, 5] = 2 * Y[:, 0] - Y[:, 2]
    elif case == "zero":
        Y = np.zeros((rows, k))
    else:
        Y = r.normal(size=(rows, 3)) @ r.normal(size=(3, k))
        if q:
            Y += Q @ r.normal(size=(q, k))
    Yg, Rg, cg, mg, ng = tg.tlr.orthog(Q, Y, 77)
    Yr, Rr, cr, mr, nr = ref.orthog(Q, Y, 77)
    scale = max(np.abs(Y).max(), 1.0)
    assert np.abs(cg - cr).max() <= 1e-12 * scale
    assert np.abs(mg - mr).max() <= 1e-12 * scale
    assert np.abs(Rg - Rr).max() <= 1e-11 * scale
    # healthy columns agree; replaced columns are random directions drawn from
    # the same stream and agree as well
    assert np.abs(Yg - Yr).max() <= 1e-9
    assert ng == pytest.approx(nr, rel=1e-12, abs=1e-14)


def test_sample_left_matches_reference_chol(tg, ref):
    A_ref = covariance_ref(ref, 1024, 128, 1e-8)
    A = to_gpu(tg, A_ref)
    k = 5
    rows = list(range(k + 1, A.nb))
    r = np.random.default_rng(23)
    om = [r.normal(size=(128, 16)) for _ in rows]
    got = tg.sample_left(A, None, k, rows, tg.AraWorkspace(parallel_buffers=32), om)
    want = ref.sample_left(A_ref, k, rows, om, parallel_buffers=32)
    for g, w, o in zip(got, want, om):
        assert np.linalg.norm(g - w) <= 1e-11 * max(np.linalg.norm(w), 1.0) * np.linalg.norm(o)
    # transpose mode (projection)
    q = [np.linalg.qr(r.normal(size=(128, 9)))[0] for _ in rows]
    got = tg.sample_left_transpose(A, None, k, rows, tg.AraWorkspace(parallel_buffers=32), q)
    want = ref.sample_left(A_ref, k, rows, q, parallel_buffers=32, transpose=True)
    for g, w in zip(got, want):
        assert np.linalg.norm(g - w) <= 1e-11 * max(np.linalg.norm(w), 1.0)


def test_sample_left_ldl_inserts_d(tg, ref):
    A_ref = covariance_ref(ref, 512, 128, 1e-8)
    A = to_gpu(tg, A_ref)
    D = dblocks_np(A.nb, [128] * A.nb, 99)
    r = np.random.default_rng(29)
    om = [r.normal(size=(128, 8))]
    got = tg.sample_left(A, D, 2, [3], tg.AraWorkspace(), om)
    want = ref.sample_left(A_ref, 2, [3], om, D=D)
    assert np.linalg.norm(got[0] - want[0]) <= 1e-11 * np.linalg.norm(want[0]) * np.linalg.norm(om[0])


def test_sample_left_rejects_undersized_workspace(tg, ref):
    A = to_gpu(tg, covariance_ref(ref, 384, 96, 1e-6))
    with pytest.raises(tg.ConfigError):
        tg.sample_left(A, None, 0, [1, 2, 3], tg.AraWorkspace(parallel_buffers=2),
                       [np.zeros((96, 4))] * 3)


@pytest.mark.parametrize("k,eps,seed", [(1, 1e-5, 1234), (0, 1e-6, 88), (3, 1e-8, 5)])
def test_chol_ara_update_matches_reference(tg, ref, k, eps, seed):
    """Same seeds -> same draws: ranks equal and Q B^T within 1e-9
    (test_ara.cpp:294-318 standard)."""
    A_ref = covariance_ref(ref, 768, 128, 1e-6)
    A = to_gpu(tg, A_ref)
    cfg = tg.AraConfig(block_samples=16, eps=eps, seed=seed)
    got = tg.chol_ara_update(A, None, k, cfg, tg.AraWorkspace(parallel_buffers=16,
                                                               subset_capacity=2))
    want = ref.chol_ara_update(A_ref, k, bs=16, eps=eps, seed=seed, parallel_buffers=16,
                               subset_capacity=2)
    assert [t.i for t in got] == [t["i"] for t in want]
    for g, w in zip(got, want):
        assert g.Q.shape[1] == w["Q"].shape[1], (g.i, g.Q.shape, w["Q"].shape)
        assert g.rounds_resident == w["rounds"]
        assert g.converged == w["converged"]
        d1, d2 = g.Q @ g.B.T, w["Q"] @ w["B"].T
        assert np.abs(d1 - d2).max() <= 1e-9 * max(np.linalg.norm(d2), 1.0)
        if g.Q.shape[1]:
            G = g.Q.T @ g.Q
            assert np.linalg.norm(G - np.eye(G.shape[0])) <= 1e-11


def test_chol_ara_update_zero_rank_column(tg, ref):
    from helpers import points
    from paper_2108_11932_b200 import geometry as G
    pts = points(G.GRID2D, 256, 64)
    A_ref = ref.build(pts, 0, 1e-5, 0.5, 64, 1e-6, 1, 32, 0)
    A = to_gpu(tg, A_ref)
    out = tg.chol_ara_update(A, None, 0, tg.AraConfig(eps=1e-6), tg.AraWorkspace())
    assert len(out) == 3
    for t in out:
        assert t.converged and t.rounds_resident == 0 and t.Q.shape[1] == 0


@pytest.mark.parametrize("n", [1, 31, 64, 100, 256, 512])
def test_potrf_matches_reference(tg, ref, n):
    r = np.random.default_rng(n)
    G = r.normal(size=(n, n))
    A = G @ G.T + 0.1 * n * np.eye(n)
    L, fail = tg.tlr.dense_cholesky(A)
    assert fail == -1
    assert np.abs(L - np.linalg.cholesky(A)).max() <= 1e-12 * np.abs(A).max()
    B = A.copy()
    B[n // 2, n // 2] = -1.0
    _, fail = tg.tlr.dense_cholesky(B)
    assert fail >= 0


def test_chol_ara_update_split_k_sampling(tg, ref):
    """Graph path (bs = 32, m = 512) at a column whose sampling reduction
    K = sum_j rank(k, j) exceeds 1024, so the H-product is split into K chunks
    summed by the stacked-identity GEMM: per tile the same rank, rounds and
    convergence as the reference, factors within 1e-9 (test_ara.cpp:294-318)."""
    from helpers import points
    from paper_2108_11932_b200 import geometry as G
    n, b, eps, bs, k = 512 * 18, 512, 1e-6, 32, 15
    A_ref = ref.build(points(G.GRID3D, n, b, 0), 1, 0.2, 1e-4, b, eps, 0, bs, 12345)
    A = to_gpu(tg, A_ref)
    rk = A.ranks()
    K = sum(int(rk[k * (k - 1) // 2 + j]) for j in range(k))
    assert K >= 1024, K  # the split-K path is taken
    cfg = tg.AraConfig(block_samples=bs, eps=eps, seed=91)
    got = tg.chol_ara_update(A, None, k, cfg, tg.AraWorkspace())
    want = ref.chol_ara_update(A_ref, k, bs=bs, eps=eps, seed=91)
    assert [t.i for t in got] == [t["i"] for t in want]
    for g, w in zip(got, want):
        assert (g.Q.shape[1], g.rounds_resident, g.converged) == \
            (w["Q"].shape[1], w["rounds"], w["converged"]), g.i
        d1, d2 = g.Q @ g.B.T, w["Q"] @ w["B"].T
        assert np.abs(d1 - d2).max() <= 1e-9 * max(np.linalg.norm(d2), 1.0)


def _decaying(r, m, n, decades=10.0):
    U, _ = np.linalg.qr(r.normal(size=(m, n)))
    W, _ = np.linalg.qr(r.normal(size=(n, n)))
    return (U * np.logspace(2, 2 - decades, n)) @ W.T


@pytest.mark.parametrize("n", [150, 276])
def test_wide_jacobi_cluster_is_bitwise_the_one_cta_kernel(tg, n):
    """Square recompression cores wider than shared memory: the cluster kernel
    runs the 1-CTA kernel's pair schedule, so every output is bitwise equal."""
    A = _decaying(np.random.default_rng(n), n, n)
    cut = 1e-3
    a = tg.tlr.jacobi_svd(A, cut)
    b = tg.tlr.jacobi_svd(A, cut, force_single=True)
    for x, y in zip(a[:3], b[:3]):
        assert np.array_equal(x, y)
    assert a[3] == b[3]


@pytest.mark.parametrize("m,n", [(1024, 276), (1024, 130), (512, 200), (256, 140)])
def test_wide_jacobi_on_the_basis_matches_numpy_svd(tg, m, n):
    """Wide ARA bases are recompressed by Jacobi on B itself (svd_truncate of
    B's R factor, dense_kernels.cpp:422-454, without the QR): singular values,
    rank at the cut and the factorization B V = U S."""
    r = np.random.default_rng(m + n)
    A = _decaying(r, m, n, decades=12.0)
    s_ref = np.linalg.svd(A, compute_uv=False)
    cut = np.sqrt(s_ref[n // 2] * s_ref[n // 2 + 1])  # away from any singular value
    US, V, sig, rank = tg.tlr.jacobi_svd(A, cut)
    assert rank == int((s_ref > cut).sum())
    assert np.abs(sig - s_ref).max() <= 1e-13 * s_ref[0] * n
    assert np.abs(V.T @ V - np.eye(n)).max() <= 1e-12
    assert np.abs(US @ V.T - A).max() <= 1e-12 * s_ref[0]
    assert np.allclose(np.linalg.norm(US, axis=0), sig, rtol=0, atol=1e-13 * s_ref[0])


@pytest.mark.parametrize("n,kind", [(5, "indef"), (64, "indef"), (128, "spd"), (200, "indef"),
                                    (512, "indef")])
def test_bunch_kaufman_matches_reference(tg, ref, n, kind):
    r = np.random.default_rng(n + 7)
    G = r.normal(size=(n, n))
    A = (G + G.T) / 2 if kind == "indef" else G @ G.T + n * np.eye(n)
    L, D, perm, info = tg.tlr.dense_ldl(A)
    Lr, dr, er, s2r, pr = ref.dense_ldl(A)
    P = A[np.ix_(perm, perm)]
    rec = L @ D.materialize() @ L.T
    assert np.abs(rec - P).max() <= 1e-11 * np.abs(A).max() * n
    # LAPACK's pivot decisions are reproduced (ties aside): same block structure
    assert (D.start2x2 == s2r).mean() >= 0.95
    assert np.allclose(np.sort(perm), np.arange(n))


def test_schur_compensation_matches_reference(tg, ref):
    """compensation_with_norm (factor.cpp:66-79) vs the reference's full SVD.
    The sketch (width <= 112, one power step) resolves the directions near eps
    to ~1e-5 relative in the row sums; an eps-rank above one sketch (104
    directions) goes through the chunked spectrum split, whose deflated Ritz
    pairs are exact to ~1e-4 relative.  Either way the absolute error is
    ~1e-5 eps, far below the eps-level correction itself."""
    r = np.random.default_rng(3)
    for n, rank, eps, rtol in [(16, 6, 0.5, 1e-6), (128, 40, 1e-3, 1e-6), (256, 90, 1e-6, 2e-5),
                               (256, 120, 1e-6, 1e-4), (512, 300, 1e-6, 1e-4)]:
        G = r.normal(size=(n, rank)) * np.logspace(0, -8, rank)
        Dk = G @ G.T
        want = ref.schur_compensation(Dk, eps)
        got, frob = tg.tlr.schur_compensation(Dk, eps)
        assert np.abs(got - want).max() <= rtol * max(np.abs(want).max(), eps) + 1e-12, (n, rank)


@pytest.mark.parametrize("bs,eps,k", [(16, 1e-2, 5), (16, 1e-4, 9), (32, 1e-4, 5), (32, 1e-6, 2)])
def test_chol_ara_update_headline_tile_size(tg, ref, bs, eps, k):
    """chol_ara_update at the headline tile m = 512 (the fused kernel's two
    rows per thread at bs = 16; the graph path at bs = 32): per tile the same
    rank, rounds and convergence flag as the reference, factors within 1e-9
    (test_ara.cpp:294-318 standard), on a 2D exponential covariance matrix."""
    from helpers import points
    from paper_2108_11932_b200 import geometry as G
    n, b = 512 * 12, 512
    A_ref = ref.build(points(G.GRID2D, n, b, 0), 0, 0.1, 0.0, b, eps, 0, bs, 12345)
    A = to_gpu(tg, A_ref)
    cfg = tg.AraConfig(block_samples=bs, eps=eps, seed=77)
    got = tg.chol_ara_update(A, None, k, cfg, tg.AraWorkspace())
    want = ref.chol_ara_update(A_ref, k, bs=bs, eps=eps, seed=77)
    assert [t.i for t in got] == [t["i"] for t in want]
    for g, w in zip(got, want):
        assert (g.Q.shape[1], g.rounds_resident, g.converged) == \
            (w["Q"].shape[1], w["rounds"], w["converged"]), g.i
        d1, d2 = g.Q @ g.B.T, w["Q"] @ w["B"].T
        assert np.abs(d1 - d2).max() <= 1e-9 * max(np.linalg.norm(d2), 1.0)
