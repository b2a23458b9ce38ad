"""Parity at the BASELINE.json configuration families, on the SAME matrix.

The reference (oracle/_ref, unmodified sources) builds A from the reference's
point sets; that A is uploaded unchanged, factored by both implementations, and
the north-star gates of BASELINE.json are checked against the reference's own
numbers:
  * ||A - LL^T||_F / ||A||_F (64-probe Hutchinson, identical probes) <= 2x ref
  * backward and forward solve error <= 2x ref
  * per-tile rank distribution of L: mean and L bytes within 10 %, p50 / p90 /
    p99 within 10 % or 1
  * the reference's own residual contract ||A - LL^T||_2 <= 10 nb eps
    (test_factor.cpp:96, acceptance.cpp:154)
Sizes: config 1 in full; configs 2-4 at the headline tile size m and bs with N
cut to what the host reference factors in seconds (the full sizes run through
bench.py --check)."""
import numpy as np
import pytest

from helpers import points, to_gpu
from paper_2108_11932_b200 import geometry as G

pytestmark = pytest.mark.gpu

SEED = 12345

FAMILIES = [
    # id, points, N, m, eps, bs, kernel, ell, nugget, mode (0 Chol, 1 LDL^T)
    ("cfg1", G.GRID2D, 16384, 256, 1e-6, 16, 0, 0.1, 0.0, 0),
    ("cfg2-family", G.GRID2D, 32768, 512, 1e-2, 16, 0, 0.1, 0.0, 0),
    ("cfg3-family", G.GRID3D, 8192, 512, 1e-4, 32, 1, 0.2, 1e-4, 1),
    ("cfg4-family", G.GRID3D, 16384, 1024, 1e-3, 32, 0, 0.2, 0.0, 0),
]


def _gates(acc, ref_acc, nb, eps, mode, solve=True):
    assert acc["resid_frob_rel"] <= 2.0 * ref_acc["resid_frob_rel"], (acc, ref_acc)
    if solve:
        assert acc["backward_err"] <= 2.0 * ref_acc["backward_err"], (acc, ref_acc)
        assert acc["forward_err"] <= 2.0 * ref_acc["forward_err"], (acc, ref_acc)
    rm, rr = acc["L_rank_mean"], ref_acc["L_rank_mean"]
    assert abs(rm - rr) <= 0.1 * rr, (rm, rr)
    lb, lr = acc["L_lowrank_bytes"], ref_acc["L_lowrank_bytes"]
    assert abs(lb - lr) <= 0.1 * lr, (lb, lr)
    for p in ("L_rank_p50", "L_rank_p90", "L_rank_p99"):
        a, r = acc[p], ref_acc[p]
        assert abs(a - r) <= max(1, 0.1 * r), (p, a, r)
    if mode == 0:
        assert acc["resid_2norm"] <= 10 * nb * eps


@pytest.mark.parametrize("fam", FAMILIES, ids=[f[0] for f in FAMILIES])
def test_config_family_parity_on_reference_built_matrix(tg, ref, fam):
    name, kind, n, b, eps, bs, kern, ell, nug, mode = fam
    pts = points(kind, n, b, 0)
    A_ref = ref.build(pts, kern, ell, nug, b, eps, 0, bs, SEED)
    F_ref = ref.factor(A_ref, mode, bs=bs, eps=eps, seed=SEED)
    ref_acc = ref.accuracy(A_ref, F_ref)
    A = to_gpu(tg, A_ref)
    cfg = tg.AraConfig(block_samples=bs, eps=eps, seed=SEED)
    factor = tg.tlr_cholesky if mode == 0 else tg.tlr_ldlt
    F = factor(A.copy(), cfg)
    acc = tg.tlr.accuracy(A, F)
    # LDL^T on the nugget-1e-4 Gaussian kernel: kappa ~ 1e7, and the solve errors
    # of BOTH implementations swing 10x with the ARA seed (tools/seed_sweep.py:
    # 3.7e-5 .. 4.0e-4 backward at N = 8,192).  A single-seed ratio is noise
    # there, so the solve gate is on the geometric mean over seeds below.
    _gates(acc, ref_acc, A.nb, eps, mode, solve=(mode == 0))
    # draw-for-draw streams: the rank maps agree tile by tile almost everywhere
    assert (F.L.ranks() == F_ref.L_ranks()).mean() >= 0.9


def test_accuracy_estimators_match_the_oracle_on_one_factor(tg, ref):
    """The device Frobenius estimator, exact ||A||_F and 2-norm power
    iteration agree with the oracle's restatement on the same A and L."""
    pts = points(G.GRID2D, 4096, 256, 0)
    A_ref = ref.build(pts, 0, 0.1, 0.0, 256, 1e-4, 0, 16, SEED)
    F_ref = ref.factor(A_ref, 0, bs=16, eps=1e-4, seed=SEED, schur_compensation=False)
    A = to_gpu(tg, A_ref)
    F = tg.tlr_cholesky(A.copy(), tg.AraConfig(block_samples=16, eps=1e-4, seed=SEED),
                        opts=tg.FactorOptions(schur_compensation=False))
    assert (F.L.ranks() == F_ref.L_ranks()).all()
    fa, fr = tg.tlr.frob_norm(A), ref.frob_norm(A_ref)
    assert abs(fa - fr) <= 1e-12 * fr
    # same probes, factors equal to ~1e-9: estimates agree to a few digits
    ea, er = tg.tlr.estimate_frob_diff(A, F, 64, 23), ref.estimate_frob_diff(A_ref, F_ref, 64, 23)
    assert abs(ea - er) <= 1e-3 * er, (ea, er)
    # the Hutchinson estimate brackets the exact ||A - LL^T||_F of the dense expansion
    Ad, Ld = A.dense(), np.tril(F.L.dense())
    exact = np.linalg.norm(Ad - Ld @ Ld.T)
    assert 0.7 * exact <= ea <= 1.3 * exact, (ea, exact)


def test_bs32_chol_ara_update_matches_reference_tile_by_tile(tg, ref):
    """bs = 32 (configs 3-5) column ARA at m = 256 with a left-looking history:
    equal ranks and rounds per tile, Q B^T within 1e-9 (test_ara.cpp:294-318)."""
    from helpers import covariance_ref
    A_ref = covariance_ref(ref, 2048, 256, 1e-6, bs=32)
    A = to_gpu(tg, A_ref)
    for k in (0, 3):
        cfg = tg.AraConfig(block_samples=32, eps=1e-6, seed=9)
        got = tg.chol_ara_update(A, None, k, cfg)
        want = ref.chol_ara_update(A_ref, k, bs=32, eps=1e-6, seed=9)
        assert [t.i for t in got] == [t["i"] for t in want]
        for g, w in zip(got, want):
            assert g.Q.shape[1] == w["Q"].shape[1], (k, g.i, g.Q.shape, w["Q"].shape)
            assert g.rounds_resident == w["rounds"]
            d1, d2 = g.Q @ g.B.T, w["Q"] @ w["B"].T
            assert np.abs(d1 - d2).max() <= 1e-9 * max(np.linalg.norm(d2), 1.0)


@pytest.mark.parametrize("n,b,bs", [(1000, 128, 16), (1000, 128, 32), (2500, 256, 16)])
def test_short_last_tile_factor_matches_reference(tg, ref, n, b, bs):
    """n % b != 0: the last tile row is short, so the last columns' ARA has only
    tiles shorter than the diagonal block (the exit projection is wider than the
    tile)."""
    eps = 1e-6
    pts = points(G.GRID2D, n, b, 0)
    A_ref = ref.build(pts, 0, 0.1, 0.0, b, eps, 0, bs, SEED)
    F_ref = ref.factor(A_ref, 0, bs=bs, eps=eps, seed=SEED)
    A = to_gpu(tg, A_ref)
    F = tg.tlr_cholesky(A.copy(), tg.AraConfig(block_samples=bs, eps=eps, seed=SEED))
    acc, ref_acc = tg.tlr.accuracy(A, F), ref.accuracy(A_ref, F_ref)
    assert acc["resid_frob_rel"] <= 2.0 * ref_acc["resid_frob_rel"]
    assert acc["backward_err"] <= 2.0 * ref_acc["backward_err"]
    assert acc["resid_2norm"] <= 10 * A.nb * eps
    rk, rkr = F.L.ranks(), F_ref.L_ranks()
    assert abs(rk.mean() - rkr.mean()) <= 0.1 * rkr.mean()
    # the short row's tiles specifically
    nb = A.nb
    last = [(nb - 1) * (nb - 2) // 2 + j for j in range(nb - 1)]
    assert np.abs(rk[last].astype(int) - rkr[last].astype(int)).max() <= 1


def test_factor_of_a_borrowed_L_view_copies_it(tg, ref):
    """tlr_cholesky(F.L, ...) deep-copies the borrowed view (the reference copies
    F.L into its by-value argument) and leaves F intact."""
    pts = points(G.GRID2D, 1024, 128, 0)
    A_ref = ref.build(pts, 0, 0.1, 0.5, 128, 1e-6, 0, 16, SEED)
    F = tg.tlr_cholesky(to_gpu(tg, A_ref), tg.AraConfig(block_samples=16, eps=1e-6, seed=1))
    before = F.L.ranks().copy()
    d0 = F.L.to_parts()[0][1].copy()
    view = F.L
    try:  # L as a symmetric TLR matrix need not be SPD: success or a clean error
        F2 = tg.tlr_cholesky(view, tg.AraConfig(block_samples=16, eps=1e-6, seed=1))
        del F2
    except tg.tlr.Error:
        pass
    assert (F.L.ranks() == before).all()
    assert np.array_equal(F.L.to_parts()[0][1], d0)
    assert view.ranks().shape == before.shape


def test_ldlt_solve_error_over_seeds(tg, ref):
    """cfg3 family (LDL^T, bs = 32, m = 512): backward and forward solve error
    within 2x of the reference as the geometric mean over sixteen ARA seeds, on
    the same reference-built A.  Either side's per-seed errors are heavy-tailed
    (Bunch-Kaufman pivot choices flip under O(1e-12) perturbations of the
    panels; the reference alone spans 2.7e-5 .. 6.0e-3 backward error over
    seeds 1-16), so four seeds did not pin the mean (tools/ldlt_seeds.py)."""
    n, b, eps, bs = 8192, 512, 1e-4, 32
    A_ref = ref.build(points(G.GRID3D, n, b, 0), 1, 0.2, 1e-4, b, eps, 0, bs, SEED)
    A = to_gpu(tg, A_ref)
    ours, theirs = [], []
    for sd in range(1, 17):
        F_ref = ref.factor(A_ref, 1, bs=bs, eps=eps, seed=sd)
        ra = ref.accuracy(A_ref, F_ref)
        oa = tg.tlr.accuracy(A, tg.tlr_ldlt(A.copy(), tg.AraConfig(block_samples=bs, eps=eps,
                                                                    seed=sd)))
        ours.append([oa["backward_err"], oa["forward_err"]])
        theirs.append([ra["backward_err"], ra["forward_err"]])
    go = np.exp(np.log(np.array(ours)).mean(axis=0))
    gr = np.exp(np.log(np.array(theirs)).mean(axis=0))
    assert (go <= 2.0 * gr).all(), (go, gr, ours, theirs)
