"""Pivoted TLR Cholesky (Alg. 8, factor.cpp:140-209), the TLRM / TLRF file
formats against the reference's own writers and readers, and the pivot trace.

Parity standard for pivoting: the same tile permutation as the reference on the
same A (the identity / reversed-permutation cases of test_factor.cpp:167-219
run unmodified in tests/test_gpu_conformance.py), the reference's residual
contract ||PAP^T - LL^T||_2 <= 10 nb eps and within 2x of
the reference's residual, solves within 2x.  Files are compared byte for byte."""
import numpy as np
import pytest

from helpers import covariance_ref, points, to_gpu
from paper_2108_11932_b200 import geometry as G

pytestmark = pytest.mark.gpu


def scaled_ref(ref, scales, n=2048, b=128, eps=1e-6, seed=42):
    """D_s A D_s with per-tile scales (test_factor.cpp:27-37): symmetric and
    definite, with a diagonal-norm ordering that pivoting must follow."""
    A = covariance_ref(ref, n, b, eps, seed=seed)
    diag, ranks, U, V = A.to_parts()
    nb = A.nb
    t = 0
    for i in range(nb):
        diag[i] = diag[i] * scales[i] ** 2
        for j in range(i):
            U[t] = U[t] * scales[i]
            V[t] = V[t] * scales[j]
            t += 1
    return ref.matrix_from_parts(n, b, eps, diag, ranks, U, V)


@pytest.mark.parametrize("order", ["decreasing", "increasing", "shuffled"])
@pytest.mark.parametrize("norm", [0, 1])
def test_pivoted_cholesky_matches_reference(tg, ref, order, norm):
    nb = 16
    base = np.linspace(3.0, 0.5, nb)
    scales = {"decreasing": base, "increasing": base[::-1],
              "shuffled": base[np.random.default_rng(3).permutation(nb)]}[order]
    eps = 1e-6
    A_ref = scaled_ref(ref, scales, eps=eps)
    F_ref = ref.factor(A_ref, 2, bs=16, eps=eps, seed=5, pivot_norm=norm)
    A = to_gpu(tg, A_ref)
    opts = tg.FactorOptions(pivot_norm=norm)
    F = tg.tlr_cholesky_pivoted(A.copy(), tg.AraConfig(block_samples=16, eps=eps, seed=5),
                                opts=opts)
    assert F.mode == 2
    assert F.perm == F_ref.perm()
    assert sorted(F.perm) == list(range(nb))
    r_gpu = tg.estimate_2norm_diff(A, F, 50, 17)
    r_ref = ref.estimate_2norm_diff(A_ref, F_ref, 50, 17)
    assert r_gpu <= 10 * nb * eps
    assert r_gpu <= 2.0 * r_ref + 1e-14, (r_gpu, r_ref)
    assert (F.L.ranks() == F_ref.L_ranks()).mean() >= 0.95
    # pivoted solve: backward error within 2x of the reference's
    x = ref.rng_gaussians(7, A.n)
    b = A_ref.matvec(x)
    bw = lambda xs: np.linalg.norm(A_ref.matvec(xs) - b) / np.linalg.norm(b)  # noqa: E731
    assert bw(tg.factor_solve(F, b)) <= 2.0 * bw(F_ref.solve(b)) + 1e-14


def test_pivoting_requires_uniform_tiles(tg, ref):
    A_ref = covariance_ref(ref, 1000, 128, 1e-4)
    A = to_gpu(tg, A_ref)
    with pytest.raises(tg.ConfigError):
        tg.tlr_cholesky_pivoted(A, tg.AraConfig(block_samples=16, eps=1e-4, seed=5))


def test_tlrm_bytes_identical_to_reference_writer(tg, ref, tmp_path):
    A_ref = covariance_ref(ref, 1000, 128, 1e-6)  # ragged last tile
    A = to_gpu(tg, A_ref)
    p1, p2 = str(tmp_path / "ours.tlrm"), str(tmp_path / "ref.tlrm")
    tg.write_tlr(A, p1)
    A_ref.write(p2)
    assert open(p1, "rb").read() == open(p2, "rb").read()
    # and each reader reads the other's file back to the same bytes
    B = tg.read_tlr(p2)
    p3 = str(tmp_path / "again.tlrm")
    tg.write_tlr(B, p3)
    assert open(p3, "rb").read() == open(p2, "rb").read()


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_tlrf_interop_with_reference(tg, ref, tmp_path, mode):
    """write_factor / read_factor (factor.cpp:308-395) both ways: our file read
    by the reference solves like our factor, the reference's file read by us
    solves like the reference's factor, and a file survives a round trip
    through the other implementation byte for byte."""
    n, b, eps = 1024, 128, 1e-6
    A_ref = covariance_ref(ref, n, b, eps) if mode != 1 else \
        covariance_ref(ref, n, b, eps, kernel=1, nugget=1e-3)
    A = to_gpu(tg, A_ref)
    cfg = tg.AraConfig(block_samples=16, eps=eps, seed=5)
    fac = {0: tg.tlr_cholesky, 1: tg.tlr_ldlt, 2: tg.tlr_cholesky_pivoted}[mode]
    F = fac(A.copy(), cfg)
    F_ref = ref.factor(A_ref, mode, bs=16, eps=eps, seed=5)
    bvec = np.sin(0.37 * np.arange(n) + 1.0)
    # ours -> reference
    p_o = str(tmp_path / "ours.tlrf")
    F.write(p_o)
    R = ref.read_factor(p_o)
    assert R.mode == mode
    xo = tg.factor_solve(F, bvec)
    assert np.abs(R.solve(bvec) - xo).max() <= 1e-10 * np.abs(xo).max()
    p_rr = str(tmp_path / "ours_via_ref.tlrf")
    R.write(p_rr)
    assert open(p_rr, "rb").read() == open(p_o, "rb").read()
    # reference -> ours
    p_r = str(tmp_path / "ref.tlrf")
    F_ref.write(p_r)
    Fo = tg.tlr.read_factor(p_r)
    assert Fo.mode == mode
    if mode == 2:
        assert Fo.perm == F_ref.perm()
    xr = F_ref.solve(bvec)
    assert np.abs(tg.factor_solve(Fo, bvec) - xr).max() <= 1e-10 * np.abs(xr).max()
    p_ro = str(tmp_path / "ref_via_ours.tlrf")
    Fo.write(p_ro)
    assert open(p_ro, "rb").read() == open(p_r, "rb").read()


def test_pivot_trace_matches_reference(tg, ref):
    """FactorStats::pivot_trace (factor.cpp:81-102): min diagonal pivot^2 of
    L_kk per column (Cholesky) and min |eigenvalue| of the D blocks (LDL^T)."""
    pts = points(G.GRID2D, 4096, 256, 0)
    A_ref = ref.build(pts, 0, 0.1, 0.0, 256, 1e-4, 0, 16, 12345)
    A = to_gpu(tg, A_ref)
    F_ref = ref.factor(A_ref, 0, bs=16, eps=1e-4, seed=12345, schur_compensation=False)
    F = tg.tlr_cholesky(A.copy(), tg.AraConfig(block_samples=16, eps=1e-4, seed=12345),
                        opts=tg.FactorOptions(schur_compensation=False))
    assert (F.L.ranks() == F_ref.L_ranks()).all()
    pg, pr = F.stats.pivot_trace, F_ref.stats().pivot_trace
    assert np.abs(pg - pr).max() <= 1e-8 * np.abs(pr).max()
    F_ref = ref.factor(A_ref, 1, bs=16, eps=1e-4, seed=12345)
    F = tg.tlr_ldlt(A.copy(), tg.AraConfig(block_samples=16, eps=1e-4, seed=12345))
    pg, pr = F.stats.pivot_trace, F_ref.stats().pivot_trace
    assert np.abs(pg - pr).max() <= 1e-8 * np.abs(pr).max()
