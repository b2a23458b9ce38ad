"""GPU path against the committed golden fixtures (no oracle at run time)."""
import numpy as np
import pytest

from golden_util import B, BS, EPS, N, SEED, load, tile_lists

pytestmark = pytest.mark.gpu


def test_device_rng_matches_golden(tg):
    g = load()
    for s in (0, 12345):  # same mt19937_64 draws; device vs libm log/sqrt last bits
        x = tg.rng_gaussians(s, 512)
        assert np.abs(x - g[f"rng_{s}"]).max() <= 4e-15 * np.abs(x).max()


def test_orthog_matches_golden(tg):
    g = load()
    Yo, R, cn, nm, nd = tg.orthog(g["orthog_Q"], g["orthog_Y_in"], 77)
    assert np.abs(R - g["orthog_R"]).max() <= 1e-12 * max(1.0, np.abs(g["orthog_R"]).max())
    assert np.abs(cn - g["orthog_cn"]).max() <= 1e-12 * max(1.0, cn.max())
    assert nd == g["orthog_next_draw"][0]


def test_cholesky_matches_golden_factor(tg):
    g = load()
    d, rk, U, V = tile_lists(g)
    A = tg.TlrMatrix.from_parts(N, B, EPS, d, rk, U, V)
    Akeep = A.copy()
    F = tg.tlr_cholesky(A, tg.AraConfig(block_samples=BS, eps=EPS, seed=SEED))
    r = tg.estimate_2norm_diff(Akeep, F, 50, 17)
    assert r <= 2.0 * g["resid_2norm"][0] and r <= 10 * (N // B) * EPS
    assert (F.L.ranks() == g["L_ranks"]).mean() >= 0.95
    assert (F.stats.ara_rounds == g["L_ara_rounds"]).mean() >= 0.75
