"""The oracle (the unmodified reference in oracle/_ref) and the host RNG port
reproduce the committed golden fixtures: pins the oracle build on every box."""
import numpy as np

from golden_util import BS, EPS, SEED, load, tile_lists
from paper_2108_11932_b200.mt64 import Mt64


def test_host_rng_port_matches_golden_streams():
    g = load()
    for s in (0, 12345):  # numpy vs libm log/sqrt: last-bit differences only
        x = Mt64(s).gaussians(512)
        assert np.abs(x - g[f"rng_{s}"]).max() <= 4e-15 * np.abs(x).max()


def test_oracle_reproduces_golden(ref):
    g = load()
    for s in (0, 12345):
        assert np.array_equal(ref.rng_gaussians(s, 512), g[f"rng_{s}"])
    Yo, R, cn, nm, nd = ref.orthog(g["orthog_Q"], g["orthog_Y_in"], 77)
    assert np.abs(R - g["orthog_R"]).max() <= 1e-12
    assert np.abs(cn - g["orthog_cn"]).max() <= 1e-12 and nd == g["orthog_next_draw"][0]
    d, rk, U, V = tile_lists(g)
    A = ref.matrix_from_parts(512, 64, EPS, d, rk, U, V)
    F = ref.factor(A, 0, bs=BS, eps=EPS, seed=SEED)
    assert np.array_equal(np.asarray(F.L_ranks()), g["L_ranks"])
    assert np.array_equal(np.asarray(F.stats().ara_rounds), g["L_ara_rounds"])
    r = ref.estimate_2norm_diff(A, F, 50, 17)
    assert abs(r - g["resid_2norm"][0]) <= 1e-9 * max(r, 1e-30)
