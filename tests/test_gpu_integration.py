"""Drop-in conformance: the reference library calls the B200 factorization
through its own types (integration/tlr_b200.cpp: tlr::tlr_cholesky_b200 /
tlr::tlr_ldlt_b200 over include/tlrg.h), and the reference's own
estimate_2norm_diff / factor_solve evaluate the returned tlr::TlrFactor next to
the reference factor of the same matrix (oracle/conformance.cpp)."""
import ctypes
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "libtlr_conformance.so")


def _run(mode, n, b, eps, bs, nugget):
    if not os.path.exists(LIB):
        pytest.skip("conformance driver not built (make -C oracle)")
    import paper_2108_11932_b200  # noqa: F401  (libtlrg.so must load first: loud failure if absent)
    lib = ctypes.CDLL(LIB)
    out = np.zeros(8)
    err = ctypes.create_string_buffer(512)
    rc = lib.conf_run(ctypes.c_int(mode), ctypes.c_int(n), ctypes.c_int(b), ctypes.c_double(eps),
                      ctypes.c_int(bs), ctypes.c_double(nugget),
                      out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), err, 512)
    assert rc == 0, err.value.decode()
    return out


@pytest.mark.parametrize("n,b,eps", [(2048, 128, 1e-6), (4096, 256, 1e-2)])
def test_cholesky_dropin_through_reference_types(n, b, eps):
    r_ref, r_gpu, bw_ref, bw_gpu, rk_ref, rk_gpu, eq, _ = _run(0, n, b, eps, 16, 0.0)
    assert r_gpu <= 2.0 * r_ref + 1e-14          # north-star residual gate
    assert bw_gpu <= 2.0 * bw_ref + 1e-14        # solve error gate
    assert abs(rk_gpu - rk_ref) <= 0.1 * rk_ref  # rank distribution gate
    assert eq >= 0.95


def test_ldlt_dropin_through_reference_types():
    r_ref, r_gpu, bw_ref, bw_gpu, rk_ref, rk_gpu, eq, _ = _run(1, 1024, 128, 1e-4, 32, 1e-4)
    assert r_gpu <= 2.0 * r_ref + 1e-14
    assert bw_gpu <= 2.0 * bw_ref + 1e-14
    assert abs(rk_gpu - rk_ref) <= 0.1 * rk_ref
