"""CPU-only checks: host ports (seeds, tlr::Rng, geometry) against the oracle,
and the C-ABI library loads and exports every symbol include/tlrg.h declares."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2108_11932_b200 import geometry as G
from paper_2108_11932_b200 import util
from paper_2108_11932_b200.mt64 import Mt64

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_seed_derivation_matches_reference(ref):
    for root in [0, 1, 12345, 2**64 - 1]:
        assert util.mix64(root) == ref.mix64(root)
        for i, k in [(1, 0), (7, 3), (255, 254)]:
            assert util.ara_column_seed(root, i, k) == ref.ara_column_seed(root, i, k)
            assert util.tile_seed(root, 0xB11D, i, k) == ref.tile_seed(root, 0xB11D, i, k)


@pytest.mark.parametrize("seed", [0, 5, 2**63 + 11])
def test_host_rng_port_matches_reference(ref, seed):
    g = Mt64(seed).gaussians(5001)
    assert np.abs(g - ref.rng_gaussians(seed, 5001)).max() <= 4e-15 * np.abs(g).max()


@pytest.mark.parametrize("kind,n,tile", [(G.GRID2D, 16384, 256), (G.GRID3D, 4096, 512),
                                         (G.BALL3D, 1024, 128), (G.GRID2D, 500, 128),
                                         (G.GRID3D, 6000, 512)])
def test_geometry_matches_reference(ref, kind, n, tile):
    p = G.kd_order(G.generate_points(kind, n, 42), tile).matrix_order()
    assert np.array_equal(p, ref.points(kind, n, 42, tile))


def test_capi_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "tlrg.h")).read()
    names = set(re.findall(r"\b(tlrg_[A-Za-z0-9_]+)\s*\(", hdr))
    assert len(names) >= 30
    from paper_2108_11932_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_lib.SIGNATURES) <= names
    assert b"sm_100a" in _lib.load().tlrg_version()


def test_library_is_sm100a_sass():
    import subprocess
    from paper_2108_11932_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH],
                          capture_output=True, text=True).stdout
    assert "DMMA" in sass  # FP64 tensor-core MMA in the grouped GEMM


def test_no_cuda_device_means_loud_failure():
    import paper_2108_11932_b200 as tg
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(tg.Error):
        tg.Context(0)
