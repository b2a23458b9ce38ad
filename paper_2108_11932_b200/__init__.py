"""B200-native TLR Cholesky / LDL^T factorization (arXiv 2108.11932).

The compute path is ``lib/libtlrg.so`` (hand-written sm_100a CUDA behind the C
ABI in ``include/tlrg.h``); :mod:`.tlr` mirrors the reference's ``tlr::`` API.
"""
from .tlr import *  # noqa: F401,F403
from .tlr import (AraConfig, AraWorkspace, FactorOptions, TlrMatrix, TlrFactor, Context,
                  tlr_cholesky, tlr_ldlt, factor_solve, factor_apply, tlr_matvec,
                  estimate_2norm, estimate_2norm_diff, sample_left, sample_left_transpose,
                  chol_ara_update, read_tlr, write_tlr, ConfigError, DataError,
                  DimensionError, NumericError)
from . import geometry, util  # noqa: F401
