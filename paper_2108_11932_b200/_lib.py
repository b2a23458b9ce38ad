"""Loader for the native library ``lib/libtlrg.so`` (C ABI in ``include/tlrg.h``).

There is no fallback: if the CUDA library is missing the import of the product
path fails loudly (run ``python -c "import __graft_entry__ as g; g.build()"``).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TLRG_LIB") or os.path.join(HERE, "lib", "libtlrg.so")

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int32)
u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p


class AraConfigC(C.Structure):
    _fields_ = [("block_samples", C.c_int32), ("eps", C.c_double), ("max_rank", C.c_int32),
                ("window", C.c_int32), ("safety", C.c_double), ("recompress", C.c_int32),
                ("seed", C.c_uint64)]


class WorkspaceC(C.Structure):
    _fields_ = [("parallel_buffers", C.c_int32), ("dense_buffers", C.c_int32),
                ("subset_capacity", C.c_int32)]


class FactorOptionsC(C.Structure):
    _fields_ = [("schur_compensation", C.c_int32), ("diag_shift", C.c_double),
                ("pivot_norm", C.c_int32), ("pivot_power_iters", C.c_int32)]


class StatsC(C.Structure):
    _fields_ = [("t_sampling", C.c_double), ("t_projection", C.c_double),
                ("t_reduction", C.c_double), ("t_dense", C.c_double), ("t_orthog", C.c_double),
                ("t_misc", C.c_double), ("t_pivot_select", C.c_double), ("wall", C.c_double),
                ("compensation_frob", C.c_double), ("modified_diagonals", C.c_int32),
                ("tile_rounds_resident", C.c_uint64), ("t_recompress", C.c_double),
                ("t_compensation", C.c_double), ("flops_exec", C.c_double),
                ("flops_gemm_ref", C.c_double), ("kernel_launches", C.c_int64),
                ("t_device", C.c_double), ("kt_gemm_seconds", C.c_double),
                ("kt_gemm_flops", C.c_double), ("kt_gemm_launches", C.c_int64),
                ("t_ara_kernel", C.c_double), ("flops_ara_kernel", C.c_double),
                ("ara_kernel_launches", C.c_int64)]


class StatusC(C.Structure):
    _fields_ = [("code", C.c_int32), ("index", C.c_int32), ("msg", C.c_char * 256)]


# exported symbol -> (restype, argtypes); this table is also the export check
SIGNATURES = {
    "tlrg_version": (C.c_char_p, []),
    "tlrg_host_alloc": (C.c_void_p, [C.c_uint64]),
    "tlrg_host_free": (None, [C.c_void_p]),
    "tlrg_profiler": (None, [C.c_int]),
    "tlrg_default_ara_config": (None, [C.POINTER(AraConfigC)]),
    "tlrg_default_workspace": (None, [C.POINTER(WorkspaceC)]),
    "tlrg_default_factor_options": (None, [C.POINTER(FactorOptionsC)]),
    "tlrg_create": (C.c_int, [C.c_int, C.POINTER(vp), C.POINTER(StatusC)]),
    "tlrg_destroy": (None, [vp]),
    "tlrg_comm_nccl_id": (C.c_int, [C.POINTER(C.c_uint8), C.POINTER(StatusC)]),
    "tlrg_comm_attach_nccl": (C.c_int, [vp, C.c_int32, C.c_int32, C.POINTER(C.c_uint8),
                                        C.POINTER(StatusC)]),
    "tlrg_comm_attach_local": (C.c_int, [C.POINTER(vp), C.c_int32, C.POINTER(StatusC)]),
    "tlrg_comm_detach": (None, [vp]),
    "tlrg_matrix_upload": (C.c_int, [vp, C.c_int64, C.c_int32, C.c_double, dp, ip, dp, dp,
                                     C.POINTER(vp), C.POINTER(StatusC)]),
    "tlrg_matrix_info": (C.c_int, [vp, C.POINTER(C.c_int64), ip, ip, dp]),
    "tlrg_matrix_ranks": (C.c_int, [vp, ip]),
    "tlrg_matrix_download": (C.c_int, [vp, dp, dp, dp, C.POINTER(StatusC)]),
    "tlrg_matrix_copy": (C.c_int, [vp, C.POINTER(vp), C.POINTER(StatusC)]),
    "tlrg_matrix_free": (None, [vp]),
    "tlrg_memory_report": (C.c_int, [vp, u64p]),
    "tlrg_write_tlr": (C.c_int, [vp, C.c_char_p, C.POINTER(StatusC)]),
    "tlrg_read_tlr": (C.c_int, [vp, C.c_char_p, C.POINTER(vp), C.POINTER(StatusC)]),
    "tlrg_build": (C.c_int, [vp, C.c_int32, C.c_int64, dp, C.c_int32, C.c_double, C.c_double,
                             C.c_int32, C.c_double, C.c_int32, C.POINTER(AraConfigC),
                             C.POINTER(vp), C.POINTER(StatusC)]),
    "tlrg_factorize": (C.c_int, [vp, vp, C.c_int32, C.POINTER(AraConfigC), C.POINTER(WorkspaceC),
                                 C.POINTER(FactorOptionsC), C.POINTER(vp), C.POINTER(StatusC)]),
    "tlrg_factor_free": (None, [vp]),
    "tlrg_factor_L": (vp, [vp]),
    "tlrg_factor_mode": (C.c_int, [vp]),
    "tlrg_factor_stats": (C.c_int, [vp, C.POINTER(StatsC), ip, dp]),
    "tlrg_factor_dblock": (C.c_int, [vp, C.c_int32, dp, dp, u8p, ip]),
    "tlrg_write_factor": (C.c_int, [vp, C.c_char_p, C.POINTER(StatusC)]),
    "tlrg_read_factor": (C.c_int, [vp, C.c_char_p, C.POINTER(vp), C.POINTER(StatusC)]),
    "tlrg_factor_perm": (C.c_int, [vp, C.POINTER(C.c_int32)]),
    "tlrg_factor_solve": (C.c_int, [vp, dp, dp, C.POINTER(StatusC)]),
    "tlrg_factor_apply": (C.c_int, [vp, dp, dp, C.POINTER(StatusC)]),
    "tlrg_tlr_matvec": (C.c_int, [vp, dp, dp, C.POINTER(StatusC)]),
    "tlrg_estimate_2norm_diff": (C.c_int, [vp, vp, C.c_int32, C.c_uint64, dp, C.POINTER(StatusC)]),
    "tlrg_estimate_2norm": (C.c_int, [vp, C.c_int32, C.c_uint64, dp, C.POINTER(StatusC)]),
    "tlrg_frob_norm": (C.c_int, [vp, dp, C.POINTER(StatusC)]),
    "tlrg_estimate_frob_diff": (C.c_int, [vp, vp, C.c_int32, C.c_uint64, dp, C.POINTER(StatusC)]),
    "tlrg_sample_left": (C.c_int, [vp, dp, dp, u8p, C.c_int32, C.c_int32, ip, C.c_int32, dp,
                                   C.c_int32, C.c_int32, dp, C.POINTER(StatusC)]),
    "tlrg_chol_ara_update": (C.c_int, [vp, dp, dp, u8p, C.c_int32, C.POINTER(AraConfigC),
                                       C.POINTER(WorkspaceC), C.POINTER(vp), C.POINTER(StatusC)]),
    "tlrg_ara_count": (C.c_int, [vp]),
    "tlrg_ara_tile": (C.c_int, [vp, C.c_int32, ip, dp, dp]),
    "tlrg_ara_free": (None, [vp]),
    "tlrg_ara_stats": (None, [vp, dp]),
    "tlrg_rng_gaussians": (C.c_int, [vp, C.c_uint64, C.c_int64, dp, C.POINTER(StatusC)]),
    "tlrg_orthog": (C.c_int, [vp, dp, C.c_int32, C.c_int32, dp, C.c_int32, C.c_uint64, dp, dp, dp,
                              dp, C.POINTER(StatusC)]),
    "tlrg_potrf": (C.c_int, [vp, dp, C.c_int32, dp, ip, C.POINTER(StatusC)]),
    "tlrg_dense_ldl": (C.c_int, [vp, dp, C.c_int32, dp, dp, dp, u8p, ip, ip, C.POINTER(StatusC)]),
    "tlrg_schur_compensation": (C.c_int, [vp, dp, C.c_int32, C.c_double, dp, dp,
                                          C.POINTER(StatusC)]),
    "tlrg_jacobi_svd": (C.c_int, [vp, dp, C.c_int32, C.c_int32, C.c_double, C.c_int32, dp, dp,
                                  dp, ip, C.POINTER(StatusC)]),
    "tlrg_gemm": (C.c_int, [vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double,
                            dp, dp, C.c_double, dp, C.POINTER(StatusC)]),
}

_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"native library missing: {LIB_PATH}; build it with "
                               "`python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib
