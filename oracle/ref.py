"""ORACLE / TEST INFRASTRUCTURE — NOT PRODUCT CODE.

ctypes view of ``oracle/_ref/libtlr_ref.so``: the UNMODIFIED reference library
(/root/reference/proj/src, compiled in place by ``oracle/Makefile``) behind the
thin C ABI in ``oracle/ref_capi.cpp``.  Only ``tests/``, ``__graft_entry__.smoke``
and ``bench.py`` (cpu_baseline / ``--impl reference``) may import this module,
and only as the checker or as the CPU baseline — never on the product path.

Storage conventions follow the reference: column-major FP64 tiles, lower tile
(i, j), i > j at flat index i*(i-1)/2 + j (tlr_matrix.hpp:36, tlr_matrix.cpp:31-34).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libtlr_ref.so")

_lib = None

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)
u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_ulonglong)
vp = C.c_void_p
i64 = C.c_longlong
u64 = C.c_ulonglong


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        # dense_kernels.cpp:17-24 pins OpenBLAS to one thread from a constructor
        # that runs too late for a dynamic OpenBLAS; set it before loading.
        os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
        if not available():
            raise RuntimeError(f"oracle reference library not built: {LIB_PATH} "
                               "(run `make -C oracle`)")
        L = C.CDLL(LIB_PATH)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_set_threads": (None, [C.c_int]),
            "ref_max_threads": (C.c_int, []),
            "ref_mix64": (u64, [u64]),
            "ref_tile_seed": (u64, [u64, u64, u64, u64]),
            "ref_ara_column_seed": (u64, [u64, C.c_int, C.c_int]),
            "ref_rng_gaussians": (None, [u64, i64, dp]),
            "ref_rng_uniforms": (None, [u64, i64, dp]),
            "ref_points": (C.c_int, [C.c_int, C.c_int, u64, C.c_int, dp]),
            "ref_build": (vp, [C.c_int, C.c_int, dp, C.c_int, C.c_double, C.c_double, C.c_int,
                               C.c_double, C.c_int, C.c_int, u64, ip]),
            "ref_kernel_block": (C.c_int, [C.c_int, C.c_int, dp, C.c_int, C.c_double, C.c_double,
                                           i64, C.c_int, i64, C.c_int, dp]),
            "ref_matrix_from_parts": (vp, [i64, C.c_int, C.c_double, dp, ip, dp, dp]),
            "ref_matrix_copy": (vp, [vp]),
            "ref_matrix_flat": (None, [vp, dp, dp, dp]),
            "ref_matrix_free": (None, [vp]),
            "ref_matrix_info": (None, [vp, C.POINTER(i64), ip, ip, dp]),
            "ref_matrix_ranks": (None, [vp, ip]),
            "ref_matrix_diag": (None, [vp, C.c_int, dp]),
            "ref_matrix_set_diag": (None, [vp, C.c_int, dp]),
            "ref_matrix_tile": (None, [vp, C.c_int, C.c_int, dp, dp]),
            "ref_matrix_write": (C.c_int, [vp, C.c_char_p]),
            "ref_matrix_read": (vp, [C.c_char_p, ip]),
            "ref_memory_report": (None, [vp, u64p]),
            "ref_tlr_matvec": (C.c_int, [vp, dp, dp]),
            "ref_estimate_2norm": (C.c_double, [vp, C.c_int, u64]),
            "ref_factor": (vp, [vp, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_double,
                                C.c_int, u64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, ip]),
            "ref_factor_free": (None, [vp]),
            "ref_set_pivot": (None, [C.c_int, C.c_int]),
            "ref_factor_L": (vp, [vp]),
            "ref_factor_mode": (C.c_int, [vp]),
            "ref_factor_stats": (None, [vp, dp, ip, dp, u64p]),
            "ref_factor_dblock": (None, [vp, C.c_int, dp, dp, u8p, ip]),
            "ref_factor_perm": (None, [vp, ip]),
            "ref_factor_solve": (C.c_int, [vp, dp, dp]),
            "ref_factor_apply": (C.c_int, [vp, dp, dp]),
            "ref_estimate_2norm_diff": (C.c_double, [vp, vp, C.c_int, u64]),
            "ref_frob_norm": (C.c_double, [vp]),
            "ref_estimate_frob_diff": (C.c_double, [vp, vp, C.c_int, u64]),
            "ref_factor_write": (C.c_int, [vp, C.c_char_p]),
            "ref_factor_read": (vp, [C.c_char_p, ip]),
            "ref_sample_left": (C.c_int, [vp, dp, dp, u8p, C.c_int, C.c_int, ip, C.c_int, dp,
                                          C.c_int, C.c_int, dp]),
            "ref_chol_ara_update": (vp, [vp, dp, dp, u8p, C.c_int, C.c_int, C.c_double, C.c_int,
                                         C.c_int, C.c_double, C.c_int, u64, C.c_int, C.c_int, ip]),
            "ref_ara_count": (C.c_int, [vp]),
            "ref_ara_tile": (None, [vp, C.c_int, ip, dp, dp]),
            "ref_ara_free": (None, [vp]),
            "ref_ara_single_dense": (C.c_int, [dp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                               C.c_int, C.c_double, C.c_int, u64, ip, dp, dp]),
            "ref_orthog": (C.c_int, [dp, C.c_int, C.c_int, dp, C.c_int, u64, dp, dp, dp, dp]),
            "ref_dense_ldl": (C.c_int, [dp, C.c_int, dp, dp, dp, u8p, ip]),
            "ref_modified_cholesky": (C.c_int, [dp, C.c_int, dp, ip]),
            "ref_schur_compensation": (C.c_int, [dp, C.c_int, C.c_double, dp]),
            "ref_svd_truncate": (C.c_int, [dp, C.c_int, C.c_int, C.c_double, dp, dp]),
            "ref_spectral_norm_estimate": (C.c_double, [dp, C.c_int, C.c_int, C.c_int, u64]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _d(a):
    return a.ctypes.data_as(dp) if a is not None else None


def _i(a):
    return a.ctypes.data_as(ip) if a is not None else None


def _u8(a):
    return a.ctypes.data_as(u8p) if a is not None else None


def _check(st, what):
    if st != 0:
        raise RefError(st, f"{what}: {lib().ref_last_error().decode()}")


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------------------
# util / geometry
def mix64(x):
    return int(lib().ref_mix64(x & 0xFFFFFFFFFFFFFFFF))


def tile_seed(root, phase, i, j):
    return int(lib().ref_tile_seed(root, phase, i, j))


def ara_column_seed(root, i, k):
    return int(lib().ref_ara_column_seed(root, i, k))


def rng_gaussians(seed, n):
    out = np.empty(n)
    lib().ref_rng_gaussians(seed, n, _d(out))
    return out


def points(kind: int, n: int, seed: int = 0, tile: int = 0) -> np.ndarray:
    """generate_points + kd_order; coords in matrix order, shape (n, dim).
    kind: 0 Grid2D, 1 Grid3D, 2 RandomBall3D (geometry.hpp:11)."""
    dim = 2 if kind == 0 else 3
    out = np.empty((n, dim))
    _check(lib().ref_points(kind, n, seed, tile, _d(out)), "points")
    return out


def kernel_block(coords, kernel_kind, ell, nugget, r0, nr, c0, nc):
    coords = f64(coords)
    out = np.empty(nr * nc)
    _check(lib().ref_kernel_block(coords.shape[1], coords.shape[0], _d(coords), kernel_kind, ell,
                                  nugget, r0, nr, c0, nc, _d(out)), "kernel_block")
    return out.reshape(nc, nr).T


# ---------------------------------------------------------------------------
class RefMatrix:
    """Handle on a reference ``TlrMatrix`` (owned)."""

    def __init__(self, h):
        self.h = h
        n, b, nb, eps = i64(), C.c_int(), C.c_int(), C.c_double()
        lib().ref_matrix_info(h, C.byref(n), C.byref(b), C.byref(nb), C.byref(eps))
        self.n, self.b, self.nb, self.eps = n.value, b.value, nb.value, eps.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_matrix_free(self.h)
            self.h = None

    def tile_rows(self, i):
        return min(self.b, self.n - i * self.b)

    def ranks(self):
        out = np.zeros(max(1, self.nb * (self.nb - 1) // 2), dtype=np.int32)
        lib().ref_matrix_ranks(self.h, _i(out))
        return out[: self.nb * (self.nb - 1) // 2]

    def diag(self, k):
        r = self.tile_rows(k)
        out = np.empty(r * r)
        lib().ref_matrix_diag(self.h, k, _d(out))
        return out.reshape(r, r).T.copy()

    def tile(self, i, j):
        k = int(self.ranks()[i * (i - 1) // 2 + j])
        U = np.empty(self.tile_rows(i) * k)
        V = np.empty(self.tile_rows(j) * k)
        lib().ref_matrix_tile(self.h, i, j, _d(U), _d(V))
        return (U.reshape(k, self.tile_rows(i)).T.copy(),
                V.reshape(k, self.tile_rows(j)).T.copy())

    def to_flat(self):
        """(diag, ranks, U, V) flat arrays in the reference's tile order."""
        ranks = self.ranks()
        rows = np.array([self.tile_rows(i) for i in range(self.nb)], dtype=np.int64)
        nd = int((rows * rows).sum())
        ii, jj = np.tril_indices(self.nb, -1)
        order = np.lexsort((jj, ii))  # (i, j) with i ascending, then j
        ii, jj = ii[order], jj[order]
        nu = int((rows[ii] * ranks).sum()) if ranks.size else 0
        nv = int((rows[jj] * ranks).sum()) if ranks.size else 0
        dg, U, V = np.empty(nd), np.empty(max(nu, 1)), np.empty(max(nv, 1))
        lib().ref_matrix_flat(self.h, _d(dg), _d(U), _d(V))
        return dg, ranks, U[:nu], V[:nv]

    def to_parts(self):
        """(diag list, ranks, U list, V list) with U/V as (rows, k) arrays."""
        dg, ranks, Uf, Vf = self.to_flat()
        diag, off = [], 0
        for k in range(self.nb):
            r = self.tile_rows(k)
            diag.append(dg[off:off + r * r].reshape(r, r).T.copy())
            off += r * r
        U, V, ou, ov, t = [], [], 0, 0, 0
        for i in range(1, self.nb):
            for j in range(i):
                k = int(ranks[t])
                ri, rj = self.tile_rows(i), self.tile_rows(j)
                U.append(Uf[ou:ou + ri * k].reshape(k, ri).T.copy())
                V.append(Vf[ov:ov + rj * k].reshape(k, rj).T.copy())
                ou += ri * k
                ov += rj * k
                t += 1
        return diag, ranks, U, V

    def copy(self):
        return RefMatrix(lib().ref_matrix_copy(self.h))

    def write(self, path):
        _check(lib().ref_matrix_write(self.h, path.encode()), "write_tlr")

    def matvec(self, x):
        x = f64(x)
        y = np.empty(self.n)
        _check(lib().ref_tlr_matvec(self.h, _d(x), _d(y)), "tlr_matvec")
        return y

    def estimate_2norm(self, iters=50, seed=1):
        return lib().ref_estimate_2norm(self.h, iters, seed)

    def memory_report(self):
        out = (C.c_ulonglong * 3)()
        lib().ref_memory_report(self.h, out)
        return {"total_bytes": out[0], "dense_bytes": out[1], "low_rank_bytes": out[2]}

    def dense(self):
        """Full dense expansion (small sizes only)."""
        n, b = self.n, self.b
        A = np.zeros((n, n))
        diag, ranks, U, V = self.to_parts()
        t = 0
        for i in range(self.nb):
            A[i * b:i * b + self.tile_rows(i), i * b:i * b + self.tile_rows(i)] = diag[i]
        for i in range(1, self.nb):
            for j in range(i):
                blk = U[t] @ V[t].T
                A[i * b:i * b + blk.shape[0], j * b:j * b + blk.shape[1]] = blk
                A[j * b:j * b + blk.shape[1], i * b:i * b + blk.shape[0]] = blk.T
                t += 1
        return A


def matrix_from_parts(n, b, eps, diag, ranks, U, V) -> RefMatrix:
    dg = f64(np.concatenate([np.asarray(d).T.ravel() for d in diag]))
    rk = np.ascontiguousarray(ranks, dtype=np.int32)
    uu = [np.asarray(u).T.ravel() for u in U]
    vv = [np.asarray(v).T.ravel() for v in V]
    Uf = f64(np.concatenate(uu)) if uu else np.zeros(1)
    Vf = f64(np.concatenate(vv)) if vv else np.zeros(1)
    if Uf.size == 0:
        Uf = np.zeros(1)
    if Vf.size == 0:
        Vf = np.zeros(1)
    return RefMatrix(lib().ref_matrix_from_parts(n, b, eps, _d(dg), _i(rk), _d(Uf), _d(Vf)))


def matrix_from_flat(n, b, eps, diag, ranks, U, V) -> RefMatrix:
    """TlrMatrix from the flat layout (diag None: zero diagonal tiles)."""
    rk = np.ascontiguousarray(ranks, dtype=np.int32)
    Uf, Vf = f64(U), f64(V)
    dg = None if diag is None else f64(diag)
    return RefMatrix(lib().ref_matrix_from_parts(n, b, eps, _d(dg), _i(rk), _d(Uf), _d(Vf)))


def build(coords, kernel_kind, ell, nugget, b, eps, compressor=0, bs=16, seed=0) -> RefMatrix:
    """build_tlr (tlr_matrix.cpp:98-152) on points given in matrix order.
    kernel_kind: 0 exponential, 1 squared exponential; compressor 0 ARA, 1 SVD."""
    coords = f64(coords)
    st = C.c_int()
    h = lib().ref_build(coords.shape[1], coords.shape[0], _d(coords), kernel_kind, ell, nugget, b,
                        eps, compressor, bs, seed, C.byref(st))
    _check(st.value, "build_tlr")
    return RefMatrix(h)


def read_tlr(path) -> RefMatrix:
    st = C.c_int()
    h = lib().ref_matrix_read(path.encode(), C.byref(st))
    _check(st.value, "read_tlr")
    return RefMatrix(h)


@dataclass
class RefStats:
    t_sampling: float = 0
    t_projection: float = 0
    t_reduction: float = 0
    t_dense: float = 0
    t_orthog: float = 0
    t_misc: float = 0
    t_pivot_select: float = 0
    wall: float = 0
    compensation_frob: float = 0
    modified_diagonals: int = 0
    ara_rounds: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    pivot_trace: np.ndarray = field(default_factory=lambda: np.zeros(0))
    tile_rounds_resident: int = 0


class RefFactor:
    def __init__(self, h):
        self.h = h
        self.L = RefMatrix.__new__(RefMatrix)
        Lh = lib().ref_factor_L(h)
        n, b, nb, eps = i64(), C.c_int(), C.c_int(), C.c_double()
        lib().ref_matrix_info(Lh, C.byref(n), C.byref(b), C.byref(nb), C.byref(eps))
        self.L.h = None  # borrowed: never freed through RefMatrix
        self.L.n, self.L.b, self.L.nb, self.L.eps = n.value, b.value, nb.value, eps.value
        self._Lh = Lh
        self.mode = lib().ref_factor_mode(h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_factor_free(self.h)
            self.h = None

    # borrowed-L accessors
    def _L(self):
        m = RefMatrix.__new__(RefMatrix)
        m.h, m.n, m.b, m.nb, m.eps = self._Lh, self.L.n, self.L.b, self.L.nb, self.L.eps
        return m

    def L_parts(self):
        m = self._L()
        try:
            return m.to_parts()
        finally:
            m.h = None

    def L_ranks(self):
        m = self._L()
        try:
            return m.ranks()
        finally:
            m.h = None

    def stats(self) -> RefStats:
        nb = self.L.nb
        v = np.zeros(10)
        ar = np.zeros(nb, dtype=np.int32)
        pt = np.zeros(nb)
        tr = C.c_ulonglong()
        lib().ref_factor_stats(self.h, _d(v), _i(ar), _d(pt), C.byref(tr))
        return RefStats(*v[:9].tolist(), int(v[9]), ar, pt, tr.value)

    def perm(self):
        """pivoted mode: factor position -> tile (factor.hpp:29); [] otherwise"""
        if self.mode != 2:
            return []
        p = np.zeros(self.L.nb, np.int32)
        lib().ref_factor_perm(self.h, _i(p))
        return [int(x) for x in p]

    def dblock(self, k):
        n = self.L.tile_rows(k)
        d, e = np.zeros(n), np.zeros(max(n - 1, 1))
        s2, p = np.zeros(n, np.uint8), np.zeros(n, np.int32)
        lib().ref_factor_dblock(self.h, k, _d(d), _d(e), _u8(s2), _i(p))
        return d, e[: n - 1], s2, p

    def solve(self, b):
        b = f64(b)
        x = np.empty(self.L.n)
        _check(lib().ref_factor_solve(self.h, _d(b), _d(x)), "factor_solve")
        return x

    def apply(self, x):
        x = f64(x)
        y = np.empty(self.L.n)
        _check(lib().ref_factor_apply(self.h, _d(x), _d(y)), "factor_apply")
        return y

    def write(self, path):
        _check(lib().ref_factor_write(self.h, path.encode()), "write_factor")


def factor(A: RefMatrix, mode=0, bs=16, eps=1e-6, max_rank=0, window=0, safety=10.0,
           recompress=True, seed=0, parallel_buffers=64, dense_buffers=20, subset_capacity=0,
           schur_compensation=True, diag_shift=0.0, pivot_norm=0,
           pivot_power_iters=50) -> RefFactor:
    """tlr_cholesky (mode 0) / tlr_ldlt (1) / tlr_cholesky_pivoted (2), factor.cpp:290-306.
    A is copied; the caller's handle stays valid."""
    st = C.c_int()
    lib().ref_set_pivot(pivot_norm, pivot_power_iters)
    h = lib().ref_factor(A.h, mode, bs, eps, max_rank, window, safety, int(recompress), seed,
                         parallel_buffers, dense_buffers, subset_capacity, int(schur_compensation),
                         diag_shift, C.byref(st))
    _check(st.value, "factor")
    return RefFactor(h)


def read_factor(path) -> RefFactor:
    """read_factor (factor.cpp:340-395)"""
    st = C.c_int()
    h = lib().ref_factor_read(str(path).encode(), C.byref(st))
    _check(st.value, "read_factor")
    return RefFactor(h)


def estimate_2norm_diff(A: RefMatrix, F: RefFactor, iters=50, seed=17):
    return lib().ref_estimate_2norm_diff(A.h, F.h, iters, seed)


def frob_norm(A: RefMatrix) -> float:
    """||A||_F, exact tile-wise (same formula as tlrg_frob_norm)."""
    return lib().ref_frob_norm(A.h)


def estimate_frob_diff(A: RefMatrix, F: RefFactor, probes=64, seed=23) -> float:
    """Hutchinson estimate of ||P A P^T - L L^T||_F (same probes as the device)."""
    return lib().ref_estimate_frob_diff(A.h, F.h, probes, seed)


def accuracy(A: RefMatrix, F: RefFactor, probes=64, seed=23, solve_seed=7):
    """The accuracy block of bench.py / the parity tests, computed exactly as
    paper_2108_11932_b200.tlr.accuracy computes it on the device (same probes,
    same solve vector x = Rng(solve_seed) draws, same rank summary)."""
    from paper_2108_11932_b200.util import rank_summary
    fa = frob_norm(A)
    fd = estimate_frob_diff(A, F, probes, seed)
    r2 = estimate_2norm_diff(A, F, 50, 17)
    a2 = A.estimate_2norm(50, 1)
    x = rng_gaussians(solve_seed, A.n)
    b = A.matvec(x)
    xs = F.solve(b)
    bwd = float(np.linalg.norm(A.matvec(xs) - b) / np.linalg.norm(b))
    fwd = float(np.linalg.norm(xs - x) / np.linalg.norm(x))
    m = F._L()
    try:
        lr = int(m.memory_report()["low_rank_bytes"])
        ranks = m.ranks()
    finally:
        m.h = None
    out = {"resid_frob_rel": fd / fa, "resid_frob": fd, "A_frob": fa, "resid_2norm": r2,
           "resid_2norm_rel": r2 / a2, "backward_err": bwd, "forward_err": fwd,
           "L_lowrank_bytes": lr}
    out.update(rank_summary(ranks))
    return out


def _dblocks_flat(A, D):
    if D is None:
        return None, None, None
    nb, b = A.nb, A.b
    dd, de, ds = np.zeros(nb * b), np.zeros(nb * b), np.zeros(nb * b, np.uint8)
    for j, (d, e, s2) in enumerate(D):
        r = len(d)
        dd[j * b:j * b + r] = d
        de[j * b:j * b + r - 1] = e
        ds[j * b:j * b + r] = s2
    return dd, de, ds


def sample_left(A: RefMatrix, k, rows, omegas, parallel_buffers=64, D=None, transpose=False):
    """sample_left / sample_left_transpose (ara.cpp:275-300).  D: list of
    (d, e, start2x2) per column for LDL mode."""
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    width = omegas[0].shape[1]
    om = f64(np.concatenate([np.asarray(o).T.ravel() for o in omegas]))
    outrows = [A.tile_rows(int(i)) if not transpose else A.tile_rows(k) for i in rows]
    out = np.empty(sum(outrows) * width)
    dd, de, ds = _dblocks_flat(A, D)
    _check(lib().ref_sample_left(A.h, _d(dd), _d(de), _u8(ds), k, len(rows), _i(rows),
                                 parallel_buffers, _d(om), width, int(transpose), _d(out)),
           "sample_left")
    res, off = [], 0
    for r in outrows:
        res.append(out[off:off + r * width].reshape(width, r).T.copy())
        off += r * width
    return res


def chol_ara_update(A: RefMatrix, k, bs=16, eps=1e-6, max_rank=0, window=0, safety=10.0,
                    recompress=True, seed=0, parallel_buffers=64, subset_capacity=0, D=None):
    """chol_ara_update (ara.cpp:302-419).  Returns list of dicts i, Q, B, converged, rounds."""
    dd, de, ds = _dblocks_flat(A, D)
    st = C.c_int()
    h = lib().ref_chol_ara_update(A.h, _d(dd), _d(de), _u8(ds), k, bs, eps, max_rank, window,
                                  safety, int(recompress), seed, parallel_buffers,
                                  subset_capacity, C.byref(st))
    _check(st.value, "chol_ara_update")
    out = []
    try:
        rk = A.tile_rows(k)
        for t in range(lib().ref_ara_count(h)):
            info = np.zeros(4, np.int32)
            lib().ref_ara_tile(h, t, _i(info), None, None)
            i, q = int(info[0]), int(info[1])
            Q = np.empty(A.tile_rows(i) * q)
            B = np.empty(rk * q)
            lib().ref_ara_tile(h, t, _i(info), _d(Q), _d(B))
            out.append(dict(i=i, Q=Q.reshape(q, -1).T.copy(), B=B.reshape(q, -1).T.copy(),
                            converged=bool(info[2]), rounds=int(info[3])))
    finally:
        lib().ref_ara_free(h)
    return out


def orthog(Q, Y, seed):
    """orthog (dense_kernels.cpp:379-420). Returns (Yout, R, col_norms, new_mass, next_draw)."""
    Y = np.asfortranarray(Y, dtype=np.float64).copy(order="F")
    rows, k = Y.shape
    q = 0 if Q is None else Q.shape[1]
    Qf = np.asfortranarray(Q, dtype=np.float64) if q else None
    R = np.zeros((k, k), order="F")
    cn, nm, nd = np.zeros(k), np.zeros(k), np.zeros(1)
    _check(lib().ref_orthog(Qf.ctypes.data_as(dp) if q else None, rows, q,
                            Y.ctypes.data_as(dp), k, seed, R.ctypes.data_as(dp), _d(cn), _d(nm),
                            _d(nd)), "orthog")
    return np.array(Y), np.array(R), cn, nm, float(nd[0])


def dense_ldl(A):
    n = A.shape[0]
    Af = np.asfortranarray(A, dtype=np.float64)
    L = np.zeros((n, n), order="F")
    d, e = np.zeros(n), np.zeros(max(n - 1, 1))
    s2, p = np.zeros(n, np.uint8), np.zeros(n, np.int32)
    _check(lib().ref_dense_ldl(Af.ctypes.data_as(dp), n, L.ctypes.data_as(dp), _d(d), _d(e),
                               _u8(s2), _i(p)), "dense_ldl")
    return np.array(L), d, e[: n - 1], s2, p


def modified_cholesky(A):
    n = A.shape[0]
    Af = np.asfortranarray(A, dtype=np.float64)
    L = np.zeros((n, n), order="F")
    mod = C.c_int()
    _check(lib().ref_modified_cholesky(Af.ctypes.data_as(dp), n, L.ctypes.data_as(dp),
                                       C.byref(mod)), "modified_cholesky")
    return np.array(L), bool(mod.value)


def schur_compensation(Dk, eps):
    n = Dk.shape[0]
    Df = np.asfortranarray(Dk, dtype=np.float64)
    out = np.zeros(n)
    _check(lib().ref_schur_compensation(Df.ctypes.data_as(dp), n, eps, _d(out)), "schur")
    return out


def ara_single_dense(A, bs=16, eps=1e-6, max_rank=0, window=0, safety=10.0, recompress=True,
                     seed=0):
    A = np.asfortranarray(A, dtype=np.float64)
    m, n = A.shape
    cap = max_rank if max_rank > 0 else min(m, n)
    Q = np.zeros(m * cap)
    B = np.zeros(n * cap)
    info = np.zeros(3, np.int32)
    _check(lib().ref_ara_single_dense(A.ctypes.data_as(dp), m, n, bs, eps, max_rank, window,
                                      safety, int(recompress), seed, _i(info), _d(Q), _d(B)),
           "ara_single")
    r = int(info[0])
    return dict(rank=r, converged=bool(info[1]), rounds=int(info[2]),
                Q=Q[: m * r].reshape(r, m).T.copy(), B=B[: n * r].reshape(r, n).T.copy())
