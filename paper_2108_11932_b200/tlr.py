"""Host-side mirror of the reference's ``tlr::`` C++ API over the C ABI.

Names, argument meaning and error behaviour follow /root/reference/proj/include/tlr:
``AraConfig`` / ``AraWorkspace`` (ara.hpp:15-30), ``FactorOptions`` (factor.hpp:15-20),
``TlrMatrix`` (tlr_matrix.hpp:26-59), ``tlr_cholesky`` / ``tlr_ldlt``
(factor.hpp:35-41; the matrix argument is consumed like the by-value
``TlrMatrix A``), ``factor_solve`` / ``factor_apply`` (solve.hpp:16-19),
``tlr_matvec`` (tlr_matrix.hpp:64), ``estimate_2norm_diff`` / ``estimate_2norm``
(solve.hpp:37-41), ``sample_left`` / ``sample_left_transpose`` /
``chol_ara_update`` (ara.hpp:102-130) and the error taxonomy (errors.hpp:10-30).

All computation runs in ``lib/libtlrg.so`` on the GPU; this module only moves
host arrays across the boundary.  Tiles are numpy arrays (rows, cols) in the
reference's column-major payload order.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as L


# ----------------------------------------------------------------- errors ---
class Error(RuntimeError):
    pass


class ConfigError(Error):
    pass


class DataError(Error):
    pass


class DimensionError(Error):
    pass


class NumericError(Error):
    def __init__(self, msg, index=-1):
        super().__init__(msg)
        self.index = index


def _raise(st: L.StatusC, rc: int):
    if rc == 0:
        return
    msg = st.msg.decode(errors="replace")
    if rc == 2:
        raise ConfigError(msg)
    if rc == 3:
        raise DataError(msg)
    if rc == 4:
        raise NumericError(msg, st.index)
    raise Error(msg)


def _call(fn, *args):
    st = L.StatusC()
    rc = fn(*args, C.byref(st))
    _raise(st, rc)


def _d(a):
    return None if a is None else a.ctypes.data_as(L.dp)


def _i(a):
    return None if a is None else a.ctypes.data_as(L.ip)


def _u8(a):
    return None if a is None else a.ctypes.data_as(L.u8p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ------------------------------------------------------------------ config --
@dataclass
class AraConfig:
    block_samples: int = 32
    eps: float = 1e-6
    max_rank: int = 0
    window: int = 0
    safety: float = 10.0
    recompress: bool = True
    seed: int = 0

    def c(self):
        return L.AraConfigC(self.block_samples, self.eps, self.max_rank, self.window, self.safety,
                            int(self.recompress), self.seed & 0xFFFFFFFFFFFFFFFF)


@dataclass
class AraWorkspace:
    parallel_buffers: int = 64
    dense_buffers: int = 20
    subset_capacity: int = 0

    def c(self):
        return L.WorkspaceC(self.parallel_buffers, self.dense_buffers, self.subset_capacity)


class PivotNorm:
    """factor.hpp:13 (enum class PivotNorm)."""
    Frobenius = 0
    TwoNormPower = 1


@dataclass
class FactorOptions:
    """factor.hpp:15-20."""
    schur_compensation: bool = True
    diag_shift: float = 0.0
    pivot_norm: int = PivotNorm.Frobenius
    pivot_power_iters: int = 50

    def c(self):
        return L.FactorOptionsC(int(self.schur_compensation), self.diag_shift,
                                int(self.pivot_norm), int(self.pivot_power_iters))


# ----------------------------------------------------------------- context --
class Context:
    """Owns one CUDA device and its stream (tlrg_create)."""

    _default = None

    def __init__(self, device: int = 0):
        self.lib = L.load()
        self.h = C.c_void_p()
        _call(self.lib.tlrg_create, device, C.byref(self.h))

    @classmethod
    def default(cls):
        if cls._default is None:
            cls._default = Context(0)
        return cls._default

    # ---- multi-GPU (intra-column tile split) -------------------
    def attach_nccl(self, rank: int, world: int, uid: bytes):
        """Join an NCCL communicator (one process per GPU); `uid` comes from
        nccl_unique_id() on rank 0, shared out of band."""
        buf = (C.c_uint8 * 128).from_buffer_copy(bytes(uid))
        _call(self.lib.tlrg_comm_attach_nccl, self.h, rank, world, buf)

    def detach(self):
        self.lib.tlrg_comm_detach(self.h)


def nccl_unique_id(ctx=None) -> bytes:
    lib = ctx.lib if ctx is not None else L.load()
    buf = (C.c_uint8 * 128)()
    _call(lib.tlrg_comm_nccl_id, buf)
    return bytes(buf)


def attach_local(ctxs):
    """In-process ranks: factorizations on these contexts, each driven by its
    own host thread, split every column between them."""
    arr = (C.c_void_p * len(ctxs))(*[c.h.value for c in ctxs])
    _call(ctxs[0].lib.tlrg_comm_attach_local, arr, len(ctxs))


def _ctx(ctx):
    return ctx if ctx is not None else Context.default()


# ------------------------------------------------------------------ matrix --
class TlrMatrix:
    """Device-resident TLR matrix (flat HBM store).  Construct with
    :meth:`from_parts`, :func:`read_tlr` or :func:`build_tlr`."""

    def __init__(self, handle, ctx, owner=None):
        self.h = handle
        self.ctx = ctx
        self._owner = owner  # keeps a factor alive for borrowed L views
        n, b, nb, eps = C.c_int64(), C.c_int32(), C.c_int32(), C.c_double()
        ctx.lib.tlrg_matrix_info(handle, C.byref(n), C.byref(b), C.byref(nb), C.byref(eps))
        self.n, self.b, self.nb, self.eps = n.value, b.value, nb.value, eps.value

    def __del__(self):
        if getattr(self, "h", None) is not None and self._owner is None:
            try:
                self.ctx.lib.tlrg_matrix_free(self.h)
            except Exception:
                pass
            self.h = None

    def _consume(self):
        if self.h is None:
            raise ConfigError("TlrMatrix was consumed by a factorization")
        if self._owner is not None:
            # borrowed view of a factor's L: the library deep-copies it (the
            # reference copies F.L into its by-value argument); the view stays valid
            return self.h
        h, self.h = self.h, None
        return h

    @staticmethod
    def from_parts(n, b, eps, diag: Sequence[np.ndarray], ranks, U: Sequence[np.ndarray],
                   V: Sequence[np.ndarray], ctx=None) -> "TlrMatrix":
        ctx = _ctx(ctx)
        dg = _f64(np.concatenate([np.asarray(d, np.float64).T.ravel() for d in diag]))
        rk = np.ascontiguousarray(ranks, dtype=np.int32)
        uu = [np.asarray(u, np.float64).T.ravel() for u in U]
        vv = [np.asarray(v, np.float64).T.ravel() for v in V]
        Uf = _f64(np.concatenate(uu)) if uu else np.zeros(1)
        Vf = _f64(np.concatenate(vv)) if vv else np.zeros(1)
        if Uf.size == 0:
            Uf = np.zeros(1)
        if Vf.size == 0:
            Vf = np.zeros(1)
        h = C.c_void_p()
        _call(ctx.lib.tlrg_matrix_upload, ctx.h, n, b, eps, _d(dg), _i(rk) if rk.size else None,
              _d(Uf), _d(Vf), C.byref(h))
        return TlrMatrix(h, ctx)

    @staticmethod
    def from_flat(n, b, eps, diag, ranks, U, V, ctx=None) -> "TlrMatrix":
        """Upload from the reference's flat layout: diag (sum rows(k)^2 or None
        for zero tiles), ranks[i(i-1)/2+j], U / V payloads concatenated in tile
        order, column-major (tlrg_matrix_upload)."""
        ctx = _ctx(ctx)
        rk = np.ascontiguousarray(ranks, dtype=np.int32)
        Uf, Vf = _f64(U), _f64(V)
        h = C.c_void_p()
        _call(ctx.lib.tlrg_matrix_upload, ctx.h, n, b, eps,
              None if diag is None else _d(_f64(diag)), _i(rk) if rk.size else None,
              _d(Uf if Uf.size else np.zeros(1)), _d(Vf if Vf.size else np.zeros(1)), C.byref(h))
        return TlrMatrix(h, ctx)

    def tile_rows(self, i):
        return min(self.b, self.n - i * self.b)

    def ranks(self):
        m = self.nb * (self.nb - 1) // 2
        out = np.zeros(max(m, 1), np.int32)
        self.ctx.lib.tlrg_matrix_ranks(self.h, _i(out))
        return out[:m]

    def rank(self, i, j):
        return int(self.ranks()[i * (i - 1) // 2 + j])

    def to_parts(self):
        ranks = self.ranks()
        nb = self.nb
        rows = [self.tile_rows(i) for i in range(nb)]
        ndiag = sum(r * r for r in rows)
        nu = nv = 0
        for i in range(1, nb):
            for j in range(i):
                k = int(ranks[i * (i - 1) // 2 + j])
                nu += rows[i] * k
                nv += rows[j] * k
        dg, Uf, Vf = np.zeros(ndiag), np.zeros(max(nu, 1)), np.zeros(max(nv, 1))
        _call(self.ctx.lib.tlrg_matrix_download, self.h, _d(dg), _d(Uf), _d(Vf))
        diag, off = [], 0
        for r in rows:
            diag.append(dg[off:off + r * r].reshape(r, r).T.copy())
            off += r * r
        U, V, ou, ov = [], [], 0, 0
        for i in range(1, nb):
            for j in range(i):
                k = int(ranks[i * (i - 1) // 2 + j])
                U.append(Uf[ou:ou + rows[i] * k].reshape(k, rows[i]).T.copy())
                V.append(Vf[ov:ov + rows[j] * k].reshape(k, rows[j]).T.copy())
                ou += rows[i] * k
                ov += rows[j] * k
        return diag, ranks, U, V

    def copy(self) -> "TlrMatrix":
        h = C.c_void_p()
        _call(self.ctx.lib.tlrg_matrix_copy, self.h, C.byref(h))
        return TlrMatrix(h, self.ctx)

    def memory_report(self):
        out = (C.c_uint64 * 3)()
        self.ctx.lib.tlrg_memory_report(self.h, out)
        r = self.ranks()
        return {"total_bytes": out[0], "dense_bytes": out[1], "low_rank_bytes": out[2],
                "rank_histogram": np.bincount(r) if r.size else np.zeros(1, np.int64)}

    def dense(self):
        diag, ranks, U, V = self.to_parts()
        n, b = self.n, self.b
        A = np.zeros((n, n))
        for i, d in enumerate(diag):
            A[i * b:i * b + d.shape[0], i * b:i * b + d.shape[0]] = d
        t = 0
        for i in range(1, self.nb):
            for j in range(i):
                blk = U[t] @ V[t].T
                A[i * b:i * b + blk.shape[0], j * b:j * b + blk.shape[1]] = blk
                A[j * b:j * b + blk.shape[1], i * b:i * b + blk.shape[0]] = blk.T
                t += 1
        return A


def write_tlr(A: TlrMatrix, path: str):
    _call(A.ctx.lib.tlrg_write_tlr, A.h, path.encode())


def read_tlr(path: str, ctx=None) -> TlrMatrix:
    ctx = _ctx(ctx)
    h = C.c_void_p()
    _call(ctx.lib.tlrg_read_tlr, ctx.h, path.encode(), C.byref(h))
    return TlrMatrix(h, ctx)


def tlr_matvec(A: TlrMatrix, x) -> np.ndarray:
    x = _f64(x)
    if x.size != A.n:
        raise DimensionError("tlr_matvec: length")
    y = np.empty(A.n)
    _call(A.ctx.lib.tlrg_tlr_matvec, A.h, _d(x), _d(y))
    return y


def estimate_2norm(A: TlrMatrix, iters=50, seed=1) -> float:
    out = C.c_double()
    _call(A.ctx.lib.tlrg_estimate_2norm, A.h, iters, seed, C.byref(out))
    return out.value


def frob_norm(A: TlrMatrix) -> float:
    """||A||_F, exact tile-wise."""
    out = C.c_double()
    _call(A.ctx.lib.tlrg_frob_norm, A.h, C.byref(out))
    return out.value


# ------------------------------------------------------------------ factor --
@dataclass
class FactorStats:
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
    tile_rounds_resident: int = 0
    t_recompress: float = 0
    t_compensation: float = 0
    flops_exec: float = 0
    flops_gemm_ref: float = 0
    kernel_launches: int = 0
    t_device: float = 0
    kt_gemm_seconds: float = 0
    kt_gemm_flops: float = 0
    kt_gemm_launches: int = 0
    t_ara_kernel: float = 0
    flops_ara_kernel: float = 0
    ara_kernel_launches: int = 0
    ara_rounds: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    pivot_trace: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def gemm_time(self):
        return self.t_sampling + self.t_projection + self.t_dense

    def gemm_share(self):
        return self.gemm_time() / self.wall if self.wall > 0 else 0.0


class BlockDiagonal:
    """D of LDL^T (dense_kernels.hpp:28-60) for one tile column."""

    def __init__(self, d, e, start2x2):
        self.d, self.e, self.start2x2 = np.asarray(d), np.asarray(e), np.asarray(start2x2)

    def materialize(self):
        n = len(self.d)
        D = np.diag(self.d.astype(float))
        for k in range(n - 1):
            if self.start2x2[k]:
                D[k + 1, k] = D[k, k + 1] = self.e[k]
        return D

    def all_positive(self):
        return bool(np.all(np.linalg.eigvalsh(self.materialize()) > 0))

    def all_negative(self):
        return bool(np.all(np.linalg.eigvalsh(self.materialize()) < 0))


class TlrFactor:
    MODES = {0: "Cholesky", 1: "LDLT", 2: "PivotedCholesky"}

    def __init__(self, handle, ctx):
        self.h = handle
        self.ctx = ctx
        self.mode = ctx.lib.tlrg_factor_mode(handle)

    @property
    def L(self) -> TlrMatrix:
        # a fresh view each time: the view keeps the factor alive, the factor
        # holds no reference back (no cycle, so `del F` frees the device memory
        # at once instead of at the next cyclic GC pass)
        return TlrMatrix(self.ctx.lib.tlrg_factor_L(self.h), self.ctx, owner=self)

    def __del__(self):
        if getattr(self, "h", None) is not None:
            try:
                self.ctx.lib.tlrg_factor_free(self.h)
            except Exception:
                pass
            self.h = None

    @property
    def stats(self) -> FactorStats:
        s = L.StatsC()
        nb = self.L.nb
        ar = np.zeros(nb, np.int32)
        pt = np.zeros(nb)
        self.ctx.lib.tlrg_factor_stats(self.h, C.byref(s), _i(ar), _d(pt))
        fs = FactorStats(**{f: getattr(s, f) for f, _ in L.StatsC._fields_})
        fs.ara_rounds, fs.pivot_trace = ar, pt
        return fs

    @property
    def D(self) -> List[BlockDiagonal]:
        if self.mode != 1:
            return []
        return [self.dblock(k)[0] for k in range(self.L.nb)]

    @property
    def intra_perm(self):
        if self.mode != 1:
            return []
        return [self.dblock(k)[1] for k in range(self.L.nb)]

    def dblock(self, k):
        n = self.L.tile_rows(k)
        d, e = np.zeros(n), np.zeros(max(n - 1, 1))
        s2, p = np.zeros(n, np.uint8), np.zeros(n, np.int32)
        self.ctx.lib.tlrg_factor_dblock(self.h, k, _d(d), _d(e), _u8(s2), _i(p))
        return BlockDiagonal(d, e[:n - 1], s2), p

    @property
    def perm(self) -> List[int]:
        """Pivoted mode: factor position -> original tile (factor.hpp:29); [] otherwise."""
        if self.mode != 2:
            return []
        p = np.zeros(self.L.nb, np.int32)
        self.ctx.lib.tlrg_factor_perm(self.h, _i(p))
        return [int(x) for x in p]

    def write(self, path):
        _call(self.ctx.lib.tlrg_write_factor, self.h, path.encode())


def read_factor(path: str, ctx=None) -> TlrFactor:
    """read_factor (factor.cpp:340-395): a TLRF file written by write_factor of
    either implementation."""
    ctx = _ctx(ctx)
    out = C.c_void_p()
    _call(ctx.lib.tlrg_read_factor, ctx.h, path.encode(), C.byref(out))
    return TlrFactor(out, ctx)


def _factor(A: TlrMatrix, mode: int, cfg: AraConfig, ws: AraWorkspace,
            opts: Optional[FactorOptions]) -> TlrFactor:
    ctx = A.ctx
    h = A._consume()
    out = C.c_void_p()
    c, w, o = cfg.c(), ws.c(), (opts or FactorOptions()).c()
    _call(ctx.lib.tlrg_factorize, ctx.h, h, mode, C.byref(c), C.byref(w), C.byref(o),
          C.byref(out))
    return TlrFactor(out, ctx)


def tlr_cholesky(A: TlrMatrix, cfg: AraConfig, ws: AraWorkspace = None,
                 opts: FactorOptions = None) -> TlrFactor:
    """factor.cpp:290-293.  ``A`` is consumed (moved into the factor)."""
    return _factor(A, 0, cfg, ws or AraWorkspace(), opts)


def tlr_cholesky_pivoted(A: TlrMatrix, cfg: AraConfig, ws: AraWorkspace = None,
                         opts: FactorOptions = None) -> TlrFactor:
    """factor.cpp:295-299 (Alg. 8 tile pivoting; uniform tiles only)."""
    return _factor(A, 2, cfg, ws or AraWorkspace(), opts)


def tlr_ldlt(A: TlrMatrix, cfg: AraConfig, ws: AraWorkspace = None,
             opts: FactorOptions = None) -> TlrFactor:
    """factor.cpp:301-306 (Schur compensation forced off)."""
    return _factor(A, 1, cfg, ws or AraWorkspace(), opts)


def factor_solve(F: TlrFactor, b) -> np.ndarray:
    b = _f64(b)
    if b.size != F.L.n:
        raise DimensionError("factor_solve: length")
    x = np.empty(F.L.n)
    _call(F.ctx.lib.tlrg_factor_solve, F.h, _d(b), _d(x))
    return x


def factor_apply(F: TlrFactor, x) -> np.ndarray:
    x = _f64(x)
    if x.size != F.L.n:
        raise DimensionError("factor_apply: length")
    y = np.empty(F.L.n)
    _call(F.ctx.lib.tlrg_factor_apply, F.h, _d(x), _d(y))
    return y


def estimate_2norm_diff(A: TlrMatrix, F: TlrFactor, iters=50, seed=17) -> float:
    out = C.c_double()
    _call(F.ctx.lib.tlrg_estimate_2norm_diff, A.h, F.h, iters, seed, C.byref(out))
    return out.value


def estimate_frob_diff(A: TlrMatrix, F: "TlrFactor", probes=64, seed=23) -> float:
    """Hutchinson estimate of ||P A P^T - L L^T||_F (north-star accuracy gate;
    the oracle's ref_estimate_frob_diff runs the identical estimator)."""
    out = C.c_double()
    _call(F.ctx.lib.tlrg_estimate_frob_diff, A.h, F.h, probes, seed, C.byref(out))
    return out.value


def accuracy(A: TlrMatrix, F: "TlrFactor", probes=64, seed=23, solve_seed=7):
    """The north-star accuracy block, computed the
    same way as oracle.ref.accuracy: relative Frobenius residual, 2-norm
    residual, backward / forward solve error, rank distribution of L."""
    from .util import rank_summary
    fa = frob_norm(A)
    fd = estimate_frob_diff(A, F, probes, seed)
    r2 = estimate_2norm_diff(A, F, 50, 17)
    a2 = estimate_2norm(A, 50, 1)
    x = rng_gaussians(solve_seed, A.n, A.ctx)
    b = tlr_matvec(A, x)
    xs = factor_solve(F, b)
    bwd = float(np.linalg.norm(tlr_matvec(A, xs) - b) / np.linalg.norm(b))
    fwd = float(np.linalg.norm(xs - x) / np.linalg.norm(x))
    L = F.L
    out = {"resid_frob_rel": fd / fa, "resid_frob": fd, "A_frob": fa, "resid_2norm": r2,
           "resid_2norm_rel": r2 / a2, "backward_err": bwd, "forward_err": fwd,
           "L_lowrank_bytes": int(L.memory_report()["low_rank_bytes"])}
    out.update(rank_summary(L.ranks()))
    return out


# --------------------------------------------------------- building blocks --
def _dblocks_flat(A: TlrMatrix, D):
    if D is None:
        return None, None, None
    nb, b = A.nb, A.b
    dd, de, ds = np.zeros(nb * b), np.zeros(nb * b), np.zeros(nb * b, np.uint8)
    for j, blk in enumerate(D):
        d, e, s2 = (blk.d, blk.e, blk.start2x2) if isinstance(blk, BlockDiagonal) else blk
        r = len(d)
        dd[j * b:j * b + r] = d
        de[j * b:j * b + r - 1] = e
        ds[j * b:j * b + r] = s2
    return dd, de, ds


def _sample(A: TlrMatrix, D, k, rows, ws: AraWorkspace, omegas, transpose):
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    if rows.size == 0:
        return []
    width = omegas[0].shape[1]
    om = _f64(np.concatenate([np.asarray(o, np.float64).T.ravel() for o in omegas]))
    outrows = [A.tile_rows(k) if transpose else A.tile_rows(int(i)) for i in rows]
    out = np.empty(sum(outrows) * width)
    dd, de, ds = _dblocks_flat(A, D)
    _call(A.ctx.lib.tlrg_sample_left, A.h, _d(dd), _d(de), _u8(ds), k, len(rows), _i(rows),
          ws.parallel_buffers, _d(om), width, int(transpose), _d(out))
    res, off = [], 0
    for r in outrows:
        res.append(out[off:off + r * width].reshape(width, r).T.copy())
        off += r * width
    return res


def sample_left(A: TlrMatrix, D, k, rows, ws: AraWorkspace, omegas):
    """ara.cpp:275-286 (D = None selects the Cholesky expression)."""
    return _sample(A, D, k, rows, ws, omegas, False)


def sample_left_transpose(A: TlrMatrix, D, k, rows, ws: AraWorkspace, q):
    """ara.cpp:288-300."""
    return _sample(A, D, k, rows, ws, q, True)


@dataclass
class TileApprox:
    i: int
    Q: np.ndarray
    B: np.ndarray
    converged: bool
    rounds_resident: int


def chol_ara_update(A: TlrMatrix, D, k, cfg: AraConfig, ws: AraWorkspace = None,
                    stats: Optional[dict] = None) -> List[TileApprox]:
    """ara.cpp:302-419: dynamic-batched ARA of every tile below the diagonal of
    column k.  Returns tiles in ascending i.  ``stats`` (a dict) receives the
    device time and work counters of the call."""
    ws = ws or AraWorkspace()
    dd, de, ds = _dblocks_flat(A, D)
    h = C.c_void_p()
    c, w = cfg.c(), ws.c()
    _call(A.ctx.lib.tlrg_chol_ara_update, A.h, _d(dd), _d(de), _u8(ds), k, C.byref(c),
          C.byref(w), C.byref(h))
    lib = A.ctx.lib
    out = []
    if stats is not None:
        v = np.zeros(5)
        lib.tlrg_ara_stats(h, _d(v))
        stats.update(t_device=v[0], tile_rounds=int(v[1]), flops_ref=v[2], t_fused=v[3],
                     flops_fused=v[4])
    try:
        rk = A.tile_rows(k)
        for t in range(lib.tlrg_ara_count(h)):
            info = np.zeros(4, np.int32)
            lib.tlrg_ara_tile(h, t, _i(info), None, None)
            i, q = int(info[0]), int(info[1])
            Q = np.zeros(max(A.tile_rows(i) * q, 1))
            B = np.zeros(max(rk * q, 1))
            lib.tlrg_ara_tile(h, t, _i(info), _d(Q), _d(B))
            out.append(TileApprox(i, Q[:A.tile_rows(i) * q].reshape(q, -1).T.copy()
                                  if q else np.zeros((A.tile_rows(i), 0)),
                                  B[:rk * q].reshape(q, -1).T.copy() if q else np.zeros((rk, 0)),
                                  bool(info[2]), int(info[3])))
    finally:
        lib.tlrg_ara_free(h)
    return out


def ara_column_seed(root: int, i: int, k: int) -> int:
    from .util import tile_seed
    return tile_seed(root, 0xFAC7, i, k)


# ------------------------------------------------------------ dense helpers --
def rng_gaussians(seed: int, n: int, ctx=None) -> np.ndarray:
    """First n draws of tlr::Rng(seed).gaussian() (util.hpp:24-53), on device."""
    ctx = _ctx(ctx)
    out = np.empty(n)
    _call(ctx.lib.tlrg_rng_gaussians, ctx.h, seed & 0xFFFFFFFFFFFFFFFF, n, _d(out))
    return out


def orthog(Q, Y, seed, ctx=None):
    """orthog (dense_kernels.cpp:379-420) with a fresh tlr::Rng(seed)."""
    ctx = _ctx(ctx)
    Y = np.asfortranarray(Y, dtype=np.float64).copy(order="F")
    rows, k = Y.shape
    q = 0 if Q is None else Q.shape[1]
    Qf = np.asfortranarray(Q, dtype=np.float64) if q else None
    R = np.zeros((k, k), order="F")
    cn, nm, nd = np.zeros(k), np.zeros(k), np.zeros(1)
    _call(ctx.lib.tlrg_orthog, ctx.h, Qf.ctypes.data_as(L.dp) if q else None, rows, q,
          Y.ctypes.data_as(L.dp), k, seed, R.ctypes.data_as(L.dp), _d(cn), _d(nm), _d(nd))
    return np.array(Y), np.array(R), cn, nm, float(nd[0])


def dense_cholesky(A, ctx=None):
    ctx = _ctx(ctx)
    n = A.shape[0]
    Af = np.asfortranarray(A, dtype=np.float64)
    Lm = np.zeros((n, n), order="F")
    fail = C.c_int32()
    _call(ctx.lib.tlrg_potrf, ctx.h, Af.ctypes.data_as(L.dp), n, Lm.ctypes.data_as(L.dp),
          C.byref(fail))
    return np.tril(np.array(Lm)), int(fail.value)


def jacobi_svd(A, cut, force_single=False, ctx=None):
    """One-sided Jacobi SVD of the recompression core (svd_truncate,
    dense_kernels.cpp:422-454): returns (A V sorted, V, sigma, rank)."""
    ctx = _ctx(ctx)
    m, n = A.shape
    Af = np.asfortranarray(A, dtype=np.float64)
    US = np.zeros((m, n), order="F")
    V = np.zeros((n, n), order="F")
    sig = np.zeros(n)
    rk = C.c_int32()
    _call(ctx.lib.tlrg_jacobi_svd, ctx.h, Af.ctypes.data_as(L.dp), m, n, float(cut),
          1 if force_single else 0, US.ctypes.data_as(L.dp), V.ctypes.data_as(L.dp), _d(sig),
          C.byref(rk))
    return np.array(US), np.array(V), sig, int(rk.value)


def dense_ldl(A, ctx=None):
    ctx = _ctx(ctx)
    n = A.shape[0]
    Af = np.asfortranarray(A, dtype=np.float64)
    Lm = np.zeros((n, n), order="F")
    d, e = np.zeros(n), np.zeros(max(n - 1, 1))
    s2, p, info = np.zeros(n, np.uint8), np.zeros(n, np.int32), C.c_int32()
    _call(ctx.lib.tlrg_dense_ldl, ctx.h, Af.ctypes.data_as(L.dp), n, Lm.ctypes.data_as(L.dp),
          _d(d), _d(e), _u8(s2), _i(p), C.byref(info))
    return np.array(Lm), BlockDiagonal(d, e[:n - 1], s2), p, int(info.value)


def schur_compensation(Dk, eps, ctx=None):
    """Diagonal of schur_compensation (factor.cpp:286-288) and ||R||_F."""
    ctx = _ctx(ctx)
    n = Dk.shape[0]
    Df = np.asfortranarray(Dk, dtype=np.float64)
    out = np.zeros(n)
    fr = C.c_double()
    _call(ctx.lib.tlrg_schur_compensation, ctx.h, Df.ctypes.data_as(L.dp), n, eps, _d(out),
          C.byref(fr))
    return out, fr.value


def gemm(alpha, A, ta, B, tb, beta=0.0, Cm=None, ctx=None):
    ctx = _ctx(ctx)
    A = np.asfortranarray(A, dtype=np.float64)
    B = np.asfortranarray(B, dtype=np.float64)
    M = A.shape[1] if ta else A.shape[0]
    K = A.shape[0] if ta else A.shape[1]
    N = B.shape[0] if tb else B.shape[1]
    Cm = np.zeros((M, N), order="F") if Cm is None else np.asfortranarray(Cm, np.float64).copy(
        order="F")
    _call(ctx.lib.tlrg_gemm, ctx.h, M, N, K, int(ta), int(tb), alpha, A.ctypes.data_as(L.dp),
          B.ctypes.data_as(L.dp), beta, Cm.ctypes.data_as(L.dp))
    return np.array(Cm)


def build_tlr(coords, kernel_kind, ell, nugget, b, eps, compressor=0, cfg: AraConfig = None,
              ctx=None) -> TlrMatrix:
    """build_tlr (tlr_matrix.cpp:98-152) on the device.  ``coords`` are the points
    in matrix order, shape (N, dim) (see geometry.kd_order(...).matrix_order()).
    kernel_kind 0 = exp(-r/ell), 1 = exp(-r^2/(2 ell^2)); compressor 0 ARA, 1 SVD."""
    ctx = _ctx(ctx)
    X = _f64(coords)
    cfg = cfg or AraConfig()
    c = cfg.c()
    h = C.c_void_p()
    _call(ctx.lib.tlrg_build, ctx.h, X.shape[1], X.shape[0], _d(X), kernel_kind, ell, nugget, b,
          eps, compressor, C.byref(c), C.byref(h))
    return TlrMatrix(h, ctx)
