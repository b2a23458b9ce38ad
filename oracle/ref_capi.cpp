// ORACLE / TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// A thin C ABI over the UNMODIFIED reference library (/root/reference/proj/src,
// compiled in place by oracle/Makefile into oracle/_ref/libtlr_ref.so).  Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
// legs may load it, and only as the checker or the CPU baseline.
//
// Every entry point forwards to the reference function named beside it.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include <omp.h>

#include "tlr/ara.hpp"
#include "tlr/factor.hpp"
#include "tlr/geometry.hpp"
#include "tlr/solve.hpp"
#include "tlr/tlr_matrix.hpp"
#include "tlr/util.hpp"

using namespace tlr;

namespace {
thread_local std::string g_err;
int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const ConfigError*>(&e)) return 2;
  if (dynamic_cast<const DataError*>(&e)) return 3;
  if (dynamic_cast<const DimensionError*>(&e)) return 3;
  if (dynamic_cast<const NumericError*>(&e)) return 4;
  return 1;
}
AraConfig mk_cfg(int bs, double eps, int max_rank, int window, double safety,
                 int recompress, unsigned long long seed) {
  AraConfig c;
  c.block_samples = bs;
  c.eps = eps;
  c.max_rank = max_rank;
  c.window = window;
  c.safety = safety;
  c.recompress = recompress != 0;
  c.seed = seed;
  return c;
}
AraWorkspace mk_ws(int pb, int db, int subset) {
  AraWorkspace w;
  w.parallel_buffers = pb;
  w.dense_buffers = db;
  w.subset_capacity = subset;
  return w;
}
DenseTile tile_from(const double* p, int r, int c) {
  DenseTile t(r, c);
  if (r * c) std::memcpy(t.data(), p, sizeof(double) * r * c);
  return t;
}
void tile_to(const DenseTile& t, double* p) {
  if (t.size()) std::memcpy(p, t.data(), sizeof(double) * t.size());
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(int t) { if (t > 0) omp_set_num_threads(t); }
int ref_max_threads() { return omp_get_max_threads(); }

// ---- util.hpp:10-53 -------------------------------------------------------
unsigned long long ref_mix64(unsigned long long x) { return mix64(x); }
unsigned long long ref_tile_seed(unsigned long long r, unsigned long long p,
                                 unsigned long long i, unsigned long long j) {
  return tile_seed(r, p, i, j);
}
unsigned long long ref_ara_column_seed(unsigned long long root, int i, int k) {
  return ara_column_seed(root, i, k);
}
void ref_rng_gaussians(unsigned long long seed, long long n, double* out) {
  Rng r(seed);
  for (long long t = 0; t < n; ++t) out[t] = r.gaussian();
}
void ref_rng_uniforms(unsigned long long seed, long long n, double* out) {
  Rng r(seed);
  for (long long t = 0; t < n; ++t) out[t] = r.uniform();
}

// ---- geometry.cpp:20-168 --------------------------------------------------
// coords_out: N*dim doubles in MATRIX order (point of matrix index p).
int ref_points(int kind, int n, unsigned long long seed, int tile, double* coords_out) {
  try {
    PointSet ps = generate_points(static_cast<PointKind>(kind), n, seed);
    if (tile > 0) ps = kd_order(std::move(ps), tile);
    for (int p = 0; p < n; ++p)
      std::memcpy(coords_out + (size_t)p * ps.dim, ps.point(ps.ordering[p]),
                  sizeof(double) * ps.dim);
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// ---- tlr_matrix.cpp:98-152 build_tlr ---------------------------------------
// Points are given in matrix order (identity ordering).
void* ref_build(int dim, int n, const double* coords, int kernel_kind, double ell,
                double nugget, int b, double eps, int compressor, int bs,
                unsigned long long seed, int* status) {
  try {
    ProblemSpec spec;
    spec.points.dim = dim;
    spec.points.coords.assign(coords, coords + (size_t)n * dim);
    spec.points.ordering.resize(n);
    for (int i = 0; i < n; ++i) spec.points.ordering[i] = i;
    spec.kernel = {static_cast<KernelKind>(kernel_kind), ell, nugget};
    AraConfig cfg;
    cfg.block_samples = bs;
    cfg.seed = seed;
    auto* A = new TlrMatrix(build_tlr(spec, b, eps, static_cast<Compressor>(compressor), cfg));
    *status = 0;
    return A;
  } catch (const std::exception& e) { *status = fail(e); return nullptr; }
}

// Dense kernel block (rows r0.., cols c0..) via kernel_entry (geometry.cpp:151-168).
int ref_kernel_block(int dim, int n, const double* coords, int kernel_kind, double ell,
                     double nugget, long long r0, int nr, long long c0, int nc, double* out) {
  try {
    PointSet ps;
    ps.dim = dim;
    ps.coords.assign(coords, coords + (size_t)n * dim);
    ps.ordering.resize(n);
    for (int i = 0; i < n; ++i) ps.ordering[i] = i;
    KernelSpec ks{static_cast<KernelKind>(kernel_kind), ell, nugget};
    for (int j = 0; j < nc; ++j)
      for (int i = 0; i < nr; ++i)
        out[(size_t)j * nr + i] = kernel_entry(ks, ps, (int)(r0 + i), (int)(c0 + j));
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// Assemble a TlrMatrix from flat parts: diag tiles concatenated, ranks per
// lower tile (index i(i-1)/2+j), U/V payloads concatenated in that order.
void* ref_matrix_from_parts(long long n, int b, double eps, const double* diag,
                            const int* ranks, const double* U, const double* V) {
  auto* A = new TlrMatrix(n, b);
  A->eps = eps;
  size_t off = 0;
  for (int i = 0; diag && i < A->nb; ++i) {  // diag == null: keep the zero tiles
    int r = A->tile_rows(i);
    A->diag[i] = tile_from(diag + off, r, r);
    off += (size_t)r * r;
  }
  size_t ou = 0, ov = 0;
  for (int i = 1; i < A->nb; ++i)
    for (int j = 0; j < i; ++j) {
      int k = ranks[(size_t)i * (i - 1) / 2 + j];
      LowRankTile& t = A->tile(i, j);
      t.U = tile_from(U + ou, A->tile_rows(i), k);
      t.V = tile_from(V + ov, A->tile_rows(j), k);
      ou += (size_t)A->tile_rows(i) * k;
      ov += (size_t)A->tile_rows(j) * k;
    }
  return A;
}
// the whole matrix in the flat layout of ref_matrix_from_parts (null = skip)
void ref_matrix_flat(void* h, double* diag, double* U, double* V) {
  auto* A = static_cast<TlrMatrix*>(h);
  size_t off = 0, ou = 0, ov = 0;
  for (int i = 0; i < A->nb; ++i) {
    if (diag) tile_to(A->diag[i], diag + off);
    off += A->diag[i].size();
  }
  for (int i = 1; i < A->nb; ++i)
    for (int j = 0; j < i; ++j) {
      const LowRankTile& t = A->tile(i, j);
      if (U) tile_to(t.U, U + ou);
      if (V) tile_to(t.V, V + ov);
      ou += t.U.size();
      ov += t.V.size();
    }
}
void* ref_matrix_copy(void* h) { return new TlrMatrix(*static_cast<TlrMatrix*>(h)); }
void ref_matrix_free(void* h) { delete static_cast<TlrMatrix*>(h); }
void ref_matrix_info(void* h, long long* n, int* b, int* nb, double* eps) {
  auto* A = static_cast<TlrMatrix*>(h);
  *n = A->n; *b = A->b; *nb = A->nb; *eps = A->eps;
}
void ref_matrix_ranks(void* h, int* out) {
  auto* A = static_cast<TlrMatrix*>(h);
  for (int i = 1; i < A->nb; ++i)
    for (int j = 0; j < i; ++j) out[(size_t)i * (i - 1) / 2 + j] = A->rank(i, j);
}
void ref_matrix_diag(void* h, int k, double* out) { tile_to(static_cast<TlrMatrix*>(h)->diag[k], out); }
void ref_matrix_set_diag(void* h, int k, const double* in) {
  auto* A = static_cast<TlrMatrix*>(h);
  int r = A->tile_rows(k);
  A->diag[k] = tile_from(in, r, r);
}
void ref_matrix_tile(void* h, int i, int j, double* U, double* V) {
  auto* A = static_cast<TlrMatrix*>(h);
  tile_to(A->tile(i, j).U, U);
  tile_to(A->tile(i, j).V, V);
}
int ref_matrix_write(void* h, const char* path) {
  try { write_tlr(*static_cast<TlrMatrix*>(h), path); return 0; }
  catch (const std::exception& e) { return fail(e); }
}
void* ref_matrix_read(const char* path, int* status) {
  try { auto* A = new TlrMatrix(read_tlr(path)); *status = 0; return A; }
  catch (const std::exception& e) { *status = fail(e); return nullptr; }
}
// memory_report (tlr_matrix.cpp:229-249): [total, dense, low_rank]
void ref_memory_report(void* h, unsigned long long* out3) {
  MemoryReport r = memory_report(*static_cast<TlrMatrix*>(h));
  out3[0] = r.total_bytes; out3[1] = r.dense_bytes; out3[2] = r.low_rank_bytes;
}
int ref_tlr_matvec(void* h, const double* x, double* y) {
  try {
    auto* A = static_cast<TlrMatrix*>(h);
    auto r = tlr_matvec(*A, std::span<const double>(x, A->n));
    std::memcpy(y, r.data(), sizeof(double) * A->n);
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}
double ref_estimate_2norm(void* h, int iters, unsigned long long seed) {
  return estimate_2norm(*static_cast<TlrMatrix*>(h), iters, seed);
}

// ---- factor.cpp:290-306 --------------------------------------------------
// mode 0 Chol, 1 LDLT, 2 pivoted.  A is COPIED (the caller keeps its handle).
// stats_out[10] = t_sampling, t_projection, t_reduction, t_dense, t_orthog,
//                 t_misc, t_pivot_select, wall, compensation_frob, modified_diagonals
// pivot selection of the next ref_factor(mode = 2) call (FactorOptions, factor.hpp:17-18)
static int g_pivot_norm = 0, g_pivot_iters = 50;
void ref_set_pivot(int norm, int iters) {
  g_pivot_norm = norm;
  g_pivot_iters = iters;
}
void* ref_factor(void* h, int mode, int bs, double eps, int max_rank, int window,
                 double safety, int recompress, unsigned long long seed, int pb, int db,
                 int subset, int schur, double shift, int* status) {
  try {
    TlrMatrix A = *static_cast<TlrMatrix*>(h);
    AraConfig cfg = mk_cfg(bs, eps, max_rank, window, safety, recompress, seed);
    AraWorkspace ws = mk_ws(pb, db, subset);
    FactorOptions o;
    o.schur_compensation = schur != 0;
    o.diag_shift = shift;
    o.pivot_norm = g_pivot_norm == 0 ? PivotNorm::Frobenius : PivotNorm::TwoNormPower;
    o.pivot_power_iters = g_pivot_iters;
    TlrFactor* F = new TlrFactor(
        mode == 0 ? tlr_cholesky(std::move(A), cfg, ws, o)
        : mode == 1 ? tlr_ldlt(std::move(A), cfg, ws, o)
                    : tlr_cholesky_pivoted(std::move(A), cfg, ws, o));
    *status = 0;
    return F;
  } catch (const std::exception& e) {
    *status = fail(e);
    if (auto* ne = dynamic_cast<const NumericError*>(&e)) g_err += " @" + std::to_string(ne->index);
    return nullptr;
  }
}
void ref_factor_free(void* f) { delete static_cast<TlrFactor*>(f); }
void* ref_factor_L(void* f) { return &static_cast<TlrFactor*>(f)->L; }
int ref_factor_mode(void* f) {
  auto m = static_cast<TlrFactor*>(f)->mode;
  return m == FactorMode::Cholesky ? 0 : m == FactorMode::LDLT ? 1 : 2;
}
void ref_factor_stats(void* f, double* out10, int* ara_rounds, double* pivot_trace,
                      unsigned long long* tile_rounds) {
  auto& s = static_cast<TlrFactor*>(f)->stats;
  double v[10] = {s.t_sampling, s.t_projection, s.t_reduction, s.t_dense, s.t_orthog,
                  s.t_misc, s.t_pivot_select, s.wall, s.compensation_frob,
                  (double)s.modified_diagonals};
  std::memcpy(out10, v, sizeof v);
  for (size_t k = 0; k < s.ara_rounds.size(); ++k) ara_rounds[k] = s.ara_rounds[k];
  for (size_t k = 0; k < s.pivot_trace.size(); ++k) pivot_trace[k] = s.pivot_trace[k];
  *tile_rounds = s.tile_rounds_resident;
}
// LDL blocks of column k: d[n], e[n-1], start2x2[n], intra_perm[n]
void ref_factor_dblock(void* f, int k, double* d, double* e, unsigned char* s2, int* perm) {
  auto* F = static_cast<TlrFactor*>(f);
  const BlockDiagonal& D = F->D[k];
  std::memcpy(d, D.d.data(), sizeof(double) * D.d.size());
  if (!D.e.empty()) std::memcpy(e, D.e.data(), sizeof(double) * D.e.size());
  std::memcpy(s2, D.start2x2.data(), D.start2x2.size());
  for (size_t i = 0; i < F->intra_perm[k].size(); ++i) perm[i] = F->intra_perm[k][i];
}
void ref_factor_perm(void* f, int* out) {
  auto* F = static_cast<TlrFactor*>(f);
  for (size_t i = 0; i < F->perm.size(); ++i) out[i] = F->perm[i];
}
int ref_factor_solve(void* f, const double* b, double* x) {
  try {
    auto* F = static_cast<TlrFactor*>(f);
    auto r = factor_solve(*F, std::span<const double>(b, F->L.n));
    std::memcpy(x, r.data(), sizeof(double) * F->L.n);
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}
int ref_factor_apply(void* f, const double* x, double* y) {
  try {
    auto* F = static_cast<TlrFactor*>(f);
    auto r = factor_apply(*F, std::span<const double>(x, F->L.n));
    std::memcpy(y, r.data(), sizeof(double) * F->L.n);
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}
double ref_estimate_2norm_diff(void* a, void* f, int iters, unsigned long long seed) {
  return estimate_2norm_diff(*static_cast<TlrMatrix*>(a), *static_cast<TlrFactor*>(f), iters, seed);
}
// ---- Frobenius accuracy gate (the reference has none) --
// Restated here with the reference's public operators so both sides run the
// identical estimator (device: tlrg_estimate_frob_diff):
//   ||A||_F^2 exact tile-wise = sum_k ||A_kk||_F^2 + 2 sum_{i>j} tr((U^T U)(V^T V));
//   ||P A P^T - L L^T||_F^2 ~= (1/p) sum_t ||E g_t||^2, g_t = first n draws of
//   Rng(tile_seed(seed, 0xF20B, t, 0)), E v as difference_apply (solve.cpp:283-297).
double ref_frob_norm(void* a) {
  const TlrMatrix& A = *static_cast<TlrMatrix*>(a);
  double s = 0.0;
#pragma omp parallel for reduction(+ : s) schedule(dynamic)
  for (int k = 0; k < A.nb; ++k) {
    const DenseTile& d = A.diag[k];
    for (long long e = 0; e < (long long)d.size(); ++e) s += d.data()[e] * d.data()[e];
  }
  const long long nt = (long long)A.lower.size();
  double l = 0.0;
#pragma omp parallel for reduction(+ : l) schedule(dynamic)
  for (long long t = 0; t < nt; ++t) {
    const LowRankTile& T = A.lower[t];
    const int r = T.rank();
    for (int p = 0; p < r; ++p)
      for (int q = 0; q < r; ++q) {
        double gu = 0.0, gv = 0.0;
        for (int i = 0; i < T.U.rows(); ++i) gu += T.U(i, p) * T.U(i, q);
        for (int i = 0; i < T.V.rows(); ++i) gv += T.V(i, p) * T.V(i, q);
        l += gu * gv;
      }
  }
  return std::sqrt(s + 2.0 * l);
}
double ref_estimate_frob_diff(void* a, void* f, int probes, unsigned long long seed) {
  const TlrMatrix& A = *static_cast<TlrMatrix*>(a);
  const TlrFactor& F = *static_cast<TlrFactor*>(f);
  const std::int64_t n = A.n;
  auto perm = [&](const std::vector<double>& v, bool inverse) {
    std::vector<double> out(v.size());
    for (int k = 0; k < F.L.nb; ++k) {
      const int src = F.perm[k], rk = F.L.tile_rows(k);
      if (!inverse)
        std::memcpy(out.data() + F.L.block_offset(k), v.data() + F.L.block_offset(src), 8 * rk);
      else
        std::memcpy(out.data() + F.L.block_offset(src), v.data() + F.L.block_offset(k), 8 * rk);
    }
    return out;
  };
  double acc = 0.0;
  for (int t = 0; t < probes; ++t) {
    Rng rng(tile_seed(seed, 0xF20BULL, (std::uint64_t)t, 0));
    std::vector<double> g(n);
    for (double& x : g) x = rng.gaussian();
    std::vector<double> av = F.perm.empty()
                                 ? tlr_matvec(A, g)
                                 : perm(tlr_matvec(A, perm(g, true)), false);
    std::vector<double> lv = factor_apply(F, g);
    double e2 = 0.0;
    for (std::int64_t i = 0; i < n; ++i) e2 += (av[i] - lv[i]) * (av[i] - lv[i]);
    acc += e2;
  }
  return std::sqrt(acc / probes);
}

int ref_factor_write(void* f, const char* path) {
  try { write_factor(*static_cast<TlrFactor*>(f), path); return 0; }
  catch (const std::exception& e) { return fail(e); }
}
void* ref_factor_read(const char* path, int* status) {
  try { auto* F = new TlrFactor(read_factor(path)); *status = 0; return F; }
  catch (const std::exception& e) { *status = fail(e); return nullptr; }
}

// ---- ara.cpp:275-300 sample_left / sample_left_transpose -----------------
// D blocks (LDL mode): dd[nb*b], de[nb*b], ds2[nb*b] per column (or null).
static std::vector<BlockDiagonal> mk_dblocks(const TlrMatrix& m, const double* dd,
                                             const double* de, const unsigned char* ds2) {
  std::vector<BlockDiagonal> d(m.nb);
  for (int j = 0; j < m.nb; ++j) {
    int r = m.tile_rows(j);
    d[j] = BlockDiagonal(r);
    for (int t = 0; t < r; ++t) {
      d[j].d[t] = dd[(size_t)j * m.b + t];
      if (t < r - 1) d[j].e[t] = de[(size_t)j * m.b + t];
      d[j].start2x2[t] = ds2[(size_t)j * m.b + t];
    }
  }
  return d;
}
int ref_sample_left(void* h, const double* dd, const double* de, const unsigned char* ds2,
                    int k, int nrows, const int* rows, int pb, const double* omega,
                    int width, int transpose, double* out) {
  try {
    auto* m = static_cast<TlrMatrix*>(h);
    std::vector<BlockDiagonal> d;
    if (dd) d = mk_dblocks(*m, dd, de, ds2);
    std::vector<int> r(rows, rows + nrows);
    AraWorkspace ws;
    ws.parallel_buffers = pb;
    std::vector<DenseTile> om;
    size_t off = 0;
    for (int t = 0; t < nrows; ++t) {
      int rr = transpose ? m->tile_rows(r[t]) : m->tile_rows(k);
      om.push_back(tile_from(omega + off, rr, width));
      off += (size_t)rr * width;
    }
    SampleMode mode = dd ? SampleMode::LDL : SampleMode::Chol;
    auto ys = transpose ? sample_left_transpose(*m, dd ? &d : nullptr, k, r, ws, om, mode)
                        : sample_left(*m, dd ? &d : nullptr, k, r, ws, om, mode);
    off = 0;
    for (auto& y : ys) { tile_to(y, out + off); off += y.size(); }
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// ---- ara.cpp:302-419 chol_ara_update --------------------------------------
// Returns a handle to the TileApprox list.
struct AraOut { std::vector<TileApprox> t; };
void* ref_chol_ara_update(void* h, const double* dd, const double* de,
                          const unsigned char* ds2, int k, int bs, double eps,
                          int max_rank, int window, double safety, int recompress,
                          unsigned long long seed, int pb, int subset, int* status) {
  try {
    auto* m = static_cast<TlrMatrix*>(h);
    std::vector<BlockDiagonal> d;
    if (dd) d = mk_dblocks(*m, dd, de, ds2);
    AraConfig cfg = mk_cfg(bs, eps, max_rank, window, safety, recompress, seed);
    AraWorkspace ws = mk_ws(pb, 20, subset);
    auto* o = new AraOut;
    o->t = chol_ara_update(*m, dd ? &d : nullptr, k, cfg, ws,
                           dd ? SampleMode::LDL : SampleMode::Chol);
    *status = 0;
    return o;
  } catch (const std::exception& e) { *status = fail(e); return nullptr; }
}
int ref_ara_count(void* o) { return (int)static_cast<AraOut*>(o)->t.size(); }
// info[4] = i, rank, converged, rounds_resident
void ref_ara_tile(void* o, int t, int* info, double* Q, double* B) {
  const TileApprox& a = static_cast<AraOut*>(o)->t[t];
  info[0] = a.i; info[1] = a.Q.cols(); info[2] = a.converged; info[3] = a.rounds_resident;
  if (Q) tile_to(a.Q, Q);
  if (B) tile_to(a.B, B);
}
void ref_ara_free(void* o) { delete static_cast<AraOut*>(o); }

// ---- ara.cpp:254-273 ara_single on a dense operator ----------------------
int ref_ara_single_dense(const double* A, int rows, int cols, int bs, double eps,
                         int max_rank, int window, double safety, int recompress,
                         unsigned long long seed, int* info, double* Q, double* B) {
  try {
    DenseTile T = tile_from(A, rows, cols);
    DenseSampler op(T);
    AraResult r = ara_single(op, mk_cfg(bs, eps, max_rank, window, safety, recompress, seed));
    info[0] = r.rank; info[1] = r.converged; info[2] = r.rounds;
    tile_to(r.Q, Q);
    tile_to(r.B, B);
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// ---- dense_kernels.cpp:379-420 orthog -------------------------------------
// Q (rows x q, may be q=0), Y (rows x k) in/out; R (k x k); norms/mass (k).
// The rng is seeded with `seed` and its state after the call is summarised by
// the next gaussian it would draw (next_draw).
int ref_orthog(const double* Q, int rows, int q, double* Y, int k, unsigned long long seed,
               double* R, double* col_norms, double* new_mass, double* next_draw) {
  try {
    DenseTile Qt = q > 0 ? tile_from(Q, rows, q) : DenseTile();
    DenseTile Yt = tile_from(Y, rows, k);
    Rng rng(seed);
    OrthogResult o = orthog(Qt, Yt, rng);
    tile_to(Yt, Y);
    tile_to(o.R, R);
    for (int j = 0; j < k; ++j) { col_norms[j] = o.col_norms[j]; new_mass[j] = o.new_mass[j]; }
    if (next_draw) *next_draw = rng.gaussian();
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// ---- dense kernels used by the factor driver ------------------------------
// dense_ldl (dense_kernels.cpp:236-281)
int ref_dense_ldl(const double* A, int n, double* L, double* d, double* e,
                  unsigned char* s2, int* perm) {
  try {
    LdlResult r = dense_ldl(tile_from(A, n, n));
    tile_to(r.L, L);
    std::memcpy(d, r.D.d.data(), sizeof(double) * n);
    if (n > 1) std::memcpy(e, r.D.e.data(), sizeof(double) * (n - 1));
    std::memcpy(s2, r.D.start2x2.data(), n);
    for (int i = 0; i < n; ++i) perm[i] = r.perm[i];
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}
// modified_cholesky (dense_kernels.cpp:283-309); returns modified flag in *mod
int ref_modified_cholesky(const double* A, int n, double* L, int* mod) {
  try {
    ModCholResult r = modified_cholesky(tile_from(A, n, n));
    tile_to(r.L, L);
    *mod = r.modified;
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}
// schur_compensation (factor.cpp:286-288): diagonal of the correction
int ref_schur_compensation(const double* Dk, int n, double eps, double* diag_out) {
  try {
    DenseTile c = schur_compensation(tile_from(Dk, n, n), eps);
    for (int i = 0; i < n; ++i) diag_out[i] = c(i, i);
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}
// svd_truncate (dense_kernels.cpp:422-454): returns rank; U (m x rank, scaled), V (n x rank)
int ref_svd_truncate(const double* A, int m, int n, double eps, double* U, double* V) {
  SvdTruncation s = svd_truncate(tile_from(A, m, n), eps);
  tile_to(s.U, U);
  tile_to(s.V, V);
  return s.rank;
}
double ref_spectral_norm_estimate(const double* A, int m, int n, int iters,
                                  unsigned long long seed) {
  return spectral_norm_estimate(tile_from(A, m, n), iters, seed);
}

}  // extern "C"
