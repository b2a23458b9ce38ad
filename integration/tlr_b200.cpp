// tlr_b200.cpp — the reference-side binding over the C ABI (include/tlrg.h).
// Compiled against the reference headers (oracle/Makefile builds it in place
// into oracle/_ref/ for the conformance test; a maintainer adds it to proj/src).
#include "tlr_b200.hpp"

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "tlr/errors.hpp"
#include "tlrg.h"

namespace tlr {
namespace {

void check(int rc, const tlrg_status& st) {
  if (rc == 0) return;
  const std::string msg = std::string("B200 factorization: ") + st.msg;
  if (rc == 2) throw ConfigError(msg);
  if (rc == 3) throw DataError(msg);
  if (rc == 4) throw NumericError(msg, st.index);
  throw Error(msg);
}

tlrg_ctx context() {  // one context per process, device 0 (a serving process pins its GPU)
  static tlrg_ctx c = [] {
    tlrg_ctx h = nullptr;
    tlrg_status st{};
    check(tlrg_create(0, &h, &st), st);
    return h;
  }();
  return c;
}

// TlrMatrix (tlr_matrix.hpp:26-40) -> flat reference layout -> device
tlrg_matrix upload(const TlrMatrix& A) {
  std::vector<double> diag, U, V;
  std::vector<int32_t> ranks;
  for (const DenseTile& d : A.diag) diag.insert(diag.end(), d.data(), d.data() + d.size());
  for (const LowRankTile& t : A.lower) {
    ranks.push_back(t.rank());
    U.insert(U.end(), t.U.data(), t.U.data() + t.U.size());
    V.insert(V.end(), t.V.data(), t.V.data() + t.V.size());
  }
  if (U.empty()) U.push_back(0.0);
  if (V.empty()) V.push_back(0.0);
  tlrg_matrix h = nullptr;
  tlrg_status st{};
  check(tlrg_matrix_upload(context(), A.n, A.b, A.eps, diag.data(),
                           ranks.empty() ? nullptr : ranks.data(), U.data(), V.data(), &h, &st),
        st);
  return h;
}

// device factor -> the reference's TlrFactor (factor.hpp:25-33), reusing A's tiles
TlrFactor download(tlrg_factor f, TlrMatrix&& A, FactorMode mode) {
  tlrg_matrix Lh = tlrg_factor_L(f);
  const int nb = A.nb;
  std::vector<int32_t> ranks((size_t)nb * (nb - 1) / 2);
  tlrg_matrix_ranks(Lh, ranks.data());
  size_t nd = 0, nu = 0, nv = 0;
  for (int k = 0; k < nb; ++k) nd += (size_t)A.tile_rows(k) * A.tile_rows(k);
  for (int i = 1, t = 0; i < nb; ++i)
    for (int j = 0; j < i; ++j, ++t) {
      nu += (size_t)A.tile_rows(i) * ranks[t];
      nv += (size_t)A.tile_rows(j) * ranks[t];
    }
  std::vector<double> diag(nd), U(nu + 1), V(nv + 1);
  tlrg_status st{};
  check(tlrg_matrix_download(Lh, diag.data(), U.data(), V.data(), &st), st);
  TlrFactor F;
  F.L = std::move(A);
  F.mode = mode;
  size_t od = 0, ou = 0, ov = 0;
  for (int k = 0; k < nb; ++k) {
    const int r = F.L.tile_rows(k);
    F.L.diag[k] = DenseTile(r, r);
    std::memcpy(F.L.diag[k].data(), diag.data() + od, sizeof(double) * r * r);
    od += (size_t)r * r;
  }
  for (int i = 1, t = 0; i < nb; ++i)
    for (int j = 0; j < i; ++j, ++t) {
      const int q = ranks[t], ri = F.L.tile_rows(i), rj = F.L.tile_rows(j);
      LowRankTile& T = F.L.lower[t];
      T.U = DenseTile(ri, q);
      T.V = DenseTile(rj, q);
      if (q) {
        std::memcpy(T.U.data(), U.data() + ou, sizeof(double) * ri * q);
        std::memcpy(T.V.data(), V.data() + ov, sizeof(double) * rj * q);
      }
      ou += (size_t)ri * q;
      ov += (size_t)rj * q;
    }
  if (mode == FactorMode::PivotedCholesky) {
    std::vector<int32_t> p(nb);
    tlrg_factor_perm(f, p.data());
    F.perm.assign(p.begin(), p.end());
  }
  if (mode == FactorMode::LDLT) {
    F.D.resize(nb);
    F.intra_perm.resize(nb);
    for (int k = 0; k < nb; ++k) {
      const int r = F.L.tile_rows(k);
      BlockDiagonal D(r);
      std::vector<int32_t> perm(r);
      tlrg_factor_dblock(f, k, D.d.data(), D.e.data(), D.start2x2.data(), perm.data());
      F.D[k] = std::move(D);
      F.intra_perm[k].assign(perm.begin(), perm.end());
    }
  }
  tlrg_stats s{};
  std::vector<int32_t> rounds(nb);
  std::vector<double> piv(nb);
  tlrg_factor_stats(f, &s, rounds.data(), piv.data());
  F.eps = F.L.eps;
  F.stats.t_sampling = s.t_sampling;
  F.stats.t_projection = s.t_projection;
  F.stats.t_reduction = s.t_reduction;
  F.stats.t_dense = s.t_dense;
  F.stats.t_orthog = s.t_orthog;
  F.stats.t_misc = s.t_misc;
  F.stats.t_pivot_select = s.t_pivot_select;
  F.stats.wall = s.wall;
  F.stats.compensation_frob = s.compensation_frob;
  F.stats.modified_diagonals = s.modified_diagonals;
  F.stats.tile_rounds_resident = s.tile_rounds_resident;
  F.stats.ara_rounds.assign(rounds.begin(), rounds.end());
  F.stats.pivot_trace = piv;
  return F;
}

TlrFactor run(TlrMatrix A, const AraConfig& c, const AraWorkspace& w, const FactorOptions& o,
              int mode) {
  tlrg_ara_config cfg{c.block_samples, c.eps, c.max_rank, c.window, c.safety,
                      c.recompress ? 1 : 0, c.seed};
  tlrg_workspace ws{w.parallel_buffers, w.dense_buffers, w.subset_capacity};
  tlrg_factor_options fo{o.schur_compensation ? 1 : 0, o.diag_shift,
                         o.pivot_norm == PivotNorm::Frobenius ? 0 : 1, o.pivot_power_iters};
  tlrg_matrix h = upload(A);  // consumed by tlrg_factorize (even when it fails)
  tlrg_factor f = nullptr;
  tlrg_status st{};
  check(tlrg_factorize(context(), h, mode, &cfg, &ws, &fo, &f, &st), st);
  // the device factor is released on every exit path (download may throw)
  std::unique_ptr<tlrg_factor_s, void (*)(tlrg_factor)> guard(f, tlrg_factor_free);
  return download(f, std::move(A),
                  mode == 0   ? FactorMode::Cholesky
                  : mode == 1 ? FactorMode::LDLT
                              : FactorMode::PivotedCholesky);
}

// D blocks of the LDL^T columns (dense_kernels.hpp:28-53) in the C ABI's flat
// nb*b layout; empty when the expression has no D (Chol mode).
struct FlatD {
  std::vector<double> d, e;
  std::vector<uint8_t> s2;
  FlatD(const TlrMatrix& m, const std::vector<BlockDiagonal>* D, SampleMode mode) {
    if (mode != SampleMode::LDL || !D) return;
    const size_t n = (size_t)m.nb * m.b;
    d.assign(n, 0.0);
    e.assign(n, 0.0);
    s2.assign(n, 0);
    for (int j = 0; j < (int)D->size() && j < m.nb; ++j) {
      const BlockDiagonal& B = (*D)[j];
      const size_t o = (size_t)j * m.b;
      std::copy(B.d.begin(), B.d.end(), d.begin() + o);
      std::copy(B.e.begin(), B.e.end(), e.begin() + o);
      std::copy(B.start2x2.begin(), B.start2x2.end(), s2.begin() + o);
    }
  }
  const double* dd() const { return d.empty() ? nullptr : d.data(); }
  const double* de() const { return e.empty() ? nullptr : e.data(); }
  const uint8_t* ds2() const { return s2.empty() ? nullptr : s2.data(); }
};

struct MatrixGuard {
  tlrg_matrix h;
  ~MatrixGuard() { tlrg_matrix_free(h); }
};

}  // namespace

std::vector<TileApprox> chol_ara_update_b200(const TlrMatrix& m,
                                             const std::vector<BlockDiagonal>* d, int k,
                                             const AraConfig& c, const AraWorkspace& w,
                                             SampleMode mode, FactorStats* stats) {
  if (k + 1 >= m.nb) return {};
  MatrixGuard A{upload(m)};
  FlatD D(m, d, mode);
  tlrg_ara_config cfg{c.block_samples, c.eps, c.max_rank, c.window, c.safety,
                      c.recompress ? 1 : 0, c.seed};
  tlrg_workspace ws{w.parallel_buffers, w.dense_buffers, w.subset_capacity};
  tlrg_ara a = nullptr;
  tlrg_status st{};
  check(tlrg_chol_ara_update(A.h, D.dd(), D.de(), D.ds2(), k, &cfg, &ws, &a, &st), st);
  std::unique_ptr<tlrg_ara_s, void (*)(tlrg_ara)> guard(a, tlrg_ara_free);
  const int rk = m.tile_rows(k);
  std::vector<TileApprox> out;
  for (int i = k + 1; i < m.nb; ++i)  // structurally zero tiles: rank 0, converged, 0 rounds
    out.push_back({i, DenseTile(m.tile_rows(i), 0), DenseTile(rk, 0), true, 0});
  for (int t = 0, n = tlrg_ara_count(a); t < n; ++t) {
    int32_t info[4];
    tlrg_ara_tile(a, t, info, nullptr, nullptr);
    TileApprox& T = out[info[0] - k - 1];
    T.Q = DenseTile(m.tile_rows(info[0]), info[1]);
    T.B = DenseTile(rk, info[1]);
    tlrg_ara_tile(a, t, info, T.Q.data(), T.B.data());
    T.converged = info[2] != 0;
    T.rounds_resident = info[3];
  }
  if (stats) {
    double s5[5];
    tlrg_ara_stats(a, s5);
    stats->t_sampling += s5[0];  // one device region: sampling, projection and orthog fused
    for (const TileApprox& T : out) stats->tile_rounds_resident += T.rounds_resident;
  }
  return out;
}

std::vector<DenseTile> sample_left_b200(const TlrMatrix& m, const std::vector<BlockDiagonal>* d,
                                        int k, const std::vector<int>& row_idx,
                                        const AraWorkspace& ws,
                                        const std::vector<DenseTile>& omega, SampleMode mode,
                                        bool transpose) {
  if (row_idx.empty()) return {};
  if (ws.parallel_buffers / (int)row_idx.size() < 1)  // ara.cpp:281-284
    throw ConfigError("sample_left: workspace smaller than one buffer per tile");
  MatrixGuard A{upload(m)};
  FlatD D(m, d, mode);
  const int width = omega.empty() ? 0 : omega[0].cols();
  std::vector<double> in, out;
  size_t otot = 0;
  for (size_t t = 0; t < row_idx.size(); ++t) {
    in.insert(in.end(), omega[t].data(), omega[t].data() + omega[t].size());
    otot += (size_t)(transpose ? m.tile_rows(k) : m.tile_rows(row_idx[t])) * width;
  }
  in.push_back(0.0);
  out.assign(otot + 1, 0.0);
  std::vector<int32_t> rows(row_idx.begin(), row_idx.end());
  tlrg_status st{};
  check(tlrg_sample_left(A.h, D.dd(), D.de(), D.ds2(), k, (int32_t)rows.size(), rows.data(),
                         ws.parallel_buffers, in.data(), width, transpose ? 1 : 0, out.data(), &st),
        st);
  std::vector<DenseTile> res;
  size_t o = 0;
  for (int i : row_idx) {
    const int r = transpose ? m.tile_rows(k) : m.tile_rows(i);
    DenseTile Y(r, width);
    std::memcpy(Y.data(), out.data() + o, sizeof(double) * r * width);
    o += (size_t)r * width;
    res.push_back(std::move(Y));
  }
  return res;
}

TlrFactor tlr_cholesky_b200(TlrMatrix A, const AraConfig& cfg, const AraWorkspace& ws,
                            const FactorOptions& opts) {
  return run(std::move(A), cfg, ws, opts, 0);
}
TlrFactor tlr_ldlt_b200(TlrMatrix A, const AraConfig& cfg, const AraWorkspace& ws,
                        FactorOptions opts) {
  return run(std::move(A), cfg, ws, opts, 1);
}
TlrFactor tlr_cholesky_pivoted_b200(TlrMatrix A, const AraConfig& cfg, const AraWorkspace& ws,
                                    const FactorOptions& opts) {
  return run(std::move(A), cfg, ws, opts, 2);
}

}  // namespace tlr
