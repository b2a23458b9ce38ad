// tlr_b200.cpp — the reference-side binding over the C ABI (include/tlrg.h).
// Compiled against the reference headers (oracle/Makefile builds it in place
// into oracle/_ref/ for the conformance test; a maintainer adds it to proj/src).
#include "tlr_b200.hpp"

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
  tlrg_factor_options fo{o.schur_compensation ? 1 : 0, o.diag_shift};
  tlrg_matrix h = upload(A);  // consumed by tlrg_factorize (even when it fails)
  tlrg_factor f = nullptr;
  tlrg_status st{};
  check(tlrg_factorize(context(), h, mode, &cfg, &ws, &fo, &f, &st), st);
  // the device factor is released on every exit path (download may throw)
  std::unique_ptr<tlrg_factor_s, void (*)(tlrg_factor)> guard(f, tlrg_factor_free);
  return download(f, std::move(A), mode == 0 ? FactorMode::Cholesky : FactorMode::LDLT);
}

}  // namespace

TlrFactor tlr_cholesky_b200(TlrMatrix A, const AraConfig& cfg, const AraWorkspace& ws,
                            const FactorOptions& opts) {
  return run(std::move(A), cfg, ws, opts, 0);
}
TlrFactor tlr_ldlt_b200(TlrMatrix A, const AraConfig& cfg, const AraWorkspace& ws,
                        FactorOptions opts) {
  return run(std::move(A), cfg, ws, opts, 1);
}

}  // namespace tlr
