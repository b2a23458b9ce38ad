// tlr_b200_dropin.cpp — the reference's own entry points resolved to the B200 path.
//
// Linking this file in place of the CPU definitions makes every existing caller
// of the reference API run on the device without a source change:
//   tlr::tlr_cholesky / tlr::tlr_ldlt          (include/tlr/factor.hpp:35-41)
//   tlr::tlr_cholesky_pivoted                  (include/tlr/factor.hpp:37-39)
//   tlr::chol_ara_update                        (include/tlr/ara.hpp:126-130)
//   tlr::sample_left / sample_left_transpose    (include/tlr/ara.hpp:102-114)
// A maintainer either drops those definitions from proj/src/factor.cpp and
// proj/src/ara.cpp, or (what oracle/Makefile does for the conformance suite)
// keeps the reference objects and marks those symbols weak with
//   objcopy --weaken-symbol=<mangled name> factor.o
// so that these strong definitions win at link time.  The unmodified
// proj/tests/test_factor.cpp, test_ara.cpp and test_solve.cpp then exercise the
// B200 factorization (tests/test_gpu_conformance.py).
#include "tlr_b200.hpp"

namespace tlr {

TlrFactor tlr_cholesky(TlrMatrix A, const AraConfig& cfg, const AraWorkspace& ws,
                       const FactorOptions& opts) {
  return tlr_cholesky_b200(std::move(A), cfg, ws, opts);
}

TlrFactor tlr_ldlt(TlrMatrix A, const AraConfig& cfg, const AraWorkspace& ws,
                   FactorOptions opts) {
  return tlr_ldlt_b200(std::move(A), cfg, ws, opts);
}

TlrFactor tlr_cholesky_pivoted(TlrMatrix A, const AraConfig& cfg, const AraWorkspace& ws,
                               const FactorOptions& opts) {
  return tlr_cholesky_pivoted_b200(std::move(A), cfg, ws, opts);
}

std::vector<TileApprox> chol_ara_update(const TlrMatrix& m, const std::vector<BlockDiagonal>* d,
                                        int k, const AraConfig& cfg, const AraWorkspace& ws,
                                        SampleMode mode, FactorStats* stats) {
  return chol_ara_update_b200(m, d, k, cfg, ws, mode, stats);
}

std::vector<DenseTile> sample_left(const TlrMatrix& m, const std::vector<BlockDiagonal>* d, int k,
                                   const std::vector<int>& row_idx, const AraWorkspace& ws,
                                   const std::vector<DenseTile>& omega, SampleMode mode) {
  return sample_left_b200(m, d, k, row_idx, ws, omega, mode, false);
}

std::vector<DenseTile> sample_left_transpose(const TlrMatrix& m,
                                             const std::vector<BlockDiagonal>* d, int k,
                                             const std::vector<int>& row_idx,
                                             const AraWorkspace& ws,
                                             const std::vector<DenseTile>& q, SampleMode mode) {
  return sample_left_b200(m, d, k, row_idx, ws, q, mode, true);
}

}  // namespace tlr
