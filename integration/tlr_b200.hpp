// tlr_b200.hpp — drop-in entry points for the reference library (proj/, namespace tlr).
//
// A maintainer adds integration/tlr_b200.cpp to proj/src and links
// paper_2108_11932_b200/lib/libtlrg.so; callers switch
//   tlr::tlr_cholesky(A, cfg, ws, opts)  ->  tlr::tlr_cholesky_b200(A, cfg, ws, opts)
//   tlr::tlr_ldlt(A, cfg, ws, opts)      ->  tlr::tlr_ldlt_b200(A, cfg, ws, opts)
//   tlr::tlr_cholesky_pivoted(...)       ->  tlr::tlr_cholesky_pivoted_b200(...)
// (include/tlr/factor.hpp:35-41).  Same value semantics: A is consumed, the
// returned TlrFactor is an ordinary host TlrFactor that tlr::factor_solve,
// tlr::factor_apply, tlr::estimate_2norm_diff, tlr::write_factor accept.
#pragma once
#include "tlr/ara.hpp"
#include "tlr/factor.hpp"

namespace tlr {
TlrFactor tlr_cholesky_b200(TlrMatrix A, const AraConfig& cfg, const AraWorkspace& ws,
                            const FactorOptions& opts = {});
TlrFactor tlr_ldlt_b200(TlrMatrix A, const AraConfig& cfg, const AraWorkspace& ws,
                        FactorOptions opts = {});
TlrFactor tlr_cholesky_pivoted_b200(TlrMatrix A, const AraConfig& cfg, const AraWorkspace& ws,
                                    const FactorOptions& opts = {});

// Building blocks the reference's own tests call directly (ara.hpp:102-130),
// evaluated on the device.  Same arguments, results and exceptions.
std::vector<TileApprox> chol_ara_update_b200(const TlrMatrix& m,
                                             const std::vector<BlockDiagonal>* d, int k,
                                             const AraConfig& cfg, const AraWorkspace& ws,
                                             SampleMode mode, FactorStats* stats = nullptr);
std::vector<DenseTile> sample_left_b200(const TlrMatrix& m, const std::vector<BlockDiagonal>* d,
                                        int k, const std::vector<int>& row_idx,
                                        const AraWorkspace& ws,
                                        const std::vector<DenseTile>& omega, SampleMode mode,
                                        bool transpose = false);
}  // namespace tlr
