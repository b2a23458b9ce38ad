// ORACLE / TEST INFRASTRUCTURE — conformance driver for the drop-in binding.
// Builds a covariance TLR matrix with the reference, factors it with BOTH the
// reference (tlr::tlr_cholesky / tlr_ldlt) and the B200 path through the
// reference's own types (tlr::tlr_cholesky_b200, integration/tlr_b200.cpp),
// and evaluates both with the reference's own estimate_2norm_diff and
// factor_solve.  Loaded by tests/test_gpu_integration.py.
#include <cmath>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "../integration/tlr_b200.hpp"
#include "tlr/geometry.hpp"
#include "tlr/solve.hpp"
#include "tlr/tlr_matrix.hpp"

using namespace tlr;

extern "C" int conf_run(int mode, int n, int b, double eps, int bs, double nugget,
                        double* out /* 8: resid_ref resid_b200 bwd_ref bwd_b200
                                       rankmean_ref rankmean_b200 rank_equal_frac status */,
                        char* err, int errlen) {
  try {
    ProblemSpec spec;
    spec.points = kd_order(generate_points(PointKind::Grid2D, n, 0), b);
    spec.kernel.kind = mode == 0 ? KernelKind::IsotropicExponential : KernelKind::SquaredExponential;
    spec.kernel.correlation_length = mode == 0 ? 0.1 : 0.2;
    spec.kernel.nugget = nugget;
    AraConfig cfg;
    cfg.block_samples = bs;
    cfg.eps = eps;
    cfg.seed = 5;
    AraWorkspace ws;
    ws.subset_capacity = 4;
    TlrMatrix A = build_tlr(spec, b, eps, Compressor::ARA, cfg);
    TlrFactor Fr = mode == 0 ? tlr_cholesky(A, cfg, ws) : tlr_ldlt(A, cfg, ws);
    TlrFactor Fg = mode == 0 ? tlr_cholesky_b200(A, cfg, ws) : tlr_ldlt_b200(A, cfg, ws);
    out[0] = estimate_2norm_diff(A, Fr, 50, 17);
    out[1] = estimate_2norm_diff(A, Fg, 50, 17);
    std::vector<double> x(n), bvec;
    for (int i = 0; i < n; ++i) x[i] = std::sin(0.37 * i + 1.0);
    bvec = tlr_matvec(A, x);
    auto bwd = [&](const TlrFactor& F) {
      std::vector<double> xs = factor_solve(F, bvec), r = tlr_matvec(A, xs);
      double num = 0, den = 0;
      for (int i = 0; i < n; ++i) {
        num += (r[i] - bvec[i]) * (r[i] - bvec[i]);
        den += bvec[i] * bvec[i];
      }
      return std::sqrt(num / den);
    };
    out[2] = bwd(Fr);
    out[3] = bwd(Fg);
    double sr = 0, sg = 0, eq = 0;
    for (size_t t = 0; t < Fr.L.lower.size(); ++t) {
      sr += Fr.L.lower[t].rank();
      sg += Fg.L.lower[t].rank();
      eq += Fr.L.lower[t].rank() == Fg.L.lower[t].rank();
    }
    const double nt = std::max<size_t>(1, Fr.L.lower.size());
    out[4] = sr / nt;
    out[5] = sg / nt;
    out[6] = eq / nt;
    out[7] = 0;
    return 0;
  } catch (const std::exception& e) {
    std::snprintf(err, errlen, "%s", e.what());
    out[7] = 1;
    return 1;
  }
}
