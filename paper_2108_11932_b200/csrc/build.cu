// Construction of a TLR matrix from a covariance kernel on the device
// (build_tlr, tlr_matrix.cpp:98-152; kernel_entry, geometry.cpp:151-168).
// Tiles are materialised in HBM in batches and compressed by the batched ARA
// with the reference's per-tile seeds tile_seed(seed, 0xb11d, i, j) — so the
// streams, and hence the ranks, follow the reference draw for draw — or by a
// one-sided Jacobi SVD truncation (Compressor::SVD).
#include <algorithm>
#include <cmath>

#include "core.h"

namespace tlrg {

namespace {
struct KTile {
  double* out;  // nr x nc, ld nr
  long long r0, c0;
  int nr, nc;
};

__global__ void __launch_bounds__(256) kernel_tiles(const KTile* tiles, const double* X, int dim,
                                                    int kind, double ell, double nugget,
                                                    int* bad) {
  const KTile T = tiles[blockIdx.y];
  long long tot = (long long)T.nr * T.nc;
  for (long long e = blockIdx.x * 256LL + threadIdx.x; e < tot; e += (long long)gridDim.x * 256) {
    int r = (int)(e % T.nr), c = (int)(e / T.nr);
    long long i = T.r0 + r, j = T.c0 + c;
    double v;
    if (i == j) {
      v = 1.0 + nugget;
    } else {
      double d2 = 0.0;
      for (int d = 0; d < dim; ++d) {
        double t = __dsub_rn(X[i * dim + d], X[j * dim + d]);
        d2 = __dadd_rn(d2, __dmul_rn(t, t));  // same evaluation order as the reference
      }
      v = kind == 0 ? exp(-sqrt(d2) / ell) : exp(-d2 / __dmul_rn(2.0, __dmul_rn(ell, ell)));
    }
    if (!isfinite(v)) atomicExch(bad, 1);
    T.out[r + (long long)c * T.nr] = v;
  }
}
}  // namespace

std::unique_ptr<Matrix> build_tlr_device(Ctx& C, int dim, int64_t n, const double* coords_host,
                                         int kind, double ell, double nugget, int b, double eps,
                                         int compressor, const AraCfg& cfg_in) {
  if (!(eps > 0)) config_error("build_tlr: eps must be positive");
  if (n < 1 || b < 1 || b > n) config_error("TlrMatrix: bad dimensions");
  if (kind != 0 && kind != 1) config_error("kernel_entry: unsupported kernel");
  if (dim < 1 || dim > 3) config_error("build_tlr: bad dimension");
  auto M = std::make_unique<Matrix>();
  M->ctx = &C;
  M->n = n;
  M->b = b;
  M->nb = (int)((n + b - 1) / b);
  M->eps = eps;
  const int nb = M->nb;
  size_t nt = (size_t)nb * (nb - 1) / 2;
  M->rank.assign(nt, 0);
  M->U.assign(nt, nullptr);
  M->V.assign(nt, nullptr);
  TLRG_CUDA(cudaMallocAsync(&M->diag, sizeof(double) * (size_t)nb * b * b, C.st_main));
  double* X = C.buf<double>("bt_X", (size_t)n * dim);
  TLRG_CUDA(cudaMemcpyAsync(X, coords_host, 8 * (size_t)n * dim, cudaMemcpyHostToDevice, C.st));
  int* bad = C.buf<int>("bt_bad", 1);
  TLRG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), C.st));
  auto eval = [&](const std::vector<KTile>& tiles) {
    for (size_t o = 0; o < tiles.size(); o += 65535) {
      std::vector<KTile> part(tiles.begin() + o, tiles.begin() + std::min(tiles.size(), o + 65535));
      dim3 grid(std::max(1, std::min(64, (b * b + 255) / 256)), (unsigned)part.size());
      kernel_tiles<<<grid, 256, 0, C.st>>>(C.push(part), X, dim, kind, ell, nugget, bad);
      TLRG_CUDA(cudaGetLastError());
      ++C.launches;
    }
  };
  {
    std::vector<KTile> d;
    for (int k = 0; k < nb; ++k)
      d.push_back({M->diag + (size_t)k * b * b, (long long)k * b, (long long)k * b, M->rows(k),
                   M->rows(k)});
    eval(d);
  }
  auto S = std::make_shared<Store>();
  S->st = C.st_main;
  S->owner = &C;
  M->stores.push_back(S);
  AraCfg cfg = cfg_in;
  cfg.eps = eps;
  // batches of lower tiles bounded by ~12 GB of dense staging + ARA bases
  std::vector<std::pair<int, int>> all;
  for (int i = 1; i < nb; ++i)
    for (int j = 0; j < i; ++j) all.push_back({i, j});
  const size_t per = (size_t)2 * b * b * 8;
  const size_t batch = std::max<size_t>(148, std::min<size_t>(all.size(), (12ull << 30) / per));
  ColumnStats cst;
  for (size_t o = 0; o < all.size(); o += batch) {
    const int T = (int)std::min(batch, all.size() - o);
    double* D = C.buf<double>("bt_dense", (size_t)T * b * b);
    std::vector<KTile> kt;
    for (int s = 0; s < T; ++s) {
      auto [i, j] = all[o + s];
      kt.push_back({D + (size_t)s * b * b, (long long)i * b, (long long)j * b, M->rows(i),
                    M->rows(j)});
    }
    eval(kt);
    if (compressor == 1) {
      // svd_truncate (dense_kernels.cpp:422-454) via one-sided Jacobi per tile
      std::vector<SvdTask> sv;
      double* Vv = C.buf<double>("bt_V", (size_t)T * b * b);
      double* sig = C.buf<double>("bt_sig", (size_t)T * b);
      double* work = C.buf<double>("bt_work", (size_t)T * 2 * b * b);
      int* rk = C.buf<int>("bt_rank", (size_t)T);
      for (int s = 0; s < T; ++s) {
        auto [i, j] = all[o + s];
        SvdTask t{};
        t.A = D + (size_t)s * b * b;
        t.V = Vv + (size_t)s * b * b;
        t.sig = sig + (size_t)s * b;
        t.work = work + (size_t)s * 2 * b * b;
        t.rank_out = rk + s;
        t.m = M->rows(i);
        t.n = M->rows(j);
        t.cut = eps;
        sv.push_back(t);
      }
      jacobi_svd(C.push(sv), T, b, C.st, b);
      ++C.launches;
      std::vector<int> hr(T);
      TLRG_CUDA(cudaMemcpyAsync(hr.data(), rk, sizeof(int) * T, cudaMemcpyDeviceToHost, C.st));
      C.sync();
      std::vector<CopyItem> cp;
      for (int s = 0; s < T; ++s) {
        auto [i, j] = all[o + s];
        long long t = tri_index(i, j);
        int r = std::min(hr[s], std::min(M->rows(i), M->rows(j)));
        M->rank[t] = r;
        if (!r) continue;
        M->U[t] = S->alloc((size_t)M->rows(i) * r);
        M->V[t] = S->alloc((size_t)M->rows(j) * r);
        cp.push_back({D + (size_t)s * b * b, M->U[t], M->rows(i), M->rows(i), M->rows(i), r});
        cp.push_back({Vv + (size_t)s * b * b, M->V[t], M->rows(j), M->rows(j), M->rows(j), r});
      }
      if (!cp.empty()) batched_copy(C.push(cp), (int)cp.size(), C.st);
      C.sync();
      continue;
    }
    AraSlots sl;
    sl.cols = b;
    for (int s = 0; s < T; ++s) {
      auto [i, j] = all[o + s];
      sl.rows.push_back(M->rows(i));
      sl.cap.push_back(std::min(M->rows(i), M->rows(j)));
      sl.seeds.push_back(tile_seed(cfg.seed, 0xb11dULL, i, j));
    }
    AraOperator op;
    op.sample_plan = [&](const double* Om, double* Y, long long Ys, const int* done,
                         std::vector<std::vector<GemmProblem>>& stages) {
      stages.assign(1, {});
      for (int s = 0; s < T; ++s) {
        GemmProblem g{};
        g.A = D + (size_t)s * b * b; g.lda = sl.rows[s];
        g.B = Om + (size_t)s * b * cfg.bs; g.ldb = b;
        g.C = Y + s * Ys; g.ldc = sl.rows[s];
        g.M = sl.rows[s]; g.N = cfg.bs; g.K = b; g.alpha = 1.0; g.skip = done + s;
        stages[0].push_back(g);
      }
    };
    op.project = [&](const std::vector<int>& q, const double* Q, long long Qs, double* Bb,
                     const std::vector<long long>& boff) {
      std::vector<GemmProblem> pr;
      for (int s = 0; s < T; ++s) {
        if (!q[s]) continue;
        GemmProblem g{};
        g.A = D + (size_t)s * b * b; g.lda = sl.rows[s]; g.transA = 1;
        g.B = Q + s * Qs; g.ldb = sl.rows[s];
        g.C = Bb + boff[s]; g.ldc = b;
        g.M = b; g.N = q[s]; g.K = sl.rows[s]; g.alpha = 1.0;
        pr.push_back(g);
      }
      C.gemm(pr);
    };
    op.fused.on = true;
    for (int s = 0; s < T; ++s) {
      op.fused.Ad.push_back(D + (size_t)s * b * b);
      op.fused.ldad.push_back(sl.rows[s]);
    }
    std::vector<int> order(T);
    for (int s = 0; s < T; ++s) order[s] = s;
    AraOut out;
    ara_batch(C, sl, op, cfg, *S, order, cst, out);
    for (int s = 0; s < T; ++s) {
      auto [i, j] = all[o + s];
      long long t = tri_index(i, j);
      M->rank[t] = out.rank[s];
      M->U[t] = out.U[s];
      M->V[t] = out.V[s];
    }
  }
  int hb = 0;
  TLRG_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, C.st));
  C.sync();
  if (hb) data_error("build_tlr: non-finite kernel entry");
  return M;
}

}  // namespace tlrg
