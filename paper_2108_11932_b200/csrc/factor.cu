// Left-looking TLR Cholesky / LDL^T driver on the device (factor.cpp:115-306).
// Columns are sequential; inside a column everything is batched over tiles:
//   Gram + H (dense phase) -> SYRK D_k -> Schur compensation -> POTRF / BK LDL
//   -> dynamic-batched ARA -> panel TRSM (+perm, D^{-1}) -> pointer update.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "core.h"

namespace tlrg {

namespace {
struct Ev {
  cudaEvent_t e;
  Ev() { cudaEventCreate(&e); }
  ~Ev() { cudaEventDestroy(e); }
};
double elapsed(Ev& a, Ev& b) {
  float f = 0;
  cudaEventElapsedTime(&f, a.e, b.e);
  return f * 1e-3;
}

__global__ void copy_tile_kernel(const double* src, double* dst, long long n) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x)
    dst[t] = src[t];
}
void dcopy(const double* src, double* dst, long long n, cudaStream_t st) {
  if (n <= 0) return;
  int blocks = (int)std::min<long long>((n + 255) / 256, 148 * 8);
  copy_tile_kernel<<<blocks, 256, 0, st>>>(src, dst, n);
  TLRG_CUDA(cudaGetLastError());
}

// BlockDiagonal::first_singular_block (dense_kernels.cpp:221-234)
__global__ void first_singular_kernel(const double* d, const double* e, const uint8_t* s2, int n,
                                      int* out) {
  int k = 0, r = -1;
  while (k < n) {
    if (s2[k]) {
      if (d[k] * d[k + 1] - e[k] * e[k] == 0.0) {
        r = k;
        break;
      }
      k += 2;
    } else {
      if (d[k] == 0.0) {
        r = k;
        break;
      }
      k += 1;
    }
  }
  *out = r;
}

// BlockDiagonal::floor_eigenvalues (dense_kernels.cpp:146-185)
__global__ void floor_eigen_kernel(double* d, double* e, const uint8_t* s2, int n, double delta) {
  int k = 0;
  while (k < n) {
    if (s2[k]) {
      double a = d[k], b = e[k], c = d[k + 1];
      double mean = 0.5 * (a + c);
      double rad = hypot(0.5 * (a - c), b);
      double l1 = mean - rad, l2 = mean + rad;
      if (l1 < delta || l2 < delta) {
        double f1 = fmax(l1, delta), f2 = fmax(l2, delta);
        double vx, vy;
        if (fabs(b) > 0.0) {
          vx = b;
          vy = l2 - a;
        } else {
          vx = a >= c ? 1.0 : 0.0;
          vy = a >= c ? 0.0 : 1.0;
        }
        double nv = hypot(vx, vy);
        vx /= nv;
        vy /= nv;
        d[k] = f2 * vx * vx + f1 * vy * vy;
        e[k] = (f2 - f1) * vx * vy;
        d[k + 1] = f2 * vy * vy + f1 * vx * vx;
      }
      k += 2;
    } else {
      if (d[k] < delta) d[k] = delta;
      k += 1;
    }
  }
}

__global__ void transpose_kernel(const double* A, double* B, int n) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)n * n) return;
  int i = (int)(t % n), j = (int)(t / n);
  B[j + (long long)i * n] = A[t];
}
__global__ void scatter_perm_kernel(const double* M, double* At, const int* perm, int n) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)n * n) return;
  int i = (int)(t % n), j = (int)(t / n);
  At[perm[i] + (long long)perm[j] * n] = M[t];
}
__global__ void add_diag_kernel(double* A, int n, double v) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) A[i + (long long)i * n] += v;
}
}  // namespace

void potrf_impl(double* A, int n, int* info, DescArena& desc, cudaStream_t st);

bool potrf_device(Ctx& C, double* A, int n) {
  int* info = C.buf<int>("potrf_info", 1);
  potrf_impl(A, n, info, C.desc, C.st);
  C.launches += 2 * ((n + 31) / 32);
  int* h = C.pinned_ints(1);
  TLRG_CUDA(cudaMemcpyAsync(h, info, sizeof(int), cudaMemcpyDeviceToHost, C.st));
  C.sync();
  return h[0] < 0;
}

bool modified_cholesky_device(Ctx& C, double* A, int n) {
  // A holds the ORIGINAL tile on entry (the caller restores it after a failed
  // potrf); dense_kernels.cpp:283-309.
  double* W = C.buf<double>("mc_W", (size_t)n * n);
  double* LT = C.buf<double>("mc_LT", (size_t)n * n);
  double* Mm = C.buf<double>("mc_M", (size_t)n * n);
  double* At = C.buf<double>("mc_At", (size_t)n * n);
  double* d = C.buf<double>("mc_d", (size_t)n);
  double* e = C.buf<double>("mc_e", (size_t)n);
  uint8_t* s2 = C.buf<uint8_t>("mc_s2", (size_t)n);
  int* perm = C.buf<int>("mc_perm", (size_t)n);
  int* info = C.buf<int>("mc_info", 1);
  double* fs = C.buf<double>("mc_fs", 1);
  dcopy(A, W, (long long)n * n, C.st);
  sytrf_bk(W, n, d, e, s2, perm, info, C.st);
  frob_sq(A, (long long)n * n, fs, C.st);
  double* h = C.pinned_dbl(1);
  TLRG_CUDA(cudaMemcpyAsync(h, fs, sizeof(double), cudaMemcpyDeviceToHost, C.st));
  C.sync();
  double base = std::sqrt(h[0]);
  if (base == 0.0) base = 1.0;
  double delta = std::ldexp(base, -26);
  floor_eigen_kernel<<<1, 1, 0, C.st>>>(d, e, s2, n, delta);
  long long nn = (long long)n * n;
  transpose_kernel<<<(unsigned)((nn + 255) / 256), 256, 0, C.st>>>(W, LT, n);
  bd_apply(d, e, s2, n, LT, n, n, C.st);
  std::vector<GemmProblem> pr(1);
  GemmProblem& g = pr[0];
  g = GemmProblem{};
  g.A = W; g.lda = n; g.B = LT; g.ldb = n; g.C = Mm; g.ldc = n;
  g.M = n; g.N = n; g.K = n; g.alpha = 1.0; g.beta = 0.0;
  C.gemm(pr);
  scatter_perm_kernel<<<(unsigned)((nn + 255) / 256), 256, 0, C.st>>>(Mm, At, perm, n);
  C.launches += 5;
  for (int attempt = 0; attempt < 60; ++attempt) {
    dcopy(At, A, nn, C.st);
    if (potrf_device(C, A, n)) return true;
    add_diag_kernel<<<(n + 255) / 256, 256, 0, C.st>>>(At, n, delta);
    delta *= 8.0;
  }
  numeric_error("modified_cholesky: could not repair tile", -1);
}

// Schur compensation (factor.cpp:66-79): R = D - svd_trunc(D, eps), corr =
// diag(rowsum |R|).  D is symmetric PSD and numerically low rank at eps
// (measured: 13-58 singular values above eps at m = 256/512), so the truncation
// is computed by Rayleigh-Ritz on a sketched range: Q = orth(D orth(D Omega)),
// SVD of Q^T D Q (one-sided Jacobi), keep sigma > eps.  The block grows until
// at least 8 retained directions of slack remain (or it spans the tile).
void schur_compensation_device(Ctx& C, const double* Dk, int n, double eps, uint64_t seed,
                               double* corr, double* frob, int& rank_hint) {
  int p = std::max(32, rank_hint + 24);
  p = ((p + 7) / 8) * 8;
  if (p > n) p = n;
  for (int attempt = 0;; ++attempt) {
    double* Om = C.buf<double>("sc_Om", (size_t)n * p);
    double* Y = C.buf<double>("sc_Y", (size_t)n * p);
    double* Bm = C.buf<double>("sc_B", (size_t)p * p);
    double* Vm = C.buf<double>("sc_V", (size_t)p * p);
    double* R = C.buf<double>("sc_R", (size_t)p * p);
    double* Rp = C.buf<double>("sc_Rp", (size_t)2 * p * p);
    double* vec = C.buf<double>("sc_vec", (size_t)4 * p);
    uint8_t* df = C.buf<uint8_t>("sc_def", (size_t)p);
    double* work = C.buf<double>("sc_work", (size_t)2 * p * p);
    double* sig = C.buf<double>("sc_sig", (size_t)p);
    int* rk = C.buf<int>("sc_rank", 1);
    // replacement directions for rank-deficient sketch columns (not part of the
    // reference's streams): a counter-based gaussian pool consumed by cursor
    double* pool = C.buf<double>("sc_pool", (size_t)4 * n * p);
    double* screp = C.buf<double>("sc_rep", (size_t)n * p);
    long long* pcur = C.buf<long long>("sc_pcur", 1);
    TLRG_CUDA(cudaMemsetAsync(pcur, 0, sizeof(long long), C.st));
    fill_gaussian_philox(pool, 4LL * n * p, mix64(seed ^ 0x5c1ULL) + attempt, C.st);
    fill_gaussian_philox(Om, (long long)n * p, seed * 0x9E3779B97F4A7C15ULL + attempt, C.st);
    auto DtimesX = [&](const double* X, double* out) {
      std::vector<GemmProblem> pr(1);
      pr[0] = GemmProblem{};
      pr[0].A = Dk; pr[0].lda = n; pr[0].B = X; pr[0].ldb = n; pr[0].C = out; pr[0].ldc = n;
      pr[0].M = n; pr[0].N = p; pr[0].K = n; pr[0].alpha = 1.0;
      C.gemm(pr);
    };
    auto orth = [&](double* X) {
      std::vector<PanelTask> t(1);
      PanelTask& P = t[0];
      P = PanelTask{};
      P.Y = X; P.Q = nullptr; P.R = R; P.Rp = Rp; P.tiny = vec; P.col_norms = vec + p;
      P.new_mass = vec + 2 * p; P.deficient = df; P.gbuf = pool; P.gcursor = pcur;
      P.rep = screp; P.repC = nullptr; P.gcap = 4LL * n * p;
      P.rows = n; P.width = p; P.q = 0;
      PanelTask* d = C.push(t);
      panel_tau(d, 1, C.st);
      panel_mgs(d, 1, 0, 0, p, n, C.st);
      panel_mgs(d, 1, 1, 0, p, n, C.st);
      C.launches += 3;
    };
    DtimesX(Om, Y);
    orth(Y);
    DtimesX(Y, Om);  // power iteration
    orth(Om);
    DtimesX(Om, Y);  // Y = D Q
    {
      std::vector<GemmProblem> pr(1);
      pr[0] = GemmProblem{};
      pr[0].A = Om; pr[0].lda = n; pr[0].transA = 1; pr[0].B = Y; pr[0].ldb = n;
      pr[0].C = Bm; pr[0].ldc = p; pr[0].M = p; pr[0].N = p; pr[0].K = n; pr[0].alpha = 1.0;
      C.gemm(pr);
    }
    std::vector<SvdTask> sv(1);
    sv[0] = SvdTask{};
    sv[0].A = Bm; sv[0].V = Vm; sv[0].sig = sig; sv[0].work = work; sv[0].rank_out = rk;
    sv[0].n = p; sv[0].cut = eps;
    jacobi_svd(C.push(sv), 1, p, C.st);
    ++C.launches;
    int* h = C.pinned_ints(1);
    TLRG_CUDA(cudaMemcpyAsync(h, rk, sizeof(int), cudaMemcpyDeviceToHost, C.st));
    C.sync();
    int r = h[0];
    if (r > p - 8 && p < n) {
      p = std::min(n, 2 * p);
      continue;
    }
    rank_hint = r;
    // R = D - (Q A_B)(Q V_B)^T restricted to the r retained directions
    double* Xl = C.buf<double>("sc_Xl", (size_t)n * std::max(r, 1));
    double* Xr = C.buf<double>("sc_Xr", (size_t)n * std::max(r, 1));
    double* Rm = C.buf<double>("sc_Rm", (size_t)n * n);
    double* fp = C.buf<double>("sc_fp", (size_t)n);
    dcopy(Dk, Rm, (long long)n * n, C.st);
    if (r > 0) {
      std::vector<GemmProblem> pr(2);
      pr[0] = GemmProblem{};
      pr[0].A = Om; pr[0].lda = n; pr[0].B = Bm; pr[0].ldb = p; pr[0].C = Xl; pr[0].ldc = n;
      pr[0].M = n; pr[0].N = r; pr[0].K = p; pr[0].alpha = 1.0;
      pr[1] = pr[0];
      pr[1].B = Vm; pr[1].C = Xr;
      C.gemm(pr);
      std::vector<GemmProblem> p2(1);
      p2[0] = GemmProblem{};
      p2[0].A = Xl; p2[0].lda = n; p2[0].B = Xr; p2[0].ldb = n; p2[0].transB = 1;
      p2[0].C = Rm; p2[0].ldc = n; p2[0].M = n; p2[0].N = n; p2[0].K = r;
      p2[0].alpha = -1.0; p2[0].beta = 1.0;
      C.gemm(p2);
    }
    rowsum_abs_residual(Rm, nullptr, nullptr, n, 0, corr, fp, C.st);
    frob_sq(Rm, (long long)n * n, frob, C.st);  // ||R||_F^2
    C.launches += 3;
    return;
  }
}

std::unique_ptr<Factor> factorize(Ctx& C, std::unique_ptr<Matrix> A, int mode, const AraCfg& cfg,
                                  int parallel_buffers, const FactorOpts& opts_in) {
  if (!(cfg.eps > 0)) config_error("factor: eps must be positive");
  if (opts_in.shift < 0) config_error("factor: negative diagonal shift");
  if (cfg.bs < 1) config_error("factor: block_samples must be >= 1");
  (void)parallel_buffers;
  FactorOpts opts = opts_in;
  const bool ldl = mode == 1;
  if (ldl) opts.schur = false;  // factor.cpp:304
  auto t_wall0 = std::chrono::steady_clock::now();
  double flops0 = C.flops;
  long long launches0 = C.launches;
  const char* kt = std::getenv("TLRG_KTIMING");
  C.ktiming = kt && kt[0] == '1';
  C.kt_seconds = C.kt_flops = 0.0;
  C.kt_launches = 0;
  Ev d0, d1;
  cudaEventRecord(d0.e, C.st);

  auto F = std::make_unique<Factor>();
  F->mode = mode;
  F->eps = cfg.eps;
  F->L = std::move(A);
  Matrix& M = *F->L;
  const int nb = M.nb, b = M.b;
  Stats& S = F->stats;
  S.ara_rounds.assign(nb, 0);
  S.pivot_trace.assign(nb, 0.0);
  if (ldl) {
    TLRG_CUDA(cudaMalloc(&F->D.d, sizeof(double) * nb * b));
    TLRG_CUDA(cudaMalloc(&F->D.e, sizeof(double) * nb * b));
    TLRG_CUDA(cudaMalloc(&F->D.s2, nb * b));
    TLRG_CUDA(cudaMalloc(&F->D.perm, sizeof(int) * nb * b));
    TLRG_CUDA(cudaMemsetAsync(F->D.d, 0, sizeof(double) * nb * b, C.st));
    TLRG_CUDA(cudaMemsetAsync(F->D.e, 0, sizeof(double) * nb * b, C.st));
    TLRG_CUDA(cudaMemsetAsync(F->D.s2, 0, nb * b, C.st));
  }
  auto store = std::make_shared<Store>();
  M.stores.push_back(store);
  double* Dk = C.buf<double>("Dk", (size_t)b * b);
  double* akk = C.buf<double>("akk", (size_t)b * b);
  double* a0 = C.buf<double>("akk0", (size_t)b * b);
  double* corr = C.buf<double>("corr", (size_t)b);
  double* frob = C.buf<double>("cfrob", 1);
  double* piv = C.buf<double>("pivot", (size_t)nb);
  int* info = C.buf<int>("finfo", 2);
  int rank_hint = 0;
  Ev e0, e1, e2, e3, e4, e5;
  StreamPrep prep;

  for (int k = 0; k < nb; ++k) {
    const int rk = M.rows(k);
    double* diagk = M.diag + (size_t)k * b * b;
    // ---- gaussian streams of this column's ARA, generated on the side stream
    //      while the diagonal path runs
    column_prepare(C, M, k, cfg, prep);
    // ---- dense phase: Gram blocks, H_k, D_k = sum_j L_kj [D_j] L_kj^T ----------
    cudaEventRecord(e0.e, C.st);
    ColumnSetup cs;
    column_setup(C, M, k, F->D, cs);
    if (cs.K > 0) {
      double* Hk = C.buf<double>("Hk", (size_t)b * cs.K);
      std::vector<int> tk{k};
      column_H(C, M, cs, tk, Hk, (long long)b * cs.K);
      std::vector<GemmProblem> pr(1);
      pr[0] = GemmProblem{};
      pr[0].A = Hk; pr[0].lda = rk; pr[0].B = cs.Ucat; pr[0].ldb = rk; pr[0].transB = 1;
      pr[0].C = Dk; pr[0].ldc = rk; pr[0].M = rk; pr[0].N = rk; pr[0].K = cs.K;
      pr[0].alpha = 1.0;
      C.gemm(pr);
      symmetrize(Dk, rk, C.st);
      ++C.launches;
    }
    cudaEventRecord(e1.e, C.st);
    // ---- diagonal tile: a = A_kk - D_k (+ compensation) (+ shift) -------------
    bool comp = opts.schur && k > 0 && cs.K > 0;
    double comp_time = 0;
    if (comp) {
      schur_compensation_device(C, Dk, rk, cfg.eps, tile_seed(cfg.seed, 0x5c4ULL, k, 0), corr,
                                frob, rank_hint);
      cudaEventRecord(e2.e, C.st);
    }
    diag_combine(diagk, cs.K > 0 ? Dk : nullptr, comp ? corr : nullptr, opts.shift, akk, rk, C.st);
    ++C.launches;
    if (!ldl) {
      dcopy(akk, a0, (long long)rk * rk, C.st);
      bool ok = potrf_device(C, akk, rk);
      if (!ok) {
        dcopy(a0, akk, (long long)rk * rk, C.st);
        modified_cholesky_device(C, akk, rk);
        S.modified_diagonals++;
      }
      dcopy(akk, diagk, (long long)rk * rk, C.st);
      min_diag_sq(diagk, rk, piv + k, C.st);
      C.launches += 3;
    } else {
      double* dk = F->D.d + (size_t)k * b;
      double* ek = F->D.e + (size_t)k * b;
      uint8_t* sk = F->D.s2 + (size_t)k * b;
      int* pk = F->D.perm + (size_t)k * b;
      sytrf_bk(akk, rk, dk, ek, sk, pk, info, C.st);
      first_singular_kernel<<<1, 1, 0, C.st>>>(dk, ek, sk, rk, info + 1);
      int* h = C.pinned_ints(1);
      TLRG_CUDA(cudaMemcpyAsync(h, info + 1, sizeof(int), cudaMemcpyDeviceToHost, C.st));
      C.sync();
      if (h[0] >= 0) numeric_error("tlr_ldlt: singular D block in column", k);
      dcopy(akk, diagk, (long long)rk * rk, C.st);
      min_block_pivot(dk, ek, sk, rk, piv + k, C.st);
      C.launches += 4;
    }
    cudaEventRecord(e3.e, C.st);
    if (comp) {
      double* h = C.pinned_dbl(1);
      TLRG_CUDA(cudaMemcpyAsync(h, frob, sizeof(double), cudaMemcpyDeviceToHost, C.st));
      C.sync();
      S.compensation_frob += std::sqrt(h[0]);
      comp_time = elapsed(e1, e2);
    }
    C.sync();
    S.t_dense += elapsed(e0, e1);
    S.t_misc += elapsed(e1, e3);
    S.t_compensation += comp_time;
    // ---- ARA over the column -------------------------------------------------
    ColumnStats cst;
    std::vector<TileResult> res = column_ara(C, M, k, cs, cfg, *store, cst, &prep);
    S.t_sampling += cst.t_sampling;
    S.t_orthog += cst.t_orthog;
    S.t_projection += cst.t_projection;
    S.t_recompress += cst.t_recompress;
    S.flops_ref += cst.flops_ref;
    // ---- TRSM of the new panel and overwrite ----------------------------------
    cudaEventRecord(e4.e, C.st);
    double* Vp = nullptr;
    long long ncols = 0;
    for (auto& r : res) {
      if (r.rank > 0 && !Vp) Vp = r.V;
      ncols += r.rank;
      S.ara_rounds[k] += r.rounds;
    }
    S.tile_rounds_resident += S.ara_rounds[k];
    if (ncols > 0) {
      if (ldl) {
        TLRG_CUDA(cudaMemsetAsync(info, 0xff, sizeof(int), C.st));
        trsm_panel(diagk, rk, Vp, ncols, F->D.perm + (size_t)k * b, F->D.d + (size_t)k * b,
                   F->D.e + (size_t)k * b, F->D.s2 + (size_t)k * b, info, C.st);
      } else {
        trsm_panel(diagk, rk, Vp, ncols, nullptr, nullptr, nullptr, nullptr, info, C.st);
      }
      ++C.launches;
    }
    for (auto& r : res) {
      long long t = M.t(r.i, k);
      M.rank[t] = r.rank;
      M.U[t] = r.U;
      M.V[t] = r.V;
    }
    cudaEventRecord(e5.e, C.st);
    C.sync();
    S.t_misc += elapsed(e4, e5);
  }
  cudaEventRecord(d1.e, C.st);
  C.sync();
  S.t_device = elapsed(d0, d1);
  S.kt_gemm_seconds = C.kt_seconds;
  S.kt_gemm_flops = C.kt_flops;
  S.kt_gemm_launches = C.kt_launches;
  C.ktiming = false;
  TLRG_CUDA(cudaMemcpy(S.pivot_trace.data(), piv, sizeof(double) * nb, cudaMemcpyDeviceToHost));
  S.wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_wall0).count();
  S.flops_exec = C.flops - flops0;
  S.launches = C.launches - launches0;
  // dense-phase reference flops: sum_{j<k} (4m k_kj^2 + 2 m^2 k_kj)
  for (int k = 0; k < nb; ++k)
    for (int j = 0; j < k; ++j) {
      double r = M.rank[M.t(k, j)];
      S.flops_ref += 4.0 * b * r * r + 2.0 * (double)b * b * r;
    }
  return F;
}

Factor::~Factor() {
  if (D.d) cudaFree(D.d);
  if (D.e) cudaFree(D.e);
  if (D.s2) cudaFree(D.s2);
  if (D.perm) cudaFree(D.perm);
}

}  // namespace tlrg
