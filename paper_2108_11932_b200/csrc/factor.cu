// Left-looking TLR Cholesky / LDL^T driver on the device (factor.cpp:115-306).
// Columns are sequential; inside a column everything is batched over tiles:
//   Gram + H (dense phase) -> SYRK D_k -> Schur compensation -> POTRF / BK LDL
//   -> dynamic-batched ARA -> panel TRSM (+perm, D^{-1}) -> pointer update.
#include <algorithm>
#include <cstdio>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "core.h"

namespace tlrg {
std::chrono::steady_clock::time_point g_fused_launch, g_ara_waited,
    g_ara_recomp;  // COLPROF probes (set in ara.cu)


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

// ---- pivoted Cholesky (Alg. 8, factor.cpp:140-209) --------------------------
// ||A_ii - D_i||_F for candidate tiles i = k0 + blockIdx.x (the running
// accumulators D_i of the reference's PivotAccumulators), fixed-order reduction
__global__ void pivot_frob_kernel(const double* diag, const double* dacc, int b, int k0,
                                  double* cand) {
  const int i = k0 + blockIdx.x;
  const long long bb = (long long)b * b, o = (long long)i * bb;
  double s = 0.0;
  for (long long t = threadIdx.x; t < bb; t += blockDim.x) {
    const double v = diag[o + t] - dacc[o + t];
    s += v * v;
  }
  __shared__ double red[32];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    cand[blockIdx.x] = sqrt(t);
  }
}

// power_norm_estimate (dense_kernels.cpp:544-564) of A_ii - D_i, one CTA per
// candidate; g: b start gaussians per candidate (tlr::Rng(tile_seed(seed, 0x9047, k, i)))
__global__ void pivot_power_kernel(const double* diag, const double* dacc, int b, int k0,
                                   const double* g, int iters, double* cand) {
  extern __shared__ double sm[];
  double* v = sm;
  double* w = sm + b;
  __shared__ double red[32];
  const int i = k0 + blockIdx.x;
  const long long o = (long long)i * b * b;
  const int nw_ = blockDim.x >> 5, lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  auto block_sum = [&](double x) {
    x = warp_sum(x);
    __syncthreads();
    if (lane == 0) red[wp] = x;
    __syncthreads();
    double t = 0.0;
    for (int q = 0; q < nw_; ++q) t += red[q];
    return t;
  };
  double ss = 0.0;
  for (int r = threadIdx.x; r < b; r += blockDim.x) {
    v[r] = g[(long long)blockIdx.x * b + r];
    ss += v[r] * v[r];
  }
  double nv = sqrt(block_sum(ss));
  if (nv == 0.0) {
    if (threadIdx.x == 0) v[0] = 1.0;
    nv = 1.0;
  }
  __syncthreads();
  for (int r = threadIdx.x; r < b; r += blockDim.x) v[r] /= nv;
  __syncthreads();
  double lambda = 0.0;
  for (int t = 0; t < iters; ++t) {
    for (int r = threadIdx.x; r < b; r += blockDim.x) {
      double a = 0.0;
      for (int c = 0; c < b; ++c) a += (diag[o + r + (long long)c * b] - dacc[o + r + (long long)c * b]) * v[c];
      w[r] = a;
    }
    __syncthreads();
    double n2 = 0.0, d = 0.0;
    for (int r = threadIdx.x; r < b; r += blockDim.x) {
      n2 += w[r] * w[r];
      d += v[r] * w[r];
    }
    const double nw = sqrt(block_sum(n2));
    lambda = fabs(block_sum(d));
    if (nw == 0.0) {
      lambda = 0.0;
      break;
    }
    for (int r = threadIdx.x; r < b; r += blockDim.x) v[r] = w[r] / nw;
    __syncthreads();
  }
  if (threadIdx.x == 0) cand[blockIdx.x] = lambda;
}

__global__ void swap_kernel(double* a, double* b, long long n) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const double x = a[t];
    a[t] = b[t];
    b[t] = x;
  }
}
void dswap(double* a, double* b, long long n, cudaStream_t st) {
  int blocks = (int)std::min<long long>((n + 255) / 256, 148 * 8);
  swap_kernel<<<blocks, 256, 0, st>>>(a, b, n);
  TLRG_CUDA(cudaGetLastError());
}

__global__ void tile_perm_kernel(const double* in, double* out, const int* perm, int b, int nb,
                                 int inverse) {
  const long long n = (long long)nb * b;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(t / b), r = (int)(t % b);
    const long long src = (long long)perm[k] * b + r;
    if (inverse) out[src] = in[t];
    else out[t] = in[src];
  }
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
__global__ void identity_kernel(double* A, int n) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)n * n) return;
  A[t] = (t % n) == (t / n) ? 1.0 : 0.0;
}
void identity(double* A, int n, cudaStream_t st) {
  long long nn = (long long)n * n;
  identity_kernel<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(A, n);
  TLRG_CUDA(cudaGetLastError());
}
}  // namespace

void tile_perm_device(Ctx& C, const Factor& F, const double* in, double* out, bool inverse) {
  const Matrix& L = *F.L;
  const long long n = (long long)L.nb * L.b;
  int blocks = (int)std::min<long long>((n + 255) / 256, 148 * 8);
  tile_perm_kernel<<<blocks, 256, 0, C.st>>>(in, out, F.d_perm, L.b, L.nb, inverse ? 1 : 0);
  TLRG_CUDA(cudaGetLastError());
  ++C.launches;
}

// TlrMatrix::pivot_swap(k, p, k) (tlr_matrix.cpp:66-82) on the host tile tables
// (rank and U/V device pointers; uniform tiles, so U and V are interchangeable).
// The diagonal tiles themselves are swapped on the device by the caller.
void pivot_swap_tables(Matrix& M, int k, int p) {
  if (k == p) return;
  if (k > p) std::swap(k, p);
  if (M.rows(k) != M.rows(p)) config_error("pivot_swap: tiles of unequal size");
  auto sw = [&](long long a, long long c) {
    std::swap(M.rank[a], M.rank[c]);
    std::swap(M.U[a], M.U[c]);
    std::swap(M.V[a], M.V[c]);
  };
  for (int j = 0; j < k; ++j) sw(M.t(k, j), M.t(p, j));
  for (int m = k + 1; m < p; ++m) {
    const long long a = M.t(m, k), c = M.t(p, m);
    sw(a, c);  // new (m,k) = old A(p,m)^T, new (p,m) = old A(m,k)^T
    std::swap(M.U[a], M.V[a]);
    std::swap(M.U[c], M.V[c]);
  }
  for (int m = p + 1; m < M.nb; ++m) sw(M.t(m, k), M.t(m, p));
  const long long pk = M.t(p, k);
  std::swap(M.U[pk], M.V[pk]);  // new (p,k) = A(p,k)^T
}

void potrf_impl(double* A, int n, int* info, DescArena& desc, cudaStream_t st);

// X = L^{-1} for a lower-triangular n x n tile by recursive block inversion on
// the grouped DMMA GEMM:  inv([L11 0; L21 L22]) = [X11 0; -X22 L21 X11  X22].
// 32x32 diagonal blocks are inverted in one launch, then every merge level
// (pairs of blocks) is two batched GEMMs.  Off the critical path (diagonal
// stream); replaces a TRSM against the identity.
void trtri_device(Ctx& C, const double* L, int n, double* X) {
  TLRG_CUDA(cudaMemsetAsync(X, 0, sizeof(double) * n * n, C.st));
  std::vector<int> offs, lens;
  for (int o = 0; o < n; o += 32) {
    offs.push_back(o);
    lens.push_back(std::min(32, n - o));
  }
  trtri_base(L, n, X, C.push(offs), C.push(lens), (int)offs.size(), C.st);
  ++C.launches;
  double* T = C.buf<double>("trtri_T", (size_t)n * n / 2 + 64);
  while (offs.size() > 1) {
    std::vector<GemmProblem> p1, p2;
    std::vector<int> no, nl;
    size_t toff = 0;
    for (size_t b = 0; b + 1 < offs.size(); b += 2) {
      const int o = offs[b], l1 = lens[b], l2 = lens[b + 1];
      GemmProblem g{};
      // T = L21 X11   (l2 x l1)
      g.A = L + (o + l1) + (long long)o * n; g.lda = n;
      g.B = X + o + (long long)o * n; g.ldb = n;
      g.C = T + toff; g.ldc = l2;
      g.M = l2; g.N = l1; g.K = l1; g.alpha = 1.0;
      p1.push_back(g);
      // X21 = -X22 T
      GemmProblem h{};
      h.A = X + (o + l1) + (long long)(o + l1) * n; h.lda = n;
      h.B = T + toff; h.ldb = l2;
      h.C = X + (o + l1) + (long long)o * n; h.ldc = n;
      h.M = l2; h.N = l1; h.K = l2; h.alpha = -1.0;
      p2.push_back(h);
      toff += (size_t)l1 * l2;
      no.push_back(o);
      nl.push_back(l1 + l2);
    }
    if (offs.size() % 2) {
      no.push_back(offs.back());
      nl.push_back(lens.back());
    }
    C.gemm(p1);
    C.gemm(p2);
    offs.swap(no);
    lens.swap(nl);
  }
}

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
// SVD of Q^T D Q (one-sided Jacobi), keep sigma > eps.  The retained rank r is
// consumed on the device (GEMM K from *rank), so the whole step enqueues without
// a host round trip; the caller checks afterwards that at least 8 directions of
// slack remained (r <= p - 8) and re-runs with a wider sketch otherwise.
// sketch width cap: the p x p core's two-sided Jacobi keeps B and V in shared
// memory up to p = 112 (the one-sided fallback in global memory was ~10x slower
// at p = 160); wider eps-ranks go through the chunked spectrum split
constexpr int kSchurMaxWidth = 112;
int schur_comp_width(int n, int rank_hint) {
  int p = std::max(24, rank_hint + 16);
  p = ((p + 7) / 8) * 8;
  p = std::min(p, kSchurMaxWidth);
  return p > n ? n : p;
}
void schur_comp_enqueue(Ctx& C, const double* Dk, int n, double eps, uint64_t seed, int p,
                        int attempt, double* corr, double* frob, int* rank_out, int power) {
  double* Om = C.buf<double>("sc_Om", (size_t)n * p);
  double* Y = C.buf<double>("sc_Y", (size_t)n * p);
  double* Bm = C.buf<double>("sc_B", (size_t)p * p);
  double* Vm = C.buf<double>("sc_V", (size_t)p * p);
  double* work = C.buf<double>("sc_work", (size_t)2 * p * p);
  double* sig = C.buf<double>("sc_sig", (size_t)p);
  fill_gaussian_philox(Om, (long long)n * p, seed * 0x9E3779B97F4A7C15ULL + attempt, C.st);
  C.launches += 1;
  auto DtimesX = [&](const double* X, double* out) {
    std::vector<GemmProblem> pr(1);
    pr[0] = GemmProblem{};
    pr[0].A = Dk; pr[0].lda = n; pr[0].B = X; pr[0].ldb = n; pr[0].C = out; pr[0].ldc = n;
    pr[0].M = n; pr[0].N = p; pr[0].K = n; pr[0].alpha = 1.0;
    C.gemm(pr);
  };
  // orthonormal basis of the sketch by shifted Cholesky-QR (3 passes; GEMMs +
  // one tiny factor kernel each): X <- X R1^{-1} R2^{-1} R3^{-1}
  double* Gq = C.buf<double>("sc_G", (size_t)p * p);
  double* Ri = C.buf<double>("sc_Ri", (size_t)p * p);
  auto orth = [&](double* X) {
    for (int pass = 0; pass < 3; ++pass) {
      std::vector<GemmProblem> pr(1);
      pr[0] = GemmProblem{};
      pr[0].A = X; pr[0].lda = n; pr[0].transA = 1; pr[0].B = X; pr[0].ldb = n;
      pr[0].C = Gq; pr[0].ldc = p; pr[0].M = p; pr[0].N = p; pr[0].K = n; pr[0].alpha = 1.0;
      C.gemm(pr);
      cholqr_factor(Gq, p, n, pass == 0, Ri, C.st);  // Ri <- R (upper)
      cholqr_apply(X, n, p, Ri, C.st);               // X <- X R^{-1}
      C.launches += 2;
    }
  };
  DtimesX(Om, Y);
  orth(Y);
  for (int it = 0; it < power; ++it) {  // power iterations
    DtimesX(Y, Om);
    orth(Om);
    if (it + 1 < power) std::swap(Y, Om);
  }
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
  sv[0].A = Bm; sv[0].V = Vm; sv[0].sig = sig; sv[0].work = work; sv[0].rank_out = rank_out;
  sv[0].n = p; sv[0].cut = eps;
  sv[0].tol = 1e-14;  // off-diagonals below 1e-14 ||B||_F: ample for the eps-level split
  // symmetric PSD core: two-sided Jacobi (no dot products; 3 barriers a step)
  if (p <= kSchurMaxWidth) sym_jacobi(C.push(sv), 1, p, C.st);
  else jacobi_svd(C.push(sv), 1, p, C.st);
  ++C.launches;
  // R = D - (Q A_B)(Q V_B)^T restricted to the r = *rank_out retained directions
  double* Xl = C.buf<double>("sc_Xl", (size_t)n * p);
  double* Xr = C.buf<double>("sc_Xr", (size_t)n * p);
  double* Rm = C.buf<double>("sc_Rm", (size_t)n * n);
  double* fp = C.buf<double>("sc_fp", (size_t)n);
  TLRG_CUDA(cudaMemcpyAsync(Rm, Dk, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, C.st));
  {
    std::vector<GemmProblem> pr(2);
    pr[0] = GemmProblem{};
    pr[0].A = Om; pr[0].lda = n; pr[0].B = Bm; pr[0].ldb = p; pr[0].C = Xl; pr[0].ldc = n;
    pr[0].M = n; pr[0].N = p; pr[0].K = p; pr[0].alpha = 1.0;
    pr[1] = pr[0];
    pr[1].B = Vm; pr[1].C = Xr;
    C.gemm(pr);
    std::vector<GemmProblem> p2(1);
    p2[0] = GemmProblem{};
    p2[0].A = Xl; p2[0].lda = n; p2[0].B = Xr; p2[0].ldb = n; p2[0].transB = 1;
    p2[0].C = Rm; p2[0].ldc = n; p2[0].M = n; p2[0].N = n; p2[0].K = p; p2[0].Kp = rank_out;
    p2[0].alpha = -1.0; p2[0].beta = 1.0;
    C.gemm(p2);
  }
  rowsum_abs_residual(Rm, nullptr, nullptr, n, 0, corr, fp, C.st);
  block_sum_device(fp, n, frob, C.st);  // ||R||_F^2 from the per-row sums of squares
  C.launches += 2;
}

// synchronous form: widen the sketch until the slack test holds; when the
// eps-rank of D exceeds what one sketch can hold (kSchurMaxWidth - 8; measured
// 82-278 at m = 1024, eps = 1e-3), split the spectrum in chunks: the top p - 32
// Ritz pairs of each full-width sketch (32 directions of oversampling plus two
// power steps behind them) are deflated from a working copy of D, and the next
// sketch runs on the deflated matrix, until one has slack.  R = D - kept parts
// is then the last chunk's residual.
void schur_compensation_device(Ctx& C, const double* Dk, int n, double eps, uint64_t seed,
                               double* corr, double* frob, int& rank_hint) {
  const int cap = std::min(n, kSchurMaxWidth);
  int p = schur_comp_width(n, rank_hint);
  int* rk = C.buf<int>("sc_rank", 1);
  const double* Dw = Dk;
  double* Dwork = nullptr;
  int deflated = 0;
  for (int attempt = 0;; ++attempt) {
    // a full-width sketch (the chunked split deflates its Ritz pairs) takes a
    // second power step: the deflated pairs' errors add up in rowsum |R|
    schur_comp_enqueue(C, Dw, n, eps, seed, p, attempt, corr, frob, rk, p >= cap ? 2 : 1);
    int* h = C.pinned_ints(1);
    TLRG_CUDA(cudaMemcpyAsync(h, rk, sizeof(int), cudaMemcpyDeviceToHost, C.st));
    C.wait();
    if (h[0] <= p - 8 || p >= n) {
      rank_hint = deflated + h[0];
      return;
    }
    if (p < cap) {
      p = std::min(cap, 2 * p);
      continue;
    }
    // full-width sketch without slack: deflate its top p - 32 Ritz pairs
    if (!Dwork) {
      Dwork = C.buf<double>("sc_Dwork", (size_t)n * n);
      dcopy(Dk, Dwork, (long long)n * n, C.st);
      Dw = Dwork;
    }
    const int kd = p - 32;  // 32 directions of oversampling behind the deflated pairs
    std::vector<GemmProblem> pr(1);
    pr[0] = GemmProblem{};
    pr[0].A = C.buf<double>("sc_Xl", (size_t)n * p); pr[0].lda = n;
    pr[0].B = C.buf<double>("sc_Xr", (size_t)n * p); pr[0].ldb = n; pr[0].transB = 1;
    pr[0].C = Dwork; pr[0].ldc = n; pr[0].M = n; pr[0].N = n; pr[0].K = kd;
    pr[0].alpha = -1.0; pr[0].beta = 1.0;
    C.gemm(pr);
    symmetrize(Dwork, n, C.st);
    ++C.launches;
    deflated += kd;
    if (deflated >= n) numeric_error("schur_compensation: spectrum split did not converge", -1);
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
  const bool pivoted = mode == 2;
  if (ldl) opts.schur = false;  // factor.cpp:304
  if (pivoted && A->n % A->b != 0)
    config_error("pivoted factorization requires uniform tiles");
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
  store->st = C.st_main;
  store->owner = &C;
  M.stores.push_back(store);
  {
    // the factor's panels come from cached chunks: reserve about A's low-rank
    // footprint (+25 %) now instead of growing the pool inside the column loop
    size_t lr = 0;
    for (int i = 1; i < nb; ++i)
      for (int j = 0; j < i; ++j) lr += (size_t)(M.rows(i) + M.rows(j)) * M.rank[M.t(i, j)];
    const auto hr0 = std::chrono::steady_clock::now();
    chunk_cache_reserve(&C, lr + lr / 4, C.st_main);
    if (std::getenv("TLRG_COLPROF"))
      std::fprintf(stderr, "factor: reserve %.3f ms host\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - hr0)
                       .count());
  }
  // device mirror of the tile tables (rank, U pointer per lower tile), kept
  // current column by column: the ARA's H_i block list is derived on the device
  const long long ntri = (long long)nb * (nb - 1) / 2;
  int* d_rank = nullptr;
  const double** d_U = nullptr;
  {
    const char* hh = std::getenv("TLRG_HOST_H");
    if (ntri > 0 && !(hh && hh[0] == '1')) {
      d_rank = C.buf<int>("tri_rank", (size_t)ntri);
      d_U = reinterpret_cast<const double**>(C.buf<uintptr_t>("tri_U", (size_t)ntri));
      TLRG_CUDA(cudaMemcpyAsync(d_rank, M.rank.data(), sizeof(int) * ntri, cudaMemcpyHostToDevice,
                                C.st));
      TLRG_CUDA(cudaMemcpyAsync(d_U, M.U.data(), sizeof(double*) * ntri, cudaMemcpyHostToDevice,
                                C.st));
    }
  }
  double* Dk = C.buf<double>("Dk", (size_t)b * b);
  double* a0 = C.buf<double>("akk0", (size_t)b * b);
  double* aorig = C.buf<double>("akk_orig", (size_t)b * b);
  double* Xinv = C.buf<double>("Linv", (size_t)b * b);
  double* corr = C.buf<double>("corr", (size_t)b);
  double* frob = C.buf<double>("cfrob", 1);
  double* piv = C.buf<double>("pivot", (size_t)nb);
  // pivoted mode (Alg. 8): running diagonal accumulators D_i = sum_{j<k} L_ij L_ij^T
  // for the not-yet-eliminated tiles, candidate norms, start vectors
  double* dacc = nullptr;
  double* cand = nullptr;
  if (pivoted) {
    F->perm.resize(nb);
    for (int i = 0; i < nb; ++i) F->perm[i] = i;
    dacc = C.buf<double>("piv_dacc", (size_t)nb * b * b);
    TLRG_CUDA(cudaMemsetAsync(dacc, 0, sizeof(double) * nb * b * b, C.st));
    cand = C.buf<double>("piv_cand", (size_t)nb);
  }
  int* info = C.buf<int>("finfo", 4);  // [0] potrf, [1] first singular D block, [2] comp rank, [3] trsm
  int rank_hint = 0;
  Ev e0, e1, e4, e5, de0, de1, de2, de3, ejoin, eprev;
  double gap_sum = 0, gap_max = 0, gap_first = 0;
  int gap_arg = -1;
  StreamPrep prep;

  const char* dfe = std::getenv("TLRG_DIAG_FIRST");
  const bool diag_first = dfe && dfe[0] == '1';
  const char* cpe = std::getenv("TLRG_COLPROF");
  const bool colprof = cpe && cpe[0] == '1';
  for (int k = 0; k < nb; ++k) {
    const auto t_col0 = std::chrono::steady_clock::now();
    auto hrel = [&] {
      return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_col0)
          .count();
    };
    double h_setup = 0, h_diag = 0, h_ara = 0;
    const int rk = M.rows(k);
    double* diagk = M.diag + (size_t)k * b * b;
    // ---- pivoted: fold column k-1 into the accumulators, pick the tile with the
    //      largest updated diagonal norm, swap it into position k (factor.cpp:156-209)
    if (pivoted) {
      Ev pv0, pv1;
      const auto hp0 = std::chrono::steady_clock::now();
      cudaEventRecord(pv0.e, C.st);
      if (k > 0) {
        std::vector<GemmProblem> g1, g2, g3;
        long long go = 0, to = 0;
        std::vector<long long> gofs, tofs;
        for (int i = k; i < nb; ++i) {
          const int r = M.rank[M.t(i, k - 1)];
          gofs.push_back(go);
          tofs.push_back(to);
          go += (long long)r * r;
          to += (long long)b * r;
        }
        double* gb = C.buf<double>("piv_g", (size_t)std::max(go, 1LL));
        double* tb = C.buf<double>("piv_t", (size_t)std::max(to, 1LL));
        for (int i = k; i < nb; ++i) {
          const long long t = M.t(i, k - 1);
          const int r = M.rank[t];
          if (!r) continue;
          double* g = gb + gofs[i - k];
          double* tt = tb + tofs[i - k];
          GemmProblem a{};  // g = V^T V   (expand_update, factor.cpp:18-30)
          a.A = M.V[t]; a.lda = b; a.transA = 1; a.B = M.V[t]; a.ldb = b;
          a.C = g; a.ldc = r; a.M = r; a.N = r; a.K = b; a.alpha = 1.0;
          g1.push_back(a);
          GemmProblem c{};  // t = U g
          c.A = M.U[t]; c.lda = b; c.B = g; c.ldb = r;
          c.C = tt; c.ldc = b; c.M = b; c.N = r; c.K = r; c.alpha = 1.0;
          g2.push_back(c);
          GemmProblem d{};  // D_i += t U^T
          d.A = tt; d.lda = b; d.B = M.U[t]; d.ldb = b; d.transB = 1;
          d.C = dacc + (size_t)i * b * b; d.ldc = b; d.M = b; d.N = b; d.K = r;
          d.alpha = 1.0; d.beta = 1.0;
          g3.push_back(d);
        }
        if (!g1.empty()) {
          C.gemm(g1);
          C.gemm(g2);
          C.gemm(g3);
        }
      }
      cudaEventRecord(pv1.e, C.st);
      const int nc = nb - k;
      if (opts.pivot_norm == 0) {
        pivot_frob_kernel<<<nc, 256, 0, C.st>>>(M.diag, dacc, b, k, cand);
      } else {
        RngState* rs = C.buf<RngState>("piv_rng", (size_t)nc);
        double* gv = C.buf<double>("piv_gv", (size_t)nc * b);
        std::vector<uint64_t> seeds(nc);
        for (int i = k; i < nb; ++i) seeds[i - k] = tile_seed(cfg.seed, 0x9047ULL, k, i);
        rng_seed(rs, C.push(seeds), nc, C.st);
        rng_draw(rs, nullptr, nc, gv, b, b, C.st);
        pivot_power_kernel<<<nc, 256, 2 * b * sizeof(double), C.st>>>(
            M.diag, dacc, b, k, gv, opts.pivot_power_iters, cand);
        C.launches += 2;
      }
      TLRG_CUDA(cudaGetLastError());
      ++C.launches;
      double* hc = C.pinned_dbl((size_t)nc);
      TLRG_CUDA(cudaMemcpyAsync(hc, cand, sizeof(double) * nc, cudaMemcpyDeviceToHost, C.st));
      C.wait();
      int p = k;
      double best = -1.0;
      for (int i = k; i < nb; ++i)
        if (hc[i - k] > best) {
          best = hc[i - k];
          p = i;
        }
      S.t_dense += elapsed(pv0, pv1);
      S.t_pivot_select += std::chrono::duration<double>(std::chrono::steady_clock::now() - hp0)
                              .count() - elapsed(pv0, pv1);
      if (p != k) {
        pivot_swap_tables(M, k, p);
        dswap(M.diag + (size_t)k * b * b, M.diag + (size_t)p * b * b, (long long)b * b, C.st);
        dswap(dacc + (size_t)k * b * b, dacc + (size_t)p * b * b, (long long)b * b, C.st);
        std::swap(F->perm[k], F->perm[p]);
        if (d_rank) {
          TLRG_CUDA(cudaMemcpyAsync(d_rank, M.rank.data(), sizeof(int) * ntri,
                                    cudaMemcpyHostToDevice, C.st));
          TLRG_CUDA(cudaMemcpyAsync(d_U, M.U.data(), sizeof(double*) * ntri,
                                    cudaMemcpyHostToDevice, C.st));
        }
        C.launches += 2;
      }
      // D_k for the diagonal path: the accumulator, symmetrized (factor.cpp:207-208)
      dcopy(dacc + (size_t)k * b * b, Dk, (long long)b * b, C.st);
      symmetrize(Dk, rk, C.st);
      C.launches += 2;
    }
    // ---- gaussian streams of this column's ARA, generated on the side stream
    //      while the column setup and the diagonal path run
    column_prepare(C, M, k, cfg, prep);
    // ---- column setup: row-k concatenation and Gram blocks (main stream) ------
    cudaEventRecord(e0.e, C.st);
    ColumnSetup cs;
    column_setup(C, M, k, F->D, cs);
    cs.d_rank = d_rank;
    cs.d_U = d_U;
    cudaEventRecord(e1.e, C.st);
    h_setup = hrel();
    const bool comp = opts.schur && k > 0 && cs.K > 0;
    int p_comp = comp ? schur_comp_width(rk, rank_hint) : 0;
    const bool comp_chunked =
        comp && p_comp >= std::min(rk, kSchurMaxWidth) && p_comp < rk && rank_hint > p_comp - 8;

    // ---- diagonal path on its own stream: it needs only row k of L, so it runs
    //      concurrently with the column's ARA (which needs L_kk only for the
    //      final TRSM).  D_k, compensation, a = A_kk - D_k (+comp) (+shift),
    //      POTRF / Bunch-Kaufman, and the panel operator X = L^{-1}
    //      (Chol) or D^{-1} L^{-1} P (LDL), so the TRSM becomes one GEMM.
    auto diag_tail = [&]() {
      diag_combine(aorig, cs.K > 0 ? Dk : nullptr, comp ? corr : nullptr, opts.shift, a0, rk,
                   C.st);
      dcopy(a0, diagk, (long long)rk * rk, C.st);
      if (!ldl) {
        potrf_impl(diagk, rk, info, C.desc, C.st);
        C.launches += 4;
      } else {
        double* dk = F->D.d + (size_t)k * b;
        double* ek = F->D.e + (size_t)k * b;
        uint8_t* sk = F->D.s2 + (size_t)k * b;
        int* pk = F->D.perm + (size_t)k * b;
        sytrf_bk(diagk, rk, dk, ek, sk, pk, info + 3, C.st);
        first_singular_kernel<<<1, 1, 0, C.st>>>(dk, ek, sk, rk, info + 1);
        C.launches += 4;
      }
    };
    auto diag_inverse = [&]() {
      if (ldl) identity(Xinv, rk, C.st);
      if (!ldl) {
        trtri_device(C, diagk, rk, Xinv);
        min_diag_sq(diagk, rk, piv + k, C.st);
      } else {
        size_t o = (size_t)k * b;
        trsm_panel(diagk, rk, Xinv, rk, F->D.perm + o, F->D.d + o, F->D.e + o, F->D.s2 + o,
                   info + 3, C.st,
                   C.buf<double>("trsm_W", (size_t)rk * rk));
        min_block_pivot(F->D.d + o, F->D.e + o, F->D.s2 + o, rk, piv + k, C.st);
      }
      C.launches += 3;
    };
    bool diag_enqueued = false;
    auto enqueue_diag = [&]() {
      if (diag_enqueued) return;
      diag_enqueued = true;
      TLRG_CUDA(cudaStreamWaitEvent(C.sd, e1.e, 0));
      {
        StreamScope on_diag(C, C.sd);
        // grow the H_k buffer before the phase timer starts: a growth frees
        // the old buffer (cudaFree waits for the whole device, i.e. the
        // column's ARA already in flight) and would land in t_dense
        double* Hk = cs.K > 0 && !pivoted ? C.buf<double>("Hk", (size_t)b * cs.K) : nullptr;
        cudaEventRecord(de0.e, C.st);
        // keep A_kk: the tile is factored in place and a retry re-reads it
        dcopy(diagk, aorig, (long long)rk * rk, C.st);
        if (cs.K > 0 && !pivoted) {
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
        cudaEventRecord(de1.e, C.st);
        if (comp_chunked) {
          // the previous column's eps-rank already exceeded one sketch: run the
          // chunked spectrum split here, on the diagonal stream while the ARA
          // runs, instead of a first sketch that the join would discard and
          // redo on the critical path (same seed and attempts: same result)
          schur_compensation_device(C, Dk, rk, cfg.eps, tile_seed(cfg.seed, 0x5c4ULL, k, 0), corr,
                                    frob, rank_hint);
        } else if (comp) {
          schur_comp_enqueue(C, Dk, rk, cfg.eps, tile_seed(cfg.seed, 0x5c4ULL, k, 0), p_comp, 0,
                             corr, frob, info + 2, p_comp >= std::min(rk, kSchurMaxWidth) ? 2 : 1);
        }
        cudaEventRecord(de2.e, C.st);
        diag_tail();
        diag_inverse();
        cudaEventRecord(de3.e, C.st);
      }
      h_diag = hrel();
    };
    // the column's ARA is the longer branch in most columns: launch it first and
    // enqueue the diagonal path while it runs (TLRG_DIAG_FIRST=1: old order)
    if (diag_first) enqueue_diag();
    // ---- ARA over the column (main stream) -------------------------------------
    ColumnStats cst;
    const int prank = C.comm ? C.comm->rank : 0, pworld = C.comm ? C.comm->world : 1;
    std::vector<TileResult> res =
        column_ara(C, M, k, cs, cfg, *store, cst, &prep, prank, pworld, enqueue_diag);
    enqueue_diag();  // no-op unless the column had no ARA work
    h_ara = hrel();
    S.t_sampling += cst.t_sampling;
    S.t_orthog += cst.t_orthog;
    S.flops_ref += cst.flops_ref;
    S.t_fused += cst.t_fused;
    S.flops_fused += cst.flops_fused;
    S.fused_launches += cst.fused_launches;
    // ---- join: diagonal status (one small read, after the TRSM is enqueued) ----
    TLRG_CUDA(cudaStreamWaitEvent(C.st, de3.e, 0));
    int* hs = C.pinned_ints(4);
    double* hf = C.pinned_dbl(1);
    TLRG_CUDA(cudaMemcpyAsync(hs, info, sizeof(int) * 4, cudaMemcpyDeviceToHost, C.st));
    if (comp) TLRG_CUDA(cudaMemcpyAsync(hf, frob, sizeof(double), cudaMemcpyDeviceToHost, C.st));
    // ---- TRSM of the new panel (one GEMM with the precomputed operator),
    //      enqueued before the status read: the rare retry / fallback below
    //      recomputes the operator and re-runs the GEMM from the saved copy Bs
    cudaEventRecord(e4.e, C.st);
    double* Vp = nullptr;
    double* Up0 = nullptr;
    double* Bs = nullptr;
    long long ncols = 0;
    for (auto& r : res) {
      if (r.rank > 0 && !Vp) {
        Vp = r.V;
        Up0 = r.U;
      }
      ncols += r.rank;  // this rank's tiles only (the others are still empty)
      S.ara_rounds[k] += r.rounds;
    }
    S.tile_rounds_resident += S.ara_rounds[k];
    auto trsm_gemm = [&]() {
      std::vector<GemmProblem> pr(1);
      pr[0] = GemmProblem{};
      pr[0].A = Xinv; pr[0].lda = rk; pr[0].B = Bs; pr[0].ldb = rk;
      pr[0].C = Vp; pr[0].ldc = rk; pr[0].M = rk; pr[0].N = (int)ncols; pr[0].K = rk;
      pr[0].alpha = 1.0;
      C.gemm(pr);
      ++C.launches;
    };
    if (ncols > 0) {
      Bs = C.buf<double>("trsm_B", (size_t)rk * ncols);
      TLRG_CUDA(cudaMemcpyAsync(Bs, Vp, sizeof(double) * rk * ncols, cudaMemcpyDeviceToDevice,
                                C.st));
      trsm_gemm();
    }
    bool redo_trsm = false;
    C.wait();
    int st_potrf = hs[0], st_sing = hs[1], st_rank = hs[2];
    if (comp && !comp_chunked && st_rank > p_comp - 8 && p_comp < rk) {
      // sketch too narrow for this column's spectrum: redo with a wider one,
      // or (eps-rank above one sketch) with the chunked spectrum split
      rank_hint = std::max(rank_hint, 2 * p_comp);
      schur_compensation_device(C, Dk, rk, cfg.eps, tile_seed(cfg.seed, 0x5c4ULL, k, 0), corr,
                                frob, rank_hint);
      diag_tail();
      TLRG_CUDA(cudaMemcpyAsync(hs, info, sizeof(int) * 4, cudaMemcpyDeviceToHost, C.st));
      TLRG_CUDA(cudaMemcpyAsync(hf, frob, sizeof(double), cudaMemcpyDeviceToHost, C.st));
      C.wait();
      st_potrf = hs[0];
      st_sing = hs[1];
      diag_inverse();
      redo_trsm = true;
    } else if (comp && !comp_chunked) {
      rank_hint = st_rank;
    }
    if (comp) S.compensation_frob += std::sqrt(hf[0]);
    if (ldl && st_sing >= 0) numeric_error("tlr_ldlt: singular D block in column", k);
    if (!ldl && st_potrf >= 0) {
      // modified Cholesky fallback (dense_kernels.cpp:283-309), rare
      dcopy(a0, diagk, (long long)rk * rk, C.st);
      modified_cholesky_device(C, diagk, rk);
      S.modified_diagonals++;
      diag_inverse();
      redo_trsm = true;
    }
    if (redo_trsm && ncols > 0) trsm_gemm();
    {
      float f = 0;
      // column setup = the Gram blocks G_ij of the re-associated sampling chain
      // (the j-sum the reference evaluates inside every sampling round)
      cudaEventElapsedTime(&f, e0.e, e1.e);
      S.t_sampling += f * 1e-3;
      cudaEventElapsedTime(&f, de0.e, de1.e);
      S.t_dense += f * 1e-3;
      cudaEventElapsedTime(&f, de1.e, de2.e);
      S.t_compensation += f * 1e-3;
      S.t_misc += f * 1e-3;
      cudaEventElapsedTime(&f, de2.e, de3.e);
      S.t_misc += f * 1e-3;
    }
    if (pworld > 1) exchange_column(C, *C.comm, M, k, column_queue(M, k), res, Up0, *store);
    for (auto& r : res) {
      long long t = M.t(r.i, k);
      M.rank[t] = r.rank;
      M.U[t] = r.U;
      M.V[t] = r.V;
    }
    if (d_rank && !res.empty()) {
      std::vector<long long> ut;
      std::vector<int> ur;
      std::vector<const double*> uu;
      for (auto& r : res) {
        ut.push_back(M.t(r.i, k));
        ur.push_back(r.rank);
        uu.push_back(r.U);
      }
      tri_update(C.push(ut), C.push(ur), C.push(uu), (int)res.size(), d_rank, d_U, C.st);
      ++C.launches;
    }
    cudaEventRecord(e5.e, C.st);
    C.sync();
    column_stats_resolve(cst);
    S.t_projection += cst.t_projection;
    S.t_recompress += cst.t_recompress;
    S.t_misc += elapsed(e4, e5);
    {
      // device time between columns (host work between e5 of k-1 and e0 of k)
      const double g = k == 0 ? elapsed(d0, e0) : elapsed(eprev, e0);
      if (k == 0) gap_first = g;
      else gap_sum += g;
      if (k > 0 && g > gap_max) {
        gap_max = g;
        gap_arg = k;
      }
      cudaEventRecord(eprev.e, C.st);
    }
    if (colprof) {
      auto ms = [](Ev& a, Ev& b) {
        float f = 0;
        cudaEventElapsedTime(&f, a.e, b.e);
        return f;
      };
      auto wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                               t_col0).count();
      std::fprintf(stderr,
                   "col %d T=%zu K=%d | setup %.3f diag %.3f (syrk %.3f comp %.3f fact %.3f) | "
                   "ara %.3f proj %.3f recomp %.3f | join->end %.3f | dev %.3f host %.3f ms | "
                   "host marks: setup %.3f diag %.3f fused-launch %.3f waited %.3f recomp-done %.3f "
                   "ara-ret %.3f\n",
                   k, res.size(), cs.K, ms(e0, e1), ms(de0, de3), ms(de0, de1), ms(de1, de2),
                   ms(de2, de3), cst.t_sampling * 1e3, cst.t_projection * 1e3,
                   cst.t_recompress * 1e3, ms(e4, e5), ms(e0, e5), wall_ms, h_setup, h_diag,
                   std::chrono::duration<double, std::milli>(g_fused_launch - t_col0).count(),
                   std::chrono::duration<double, std::milli>(g_ara_waited - t_col0).count(),
                   std::chrono::duration<double, std::milli>(g_ara_recomp - t_col0).count(),
                   h_ara);
    }
  }
  cudaEventRecord(d1.e, C.st);
  C.sync();
  S.t_device = elapsed(d0, d1);
  if (colprof)
    std::fprintf(stderr, "factor: start->col0 %.3f ms, between columns %.3f ms (max %.3f at %d), "
                 "last->end %.3f ms, total %.3f ms\n", gap_first * 1e3, gap_sum * 1e3,
                 gap_max * 1e3, gap_arg, elapsed(eprev, d1) * 1e3, S.t_device * 1e3);
  S.kt_gemm_seconds = C.kt_seconds;
  S.kt_gemm_flops = C.kt_flops;
  S.kt_gemm_launches = C.kt_launches;
  C.ktiming = false;
  TLRG_CUDA(cudaMemcpy(S.pivot_trace.data(), piv, sizeof(double) * nb, cudaMemcpyDeviceToHost));
  if (pivoted) {
    TLRG_CUDA(cudaMalloc(&F->d_perm, sizeof(int) * nb));
    TLRG_CUDA(cudaMemcpy(F->d_perm, F->perm.data(), sizeof(int) * nb, cudaMemcpyHostToDevice));
  }
  S.wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_wall0).count();
  S.flops_exec = C.flops - flops0 + S.flops_fused;
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
  if (d_perm) cudaFree(d_perm);
  if (D.d) cudaFree(D.d);
  if (D.e) cudaFree(D.e);
  if (D.s2) cudaFree(D.s2);
  if (D.perm) cudaFree(D.perm);
}

}  // namespace tlrg
