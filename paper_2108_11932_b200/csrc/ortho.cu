// ARA device kernels: per-tile Gaussian draws, the reference's two-sweep
// block Gram-Schmidt with column-wise MGS2 and random replacement of deficient
// columns (dense_kernels.cpp:331-420), the adaptive absorb/convergence state
// machine (ara.cpp:155-195), small one-sided Jacobi SVDs for recompression
// (ara.cpp:201-211), block-diagonal products and gathers.
#include <cfloat>

#include "kernels.h"

namespace tlrg {

// --------------------------------------------------------------- ABSORB ---
__global__ void __launch_bounds__(128) ara_absorb_kernel(AbsorbTask* tasks) {
  AbsorbTask& T = tasks[blockIdx.x];
  __shared__ int keep[256];
  __shared__ int nkeep;
  if (threadIdx.x == 0) {
    int q = *T.qcols;
    *T.rounds += 1;
    // push this round's post-deflation norms through the window (ara.cpp:174-177)
    int cnt = *T.recent_count, pos = *T.recent_pos;
    for (int j = 0; j < T.bs; ++j) {
      T.recent[pos] = T.col_norms[j];
      pos = (pos + 1) % T.window;
      if (cnt < T.window) ++cnt;
    }
    *T.recent_count = cnt;
    *T.recent_pos = pos;
    // keep filter (ara.cpp:179-182)
    int room = T.cap - q, n = 0;
    for (int j = 0; j < T.bs && n < room; ++j)
      if (T.new_mass[j] * T.eta > T.eps) keep[n++] = j;
    nkeep = n;
    double e = 0.0;
    for (int t = 0; t < cnt; ++t) e = fmax(e, T.recent[t]);
    int conv = e * T.eta <= T.eps;
    *T.converged = conv;
    *T.qcols = q + n;
    *T.done = conv || (q + n) >= T.cap;
  }
  __syncthreads();
  int q0 = *T.qcols - nkeep;
  for (long long e = threadIdx.x; e < (long long)nkeep * T.rows; e += blockDim.x) {
    int c = (int)(e / T.rows), r = (int)(e % T.rows);
    T.Q[(long long)(q0 + c) * T.rows + r] = T.Y[(long long)keep[c] * T.rows + r];
  }
}

void ara_absorb(AbsorbTask* d_tasks, int ntask, cudaStream_t st) {
  if (ntask <= 0) return;
  ara_absorb_kernel<<<ntask, 128, 0, st>>>(d_tasks);
  TLRG_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------- JACOBI SVD ----
// One-sided Jacobi on the columns of A (n x n): A V = U Sigma.  Round-robin
// ordering; a warp owns one column pair per step.  Works on a staged copy
// (shared memory when it fits, else T.work) and writes the columns back sorted
// by singular value (descending, ties by index) like dgesdd's output order.
constexpr int JT = 1024;

__global__ void __launch_bounds__(JT) jacobi_svd_kernel(SvdTask* tasks, int staged) {
  extern __shared__ double jsm[];
  SvdTask& T = tasks[blockIdx.x];
  const int n = T.n, m = T.m > 0 ? T.m : T.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = JT / 32;
  if (n == 0) {
    if (tid == 0) *T.rank_out = 0;
    return;
  }
  double* A = staged ? jsm : T.work;       // m x n
  double* V = A + (long long)m * n;        // n x n
  for (long long e = tid; e < (long long)m * n; e += JT) A[e] = T.A[e];
  for (long long e = tid; e < (long long)n * n; e += JT) V[e] = (e % n == e / n) ? 1.0 : 0.0;
  __shared__ int rotated;
  __shared__ double s_tiny;
  {
    __shared__ double red[32];
    double f = 0.0;
    for (long long e = tid; e < (long long)m * n; e += JT) f += A[e] * A[e];
    f = block_sum(f, red);
    if (tid == 0) s_tiny = f * 1e-34;  // (1e-17 ||A||_F)^2: below rounding of any column
  }
  __syncthreads();
  const double tiny2 = s_tiny;
  // rotation threshold: rounding level of an m-term dot product (dgesvj style)
  const double tol = fmax(1e-15, 2.0 * sqrt((double)m) * 2.220446049250313e-16);
  const int nn = n + (n & 1);
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int step = 0; step < nn - 1; ++step) {
      for (int pi = warp; pi < nn / 2; pi += nw) {
        int p = (step + pi) % (nn - 1);
        int q = pi == 0 ? nn - 1 : (step - pi + nn - 1) % (nn - 1);
        if (p >= n || q >= n) continue;
        double* ap = A + (long long)p * m;
        double* aq = A + (long long)q * m;
        double al = 0, be = 0, ga = 0;
        for (int r = lane; r < m; r += 32) {
          al += ap[r] * ap[r];
          be += aq[r] * aq[r];
          ga += ap[r] * aq[r];
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (al > tiny2 && be > tiny2 && fabs(ga) > tol * sqrt(al * be)) {
          double zeta = (be - al) / (2.0 * ga);
          double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          for (int r = lane; r < m; r += 32) {
            double x = ap[r], y = aq[r];
            ap[r] = c * x - s * y;
            aq[r] = s * x + c * y;
          }
          double* vp = V + (long long)p * n;
          double* vq = V + (long long)q * n;
          for (int r = lane; r < n; r += 32) {
            double x = vp[r], y = vq[r];
            vp[r] = c * x - s * y;
            vq[r] = s * x + c * y;
          }
          if (lane == 0) rotated = 1;
        }
      }
      __syncthreads();
    }
    if (!rotated) break;
    __syncthreads();
  }
  // singular values = column norms of A
  for (int p = warp; p < n; p += nw) {
    double s = 0.0;
    for (int r = lane; r < m; r += 32) s += A[(long long)p * m + r] * A[(long long)p * m + r];
    s = warp_sum(s);
    if (lane == 0) T.sig[p] = sqrt(s);
  }
  __syncthreads();
  __shared__ int cnt;
  if (tid == 0) cnt = 0;
  __syncthreads();
  for (int p = warp; p < n; p += nw) {
    double sp = T.sig[p];
    int rk = 0;
    for (int q = lane; q < n; q += 32) {
      double sq = T.sig[q];
      rk += (sq > sp || (sq == sp && q < p)) ? 1 : 0;
    }
    rk = warp_sum_int(rk);
    if (lane == 0 && sp > T.cut) atomicAdd(&cnt, 1);
    for (int r = lane; r < m; r += 32) T.A[(long long)rk * m + r] = A[(long long)p * m + r];
    for (int r = lane; r < n; r += 32) T.V[(long long)rk * n + r] = V[(long long)p * n + r];
  }
  __syncthreads();
  // sigma in descending order
  for (int p = warp; p < n; p += nw) {
    double s = 0.0;
    for (int r = lane; r < m; r += 32) s += T.A[(long long)p * m + r] * T.A[(long long)p * m + r];
    s = warp_sum(s);
    if (lane == 0) T.sig[p] = sqrt(s);
  }
  if (tid == 0) *T.rank_out = cnt;
}

void jacobi_svd(SvdTask* d_tasks, int ntask, int max_n, cudaStream_t st, int max_m) {
  static size_t lim = enable_max_dyn_smem(jacobi_svd_kernel);
  if (ntask <= 0) return;
  if (max_m <= 0) max_m = max_n;
  size_t bytes = ((size_t)max_m * max_n + (size_t)max_n * max_n) * 8;
  int staged = bytes <= lim;
  jacobi_svd_kernel<<<ntask, JT, staged ? bytes : 16, st>>>(d_tasks, staged);
  TLRG_CUDA(cudaGetLastError());
}

// ------------------------------------------------------ BLOCK PRODUCTS ----
__global__ void __launch_bounds__(128) block_products_kernel(const BlockItem* items) {
  const BlockItem& B = items[blockIdx.x];
  for (int r = threadIdx.x; r < B.rows; r += blockDim.x) {
    for (int c = 0; c < B.kkj; ++c) {
      double s = 0.0;
      for (int p = 0; p < B.kij; ++p) s += B.U[(long long)p * B.rows + r] * B.G[p + c * B.ldg];
      B.H[r + c * B.ldh] = s;
    }
  }
}

void block_products(BlockItem* d_items, int nitems, int, cudaStream_t st) {
  if (nitems <= 0) return;
  block_products_kernel<<<nitems, 128, 0, st>>>(d_items);
  TLRG_CUDA(cudaGetLastError());
}

__global__ void batched_copy_kernel(const CopyItem* items) {
  const CopyItem& C = items[blockIdx.x];
  long long n = (long long)C.rows * C.cols;
  for (long long e = threadIdx.x; e < n; e += blockDim.x) {
    int r = (int)(e % C.rows), c = (int)(e / C.rows);
    C.dst[r + c * C.ldd] = C.src[r + c * C.lds];
  }
}

void batched_copy(CopyItem* d_items, int n, cudaStream_t st) {
  if (n <= 0) return;
  batched_copy_kernel<<<n, 256, 0, st>>>(d_items);
  TLRG_CUDA(cudaGetLastError());
}

__global__ void fill_zero_kernel(double* p, long long n) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    p[e] = 0.0;
}
void fill_zero(double* p, long long n, cudaStream_t st) {
  if (n <= 0) return;
  int blocks = (int)std::min<long long>((n + 255) / 256, 148 * 16);
  fill_zero_kernel<<<blocks, 256, 0, st>>>(p, n);
  TLRG_CUDA(cudaGetLastError());
}

}  // namespace tlrg
