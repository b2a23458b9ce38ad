// ARA device kernels: per-tile Gaussian draws, the reference's two-sweep
// block Gram-Schmidt with column-wise MGS2 and random replacement of deficient
// columns (dense_kernels.cpp:331-420), the adaptive absorb/convergence state
// machine (ara.cpp:155-195), small one-sided Jacobi SVDs for recompression
// (ara.cpp:201-211), block-diagonal products and gathers.
#include <cfloat>

#include "kernels.h"

namespace tlrg {

// ------------------------------------------------------------------ RNG ---
__global__ void rng_seed_kernel(RngState* states, const uint64_t* seeds, int n) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) rng_seed(&states[t], seeds[t]);
}

__global__ void __launch_bounds__(128) rng_draw_kernel(RngState* states, const int* idx,
                                                       int ntiles, double* out, long long count,
                                                       long long out_stride) {
  __shared__ uint64_t smt[4][MT_N];
  int warp = threadIdx.x >> 5;
  int t = blockIdx.x * 4 + warp;
  if (t >= ntiles) return;
  RngState* g = &states[idx ? idx[t] : t];
  int ix, hc;
  double c;
  warp_rng_load(g, smt[warp], ix, hc, c);
  warp_rng_draw(smt[warp], ix, hc, c, out + (long long)t * out_stride, count);
  warp_rng_store(g, smt[warp], ix, hc, c);
}

void rng_seed(RngState* states, const uint64_t* d_seeds, int n, cudaStream_t st) {
  if (n <= 0) return;
  rng_seed_kernel<<<(n + 127) / 128, 128, 0, st>>>(states, d_seeds, n);
  TLRG_CUDA(cudaGetLastError());
}
void rng_draw(RngState* states, const int* d_idx, int ntiles, double* out, long long count,
              long long out_stride, cudaStream_t st) {
  if (ntiles <= 0 || count <= 0) return;
  rng_draw_kernel<<<(ntiles + 3) / 4, 128, 0, st>>>(states, d_idx, ntiles, out, count,
                                                    out_stride);
  TLRG_CUDA(cudaGetLastError());
}

// --------------------------------------------------------------- ORTHOG ---
constexpr int PT = 256;  // threads per panel CTA

__global__ void __launch_bounds__(PT) panel_tau_kernel(PanelTask* tasks) {
  __shared__ double red[32];
  PanelTask& T = tasks[blockIdx.x];
  long long n = (long long)T.rows * T.width;
  double s = 0.0;
  for (long long e = threadIdx.x; e < n; e += PT) s += T.Y[e] * T.Y[e];
  s = block_sum(s, red);
  if (threadIdx.x == 0) {
    double tau = 100.0 * DBL_EPSILON * sqrt(s);  // dense_kernels.cpp:391-392
    T.tau = tau == 0.0 ? DBL_MIN : tau;
  }
}

void panel_tau(PanelTask* d_tasks, int ntask, cudaStream_t st) {
  if (ntask <= 0) return;
  panel_tau_kernel<<<ntask, PT, 0, st>>>(d_tasks);
  TLRG_CUDA(cudaGetLastError());
}

// y_j -= sum_{p<j} <y_p, y_j> y_p  (one classical pass; returns via cbuf)
__device__ __forceinline__ void cgs_pass(double* Y, int rows, int j, double* cbuf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = PT / 32;
  const double* yj = Y + (long long)j * rows;
  for (int p = warp; p < j; p += nw) {
    const double* yp = Y + (long long)p * rows;
    double s = 0.0;
    for (int r = lane; r < rows; r += 32) s += yp[r] * yj[r];
    s = warp_sum(s);
    if (lane == 0) cbuf[p] = s;
  }
  __syncthreads();
  double* yw = Y + (long long)j * rows;
  for (int r = threadIdx.x; r < rows; r += PT) {
    double s = 0.0;
    for (int p = 0; p < j; ++p) s += cbuf[p] * Y[(long long)p * rows + r];
    yw[r] -= s;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(PT) panel_mgs_kernel(PanelTask* tasks, int sweep, int finalize,
                                                       int ys_in_smem, int cbuf_len) {
  extern __shared__ double smem[];
  double* cbuf = smem;                                  // cbuf_len
  double* red = cbuf + cbuf_len;                        // 32
  uint64_t* smt = reinterpret_cast<uint64_t*>(red + 32);  // MT_N
  double* ysm = reinterpret_cast<double*>(smt + MT_N);  // rows*width when staged

  PanelTask& T = tasks[blockIdx.x];
  const int rows = T.rows, w = T.width, q = T.q;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* Y = ys_in_smem ? ysm : T.Y;
  if (ys_in_smem)
    for (long long e = tid; e < (long long)rows * w; e += PT) ysm[e] = T.Y[e];
  double* Rp = T.Rp;
  for (long long e = tid; e < (long long)w * w; e += PT) Rp[e] = 0.0;
  if (sweep == 0)
    for (int j = tid; j < w; j += PT) {
      T.deficient[j] = 0;
      T.tiny[j] = 0.0;
    }
  __shared__ int rng_loaded;
  __shared__ int s_idx, s_hc;
  __shared__ double s_c;
  if (tid == 0) rng_loaded = 0;
  __syncthreads();
  const double tau = T.tau;

  for (int j = 0; j < w; ++j) {
    double* yj = Y + (long long)j * rows;
    for (int pass = 0; pass < 2; ++pass) {
      if (j == 0) break;
      cgs_pass(Y, rows, j, cbuf);
      for (int p = tid; p < j; p += PT) Rp[p + (long long)j * w] += cbuf[p];
      __syncthreads();
    }
    double ss = 0.0;
    for (int r = tid; r < rows; r += PT) ss += yj[r] * yj[r];
    double nj = sqrt(block_sum(ss, red));
    if (!(nj >= tau)) {
      // deficient column: record, then restart from a fresh random direction
      if (tid == 0 && !T.deficient[j]) {
        T.deficient[j] = 1;
        T.tiny[j] = isfinite(nj) ? nj : 0.0;
      }
      if (warp == 0) {
        int ix, hc;
        double c;
        if (!rng_loaded) {
          warp_rng_load(T.rng, smt, ix, hc, c);
        } else {
          ix = s_idx;
          hc = s_hc;
          c = s_c;
        }
        warp_rng_draw(smt, ix, hc, c, yj, rows);
        if (lane == 0) {
          s_idx = ix;
          s_hc = hc;
          s_c = c;
          rng_loaded = 1;
        }
      }
      __syncthreads();
      if (q > 0) {
        // y -= Q (Q^T y)   (dense_kernels.cpp:352-358)
        for (int t = warp; t < q; t += PT / 32) {
          const double* qt = T.Q + (long long)t * rows;
          double s = 0.0;
          for (int r = lane; r < rows; r += 32) s += qt[r] * yj[r];
          s = warp_sum(s);
          if (lane == 0) cbuf[t] = s;
        }
        __syncthreads();
        for (int r = tid; r < rows; r += PT) {
          double s = 0.0;
          for (int t = 0; t < q; ++t) s += T.Q[(long long)t * rows + r] * cbuf[t];
          yj[r] -= s;
        }
        __syncthreads();
      }
      for (int pass = 0; pass < 2; ++pass)
        if (j > 0) cgs_pass(Y, rows, j, cbuf);
      ss = 0.0;
      for (int r = tid; r < rows; r += PT) ss += yj[r] * yj[r];
      nj = sqrt(block_sum(ss, red));
      if (nj == 0.0) {
        __syncthreads();
        if (tid == 0) yj[j % rows] = 1.0;
        nj = 1.0;
      }
      if (tid == 0) Rp[j + (long long)j * w] = 0.0;
    } else {
      if (tid == 0) Rp[j + (long long)j * w] = nj;
    }
    const double inv = 1.0 / nj;
    __syncthreads();
    for (int r = tid; r < rows; r += PT) yj[r] *= inv;
    __syncthreads();
  }
  if (rng_loaded && warp == 0) warp_rng_store(T.rng, smt, s_idx, s_hc, s_c);
  if (ys_in_smem)
    for (long long e = tid; e < (long long)rows * w; e += PT) T.Y[e] = ysm[e];
  __syncthreads();

  // R <- Rp * R  (R = I before the first sweep)
  double* R = T.R;
  double* Rt = T.Rp + (long long)w * w;  // second scratch half
  if (sweep == 0) {
    for (long long e = tid; e < (long long)w * w; e += PT) R[e] = Rp[e];
  } else {
    for (long long e = tid; e < (long long)w * w; e += PT) {
      int p = (int)(e % w), jj = (int)(e / w);
      double s = 0.0;
      for (int t = p; t <= jj; ++t) s += Rp[p + (long long)t * w] * R[t + (long long)jj * w];
      Rt[e] = p <= jj ? s : 0.0;
    }
    __syncthreads();
    for (long long e = tid; e < (long long)w * w; e += PT) R[e] = Rt[e];
  }
  __syncthreads();
  if (finalize) {
    // dense_kernels.cpp:407-417
    for (int jj = tid; jj < w; jj += PT) {
      if (T.deficient[jj]) {
        for (int i = 0; i < w; ++i) R[i + (long long)jj * w] = 0.0;
        R[jj + (long long)jj * w] = T.tiny[jj];
        T.col_norms[jj] = T.tiny[jj];
        T.new_mass[jj] = T.tiny[jj];
      } else {
        double s = 0.0;
        for (int i = 0; i <= jj; ++i) s += R[i + (long long)jj * w] * R[i + (long long)jj * w];
        T.col_norms[jj] = sqrt(s);
        T.new_mass[jj] = fabs(R[jj + (long long)jj * w]);
      }
    }
  }
}

void panel_mgs(PanelTask* d_tasks, int ntask, int sweep, int finalize, int max_width,
               int max_rows, cudaStream_t st) {
  if (ntask <= 0) return;
  int cbuf_len = max_width > max_rows ? max_width : max_rows;
  size_t base = (size_t)(cbuf_len + 32 + MT_N) * 8;
  size_t ys = (size_t)max_rows * max_width * 8;
  static size_t lim = enable_max_dyn_smem(panel_mgs_kernel);
  int in_smem = base + ys <= lim;
  size_t bytes = base + (in_smem ? ys : 0);
  panel_mgs_kernel<<<ntask, PT, bytes, st>>>(d_tasks, sweep, finalize, in_smem, cbuf_len);
  TLRG_CUDA(cudaGetLastError());
}

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
constexpr int JT = 256;

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
  __syncthreads();
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
        if (ga != 0.0 && fabs(ga) > 1e-15 * sqrt(al * be)) {
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
  if (ntask <= 0) return;
  if (max_m <= 0) max_m = max_n;
  size_t bytes = ((size_t)max_m * max_n + (size_t)max_n * max_n) * 8;
  static size_t lim = enable_max_dyn_smem(jacobi_svd_kernel);
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
