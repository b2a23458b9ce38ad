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
  // rotation threshold: rounding level of an m-term dot product (m eps); a
  // stricter one only makes the final sweeps chase rounding noise
  const double tol = T.tol > 0.0 ? T.tol : fmax(1e-15, (double)m * 2.220446049250313e-16);
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
        if (al > tiny2 && be > tiny2 && ga * ga > tol * tol * (al * be)) {
          // t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = (be - al) / (2 ga),
          // rewritten with one sqrt, one division and one rsqrt
          const double dl = be - al;
          double t = (dl >= 0 ? 2.0 * ga : -2.0 * ga) / (fabs(dl) + sqrt(dl * dl + 4.0 * ga * ga));
          double c = rsqrt(1.0 + t * t), s = c * t;
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

// ------------------------------------------- ONE-SIDED JACOBI (small) ------
// Same algorithm and output as jacobi_svd for cores n <= 64 held in shared
// memory, but instruction-lean: 256 threads, EIGHT lanes per column pair (4
// pairs per warp, 3-level shuffle reductions), pair lists precomputed per
// step.  The kernels on this path are issue-bound on a single SM.
constexpr int JS_T = 256;
__global__ void __launch_bounds__(JS_T) jacobi_small_kernel(SvdTask* tasks) {
  extern __shared__ double jsm2[];
  SvdTask& T = tasks[blockIdx.x];
  const int n = T.n, m = T.m > 0 ? T.m : T.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int sub = lane >> 3, l8 = lane & 7;  // pair slot within the warp, lane within the pair
  if (n == 0) {
    if (tid == 0) *T.rank_out = 0;
    return;
  }
  double* A = jsm2;                        // m x n
  double* V = A + (long long)m * n;        // n x n
  for (int e = tid; e < m * n; e += JS_T) A[e] = T.A[e];
  for (int e = tid; e < n * n; e += JS_T) V[e] = (e % n == e / n) ? 1.0 : 0.0;
  __shared__ int rotated;
  __shared__ double red[JS_T / 32];
  {
    double f = 0.0;
    for (int e = tid; e < m * n; e += JS_T) f += A[e] * A[e];
    f = warp_sum(f);
    if (lane == 0) red[warp] = f;
  }
  __syncthreads();
  double fro = 0.0;
  for (int w = 0; w < JS_T / 32; ++w) fro += red[w];
  const double tiny2 = fro * 1e-34;
  const double tol = T.tol > 0.0 ? T.tol : fmax(1e-15, (double)m * 2.220446049250313e-16);
  const int nn = n + (n & 1), np = nn / 2;
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int step = 0; step < nn - 1; ++step) {
      for (int base = warp * 4; base < np; base += (JS_T / 32) * 4) {
        const int pi = base + sub;  // warp-uniform trip count (shuffles use the full mask)
        int p = step + pi;
        if (p >= nn - 1) p -= nn - 1;
        int q = nn - 1;
        if (pi != 0) {
          q = step - pi;
          if (q < 0) q += nn - 1;
        }
        const bool live = pi < np && p < n && q < n;
        double al = 0, be = 0, ga = 0;
        double* ap = A + (long long)p * m;
        double* aq = A + (long long)q * m;
        if (live)
          for (int r = l8; r < m; r += 8) {
            const double x = ap[r], y = aq[r];
            al += x * x;
            be += y * y;
            ga += x * y;
          }
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (live && al > tiny2 && be > tiny2 && ga * ga > tol * tol * (al * be)) {
          const double dl = be - al;
          const double t = (dl >= 0 ? 2.0 * ga : -2.0 * ga) / (fabs(dl) + sqrt(dl * dl + 4.0 * ga * ga));
          const double c = rsqrt(1.0 + t * t), sn = c * t;
          for (int r = l8; r < m; r += 8) {
            const double x = ap[r], y = aq[r];
            ap[r] = c * x - sn * y;
            aq[r] = sn * x + c * y;
          }
          double* vp = V + (long long)p * n;
          double* vq = V + (long long)q * n;
          for (int r = l8; r < n; r += 8) {
            const double x = vp[r], y = vq[r];
            vp[r] = c * x - sn * y;
            vq[r] = sn * x + c * y;
          }
          if (l8 == 0) rotated = 1;
        }
      }
      __syncthreads();
    }
    if (!rotated) break;
    __syncthreads();
  }
  for (int p = warp; p < n; p += JS_T / 32) {
    double v = 0.0;
    for (int r = lane; r < m; r += 32) v += A[(long long)p * m + r] * A[(long long)p * m + r];
    v = warp_sum(v);
    if (lane == 0) T.sig[p] = sqrt(v);
  }
  __syncthreads();
  __shared__ int cnt;
  if (tid == 0) cnt = 0;
  __syncthreads();
  for (int p = warp; p < n; p += JS_T / 32) {
    const double sp = T.sig[p];
    int rk = 0;
    for (int q = lane; q < n; q += 32) {
      const double sq = T.sig[q];
      rk += (sq > sp || (sq == sp && q < p)) ? 1 : 0;
    }
    rk = warp_sum_int(rk);
    if (lane == 0 && sp > T.cut) atomicAdd(&cnt, 1);
    for (int r = lane; r < m; r += 32) T.A[(long long)rk * m + r] = A[(long long)p * m + r];
    for (int r = lane; r < n; r += 32) T.V[(long long)rk * n + r] = V[(long long)p * n + r];
  }
  __syncthreads();
  for (int p = warp; p < n; p += JS_T / 32) {
    double v = 0.0;
    for (int r = lane; r < m; r += 32) v += T.A[(long long)p * m + r] * T.A[(long long)p * m + r];
    v = warp_sum(v);
    if (lane == 0) T.sig[p] = sqrt(v);
  }
  if (tid == 0) *T.rank_out = cnt;
}

void jacobi_svd(SvdTask* d_tasks, int ntask, int max_n, cudaStream_t st, int max_m) {
  static size_t lim = enable_max_dyn_smem(jacobi_svd_kernel);
  static size_t lim2 = enable_max_dyn_smem(jacobi_small_kernel);
  if (ntask <= 0) return;
  if (max_m <= 0) max_m = max_n;
  size_t bytes = ((size_t)max_m * max_n + (size_t)max_n * max_n) * 8;
  if (max_n <= 128 && bytes <= lim2) {
    jacobi_small_kernel<<<ntask, JS_T, bytes, st>>>(d_tasks);
    TLRG_CUDA(cudaGetLastError());
    return;
  }
  int staged = bytes <= lim;
  jacobi_svd_kernel<<<ntask, JT, staged ? bytes : 16, st>>>(d_tasks, staged);
  TLRG_CUDA(cudaGetLastError());
}

// ------------------------------------------- ONE-SIDED JACOBI (wide) ------
// The same one-sided Jacobi (same pair schedule, rotation rule, tolerances and
// output order as jacobi_svd_kernel, so the result is bitwise identical) for
// cores too wide for shared memory (n > ~118, A and V in L2).  One task per
// thread-block cluster of JW_CL CTAs: the n/2 disjoint pairs of a step are
// spread over all JW_CL * 16 warps of the cluster, a cluster barrier
// (release/acquire) separates the steps, and each warp keeps its two columns
// in registers between the dot products and the rotation (one L2 round trip
// per column instead of two, and no serial pair loop per warp).  At cfg4's
// recompression (q-hat up to 276) this is the column's critical path.
constexpr int JW_T = 512, JW_CL = 8;

template <int E>
__global__ void __launch_bounds__(JW_T) jacobi_wide_kernel(SvdTask* tasks) {
  const int crank = (int)cluster_ctarank();
  SvdTask& T = tasks[blockIdx.x / JW_CL];
  const int n = T.n, m = T.m > 0 ? T.m : T.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = JW_T / 32;
  const int gw = crank * nw + warp, gnw = JW_CL * nw, gtid = crank * JW_T + tid;
  __shared__ int s_rot[2];
  __shared__ double red[32];
  __shared__ int cnt;
  if (tid == 0) cnt = 0;
  if (n == 0) {
    if (crank == 0 && tid == 0) *T.rank_out = 0;
    return;
  }
  double* A = T.work;                  // m x n
  double* V = A + (long long)m * n;    // n x n
  for (long long e = gtid; e < (long long)m * n; e += JW_CL * JW_T) __stcg(A + e, T.A[e]);
  for (long long e = gtid; e < (long long)n * n; e += JW_CL * JW_T)
    __stcg(V + e, (e % n == e / n) ? 1.0 : 0.0);
  if (tid == 0) s_rot[0] = s_rot[1] = 0;
  double f = 0.0;  // every CTA forms the same Frobenius norm (same order as the 1-CTA kernel)
  {
    // the 1-CTA kernel reduces with 1024 threads: reproduce its partition
    double p0 = 0.0, p1 = 0.0;
    for (long long e = tid; e < (long long)m * n; e += 1024) p0 += T.A[e] * T.A[e];
    for (long long e = tid + 512; e < (long long)m * n; e += 1024) p1 += T.A[e] * T.A[e];
    p0 = warp_sum(p0);
    p1 = warp_sum(p1);
    if (lane == 0) {
      red[warp] = p0;
      red[warp + 16] = p1;
    }
    __syncthreads();
    for (int i = 0; i < 32; ++i) f += red[i];
  }
  const double tiny2 = f * 1e-34;
  const double tol = T.tol > 0.0 ? T.tol : fmax(1e-15, (double)m * 2.220446049250313e-16);
  const int nn = n + (n & 1);
  int* rot0 = static_cast<int*>(__cluster_map_shared_rank(s_rot, 0));
  int* cnt0 = static_cast<int*>(__cluster_map_shared_rank(&cnt, 0));
  cluster_sync_all();
  for (int sweep = 0; sweep < 60; ++sweep) {
    for (int step = 0; step < nn - 1; ++step) {
      for (int pi = gw; pi < nn / 2; pi += gnw) {
        int p = (step + pi) % (nn - 1);
        int q = pi == 0 ? nn - 1 : (step - pi + nn - 1) % (nn - 1);
        if (p >= n || q >= n) continue;
        double* ap = A + (long long)p * m;
        double* aq = A + (long long)q * m;
        double x[E], y[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int r = lane + 32 * e;
          x[e] = r < m ? __ldcg(ap + r) : 0.0;
          y[e] = r < m ? __ldcg(aq + r) : 0.0;
        }
        double al = 0, be = 0, ga = 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          al += x[e] * x[e];
          be += y[e] * y[e];
          ga += x[e] * y[e];
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (al > tiny2 && be > tiny2 && ga * ga > tol * tol * (al * be)) {
          const double dl = be - al;
          double t = (dl >= 0 ? 2.0 * ga : -2.0 * ga) / (fabs(dl) + sqrt(dl * dl + 4.0 * ga * ga));
          double c = rsqrt(1.0 + t * t), s = c * t;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int r = lane + 32 * e;
            if (r < m) {
              __stcg(ap + r, c * x[e] - s * y[e]);
              __stcg(aq + r, s * x[e] + c * y[e]);
            }
          }
          double* vp = V + (long long)p * n;
          double* vq = V + (long long)q * n;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int r = lane + 32 * e;
            x[e] = r < n ? __ldcg(vp + r) : 0.0;
            y[e] = r < n ? __ldcg(vq + r) : 0.0;
          }
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int r = lane + 32 * e;
            if (r < n) {
              __stcg(vp + r, c * x[e] - s * y[e]);
              __stcg(vq + r, s * x[e] + c * y[e]);
            }
          }
          if (lane == 0) atomicOr(rot0 + (sweep & 1), 1);
        }
      }
      cluster_sync_all();
      // the other parity's flag was read by every CTA before this barrier
      if (step == 0 && crank == 0 && tid == 0) s_rot[(sweep + 1) & 1] = 0;
    }
    if (!*reinterpret_cast<volatile int*>(rot0 + (sweep & 1))) break;
  }
  // singular values = column norms of A; then the sorted write-back
  for (int p = gw; p < n; p += gnw) {
    double s = 0.0;
    for (int r = lane; r < m; r += 32) s += __ldcg(A + (long long)p * m + r) * __ldcg(A + (long long)p * m + r);
    s = warp_sum(s);
    if (lane == 0) __stcg(T.sig + p, sqrt(s));
  }
  cluster_sync_all();
  for (int p = gw; p < n; p += gnw) {
    double sp = __ldcg(T.sig + p);
    int rk = 0;
    for (int q = lane; q < n; q += 32) {
      double sq = __ldcg(T.sig + q);
      rk += (sq > sp || (sq == sp && q < p)) ? 1 : 0;
    }
    rk = warp_sum_int(rk);
    if (lane == 0 && sp > T.cut) atomicAdd(cnt0, 1);
    for (int r = lane; r < m; r += 32)
      __stcg(T.A + (long long)rk * m + r, __ldcg(A + (long long)p * m + r));
    for (int r = lane; r < n; r += 32)
      __stcg(T.V + (long long)rk * n + r, __ldcg(V + (long long)p * n + r));
  }
  cluster_sync_all();
  // sigma in descending order
  for (int p = gw; p < n; p += gnw) {
    double s = 0.0;
    for (int r = lane; r < m; r += 32) {
      const double v = __ldcg(T.A + (long long)p * m + r);
      s += v * v;
    }
    s = warp_sum(s);
    if (lane == 0) T.sig[p] = sqrt(s);
  }
  if (crank == 0 && tid == 0) *T.rank_out = cnt;
  cluster_sync_all();  // no CTA leaves while its shared memory may still be addressed
}

void jacobi_svd_wide(SvdTask* d_tasks, int ntask, int max_n, cudaStream_t st) {
  if (ntask <= 0) return;
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((unsigned)(ntask * JW_CL));
  lc.blockDim = dim3(JW_T);
  lc.dynamicSmemBytes = 0;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = JW_CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  if (max_n <= 256)
    TLRG_CUDA(cudaLaunchKernelEx(&lc, jacobi_wide_kernel<8>, d_tasks));
  else if (max_n <= 512)
    TLRG_CUDA(cudaLaunchKernelEx(&lc, jacobi_wide_kernel<16>, d_tasks));
  else
    throw CudaError("jacobi_svd_wide: core wider than 512");
}

int jacobi_staged_max_n() {
  static int nmax = [] {
    size_t lim = enable_max_dyn_smem(jacobi_svd_kernel);
    int n = 1;
    while ((size_t)2 * (n + 1) * (n + 1) * 8 <= lim) ++n;
    return n;
  }();
  return nmax;
}

// ------------------------------------------------- SYMMETRIC JACOBI ------
// Two-sided cyclic Jacobi for a small symmetric matrix B (n x n, n <= 160):
// B = V diag(lam) V^T.  Each parallel step applies n/2 disjoint rotations
// (no dot products: the 2x2 blocks come straight from B), rows then columns,
// three barriers per step.  Output in the SvdTask convention of jacobi_svd for
// a symmetric PSD core: A <- V diag(lam), V, sig = |lam| sorted descending,
// rank_out = #{|lam| > cut}.  Used by the Schur compensation's Rayleigh-Ritz.
constexpr int SJ_T = 1024;
__global__ void __launch_bounds__(SJ_T) sym_jacobi_kernel(SvdTask* tasks) {
  extern __shared__ double sjm[];
  SvdTask& T = tasks[blockIdx.x];
  const int n = T.n, ld = n + 1;
  double* B = sjm;              // n x ld (row-major)
  double* V = B + n * ld;       // n x ld (row-major: V[k][col])
  double* rc = V + n * ld;      // c per pair
  double* rs = rc + 96;         // s per pair
  int* rp = reinterpret_cast<int*>(rs + 96);
  int* rq = rp + 96;
  __shared__ int s_rot;
  __shared__ double s_fro;
  const int tid = threadIdx.x;
  if (n == 0) {
    if (tid == 0) *T.rank_out = 0;
    return;
  }
  for (int e = tid; e < n * n; e += SJ_T) {
    const int i = e % n, j = e / n;
    B[i * ld + j] = 0.5 * (T.A[i + (long long)j * n] + T.A[j + (long long)i * n]);
    V[i * ld + j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    double f = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) f += B[i * ld + j] * B[i * ld + j];
    s_fro = sqrt(f);
  }
  __syncthreads();
  const double tol_abs = (T.tol > 0.0 ? T.tol : 2.220446049250313e-16) * s_fro;
  const int nn = n + (n & 1), np = nn / 2;
  const int lane = tid & 31, warp = tid >> 5;
  for (int sweep = 0; sweep < 30; ++sweep) {
    if (tid == 0) s_rot = 0;
    for (int step = 0; step < nn - 1; ++step) {
      // rotation parameters, one thread per pair (round-robin ordering)
      if (tid < np) {
        const int pi = tid;
        int p = step + pi;
        if (p >= nn - 1) p -= nn - 1;
        int q = nn - 1;
        if (pi != 0) {
          q = step - pi;
          if (q < 0) q += nn - 1;
        }
        if (p > q) { const int t2 = p; p = q; q = t2; }
        double c = 1.0, sn = 0.0;
        if (q < n) {
          const double bpq = B[p * ld + q];
          if (fabs(bpq) > tol_abs) {
            const double tau = (B[q * ld + q] - B[p * ld + p]) / (2.0 * bpq);
            const double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = rsqrt(1.0 + t * t);
            sn = t * c;
            s_rot = 1;
          }
        }
        rc[pi] = c;
        rs[pi] = sn;
        rp[pi] = p;
        rq[pi] = (q < n && sn != 0.0) ? q : -1;
      }
      __syncthreads();
      // rows p, q of B: warp per pair, lanes over columns (no index division)
      for (int pi = warp; pi < np; pi += SJ_T / 32) {
        const int q = rq[pi];
        if (q < 0) continue;
        const int p = rp[pi];
        const double c = rc[pi], sn = rs[pi];
        for (int k = lane; k < n; k += 32) {
          const double x = B[p * ld + k], y = B[q * ld + k];
          B[p * ld + k] = c * x - sn * y;
          B[q * ld + k] = sn * x + c * y;
        }
      }
      __syncthreads();
      // columns p, q of B and of V
      for (int pi = warp; pi < np; pi += SJ_T / 32) {
        const int q = rq[pi];
        if (q < 0) continue;
        const int p = rp[pi];
        const double c = rc[pi], sn = rs[pi];
        for (int k = lane; k < n; k += 32) {
          const double x = B[k * ld + p], y = B[k * ld + q];
          B[k * ld + p] = c * x - sn * y;
          B[k * ld + q] = sn * x + c * y;
          const double vx = V[k * ld + p], vy = V[k * ld + q];
          V[k * ld + p] = c * vx - sn * vy;
          V[k * ld + q] = sn * vx + c * vy;
        }
      }
      __syncthreads();
    }
    if (!s_rot) break;
    __syncthreads();
  }
  // eigenvalues, order by |lam| descending (ties by index), scaled output
  __shared__ int cnt;
  if (tid == 0) cnt = 0;
  __syncthreads();
  for (int p = tid; p < n; p += SJ_T) {
    const double lp = fabs(B[p * ld + p]);
    int rk = 0;
    for (int q = 0; q < n; ++q) {
      const double lq = fabs(B[q * ld + q]);
      rk += (lq > lp || (lq == lp && q < p)) ? 1 : 0;
    }
    if (lp > T.cut) atomicAdd(&cnt, 1);
    T.sig[rk] = lp;
    const double lam = B[p * ld + p];
    for (int k = 0; k < n; ++k) {
      T.A[k + (long long)rk * n] = V[k * ld + p] * lam;
      T.V[k + (long long)rk * n] = V[k * ld + p];
    }
  }
  __syncthreads();
  if (tid == 0) *T.rank_out = cnt;
}

void sym_jacobi(SvdTask* d_tasks, int ntask, int max_n, cudaStream_t st) {
  static size_t lim = enable_max_dyn_smem(sym_jacobi_kernel);
  if (ntask <= 0) return;
  size_t bytes = ((size_t)2 * max_n * (max_n + 1) + 4 * 96) * 8;
  if (bytes > lim) throw CudaError("sym_jacobi: core too large for shared memory");
  sym_jacobi_kernel<<<ntask, SJ_T, bytes, st>>>(d_tasks);
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

__global__ void __launch_bounds__(128) h_products_kernel(HProductArgs a) {
  const int t = blockIdx.x / a.nJ, jj = blockIdx.x - t * a.nJ;
  const long long* tg = a.cols;
  const long long* Jl = tg + a.T;
  const int i = (int)tg[t], j = (int)Jl[jj];
  const int rows = (int)min((long long)a.b, a.n - (long long)i * a.b);
  const long long tij = tri_index(i, j);
  const int kij = a.rank[tij], kkj = (int)Jl[3 * a.nJ + jj];
  // row offset of G_ij inside G_j: ranks of rows k .. i-1 in column j
  __shared__ int s_pre;
  if (threadIdx.x < 32) {
    int s = 0;
    for (int r = a.k + (int)threadIdx.x; r < i; r += 32) s += a.rank[tri_index(r, j)];
    s = warp_sum_int(s);
    if (threadIdx.x == 0) s_pre = s;
  }
  __syncthreads();
  const long long ldg = max((long long)Jl[a.nJ + jj], 1LL);
  const double* U = kij ? a.U[tij] : nullptr;
  const double* G = a.G + Jl[4 * a.nJ + jj] + s_pre;
  double* H = a.H + t * a.stride + Jl[2 * a.nJ + jj] * rows;
  for (int r = threadIdx.x; r < rows; r += blockDim.x) {
    for (int c = 0; c < kkj; ++c) {
      double s = 0.0;
      for (int p = 0; p < kij; ++p) s += U[(long long)p * rows + r] * G[p + c * ldg];
      H[r + c * rows] = s;
    }
  }
}

void h_products(const HProductArgs& a, cudaStream_t st) {
  if (a.T <= 0 || a.nJ <= 0) return;
  h_products_kernel<<<a.T * a.nJ, 128, 0, st>>>(a);
  TLRG_CUDA(cudaGetLastError());
}

__global__ void tri_update_kernel(const long long* t, const int* r, const double* const* u, int n,
                                  int* rank, const double** U) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) {
    rank[t[e]] = r[e];
    U[t[e]] = u[e];
  }
}

void tri_update(const long long* t, const int* r, const double* const* u, int n, int* rank,
                const double** U, cudaStream_t st) {
  if (n <= 0) return;
  tri_update_kernel<<<(n + 127) / 128, 128, 0, st>>>(t, r, u, n, rank, U);
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
