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
// the rotation and the sums are written with explicit rounding intrinsics so
// that the one-CTA and the cluster kernel (jacobi_wide_kernel) compile to the
// same arithmetic (no compiler choice of FMA contraction): bitwise-equal results
__device__ __forceinline__ double jrot_a(double c, double s, double x, double y) {
  return __dadd_rn(__dmul_rn(c, x), -__dmul_rn(s, y));
}
__device__ __forceinline__ double jrot_b(double c, double s, double x, double y) {
  return __dadd_rn(__dmul_rn(s, x), __dmul_rn(c, y));
}

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
    for (long long e = tid; e < (long long)m * n; e += JT) f = __fma_rn(A[e], A[e], f);
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
          al = __fma_rn(ap[r], ap[r], al);
          be = __fma_rn(aq[r], aq[r], be);
          ga = __fma_rn(ap[r], aq[r], ga);
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
            ap[r] = jrot_a(c, s, x, y);
            aq[r] = jrot_b(c, s, x, y);
          }
          double* vp = V + (long long)p * n;
          double* vq = V + (long long)q * n;
          for (int r = lane; r < n; r += 32) {
            double x = vp[r], y = vq[r];
            vp[r] = jrot_a(c, s, x, y);
            vq[r] = jrot_b(c, s, x, y);
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
    for (int r = lane; r < m; r += 32) s = __fma_rn(A[(long long)p * m + r], A[(long long)p * m + r], s);
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
    for (int r = lane; r < m; r += 32) s = __fma_rn(T.A[(long long)p * m + r], T.A[(long long)p * m + r], s);
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
// JS_T = 256 threads give 32 pair slots per pass; cores with more than 32 pairs
// (n > 64) take the 512-thread instance so every step is one pass.
template <int JS_T>
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
  static size_t lim2 = std::min(enable_max_dyn_smem(jacobi_small_kernel<256>),
                                enable_max_dyn_smem(jacobi_small_kernel<512>));
  if (ntask <= 0) return;
  if (max_m <= 0) max_m = max_n;
  size_t bytes = ((size_t)max_m * max_n + (size_t)max_n * max_n) * 8;
  if (max_n <= 128 && bytes <= lim2) {
    if (max_n > 64) jacobi_small_kernel<512><<<ntask, 512, bytes, st>>>(d_tasks);
    else jacobi_small_kernel<256><<<ntask, 256, bytes, st>>>(d_tasks);
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
// E = column elements per lane (m <= 32 E); EV > 0: the two V columns (n <= 32 EV)
// are loaded with the A columns (one L2 round trip per pair instead of two);
// JW_T threads per CTA, JW_CL CTAs per cluster (16 = non-portable size, for the
// 1024-row panels of cfg4).
template <int E, int EV, int JW_T, int JW_CL>
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
    constexpr int V = 1024 / JW_T;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      double pk = 0.0;
      for (long long e = tid + k * JW_T; e < (long long)m * n; e += 1024) pk = __fma_rn(T.A[e], T.A[e], pk);
      pk = warp_sum(pk);
      if (lane == 0) red[warp + k * nw] = pk;
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
        double* vp = V + (long long)p * n;
        double* vq = V + (long long)q * n;
        double x[E], y[E];
        double xv[EV > 0 ? EV : 1], yv[EV > 0 ? EV : 1];
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int r = lane + 32 * e;
          x[e] = r < m ? __ldcg(ap + r) : 0.0;
          y[e] = r < m ? __ldcg(aq + r) : 0.0;
        }
#pragma unroll
        for (int e = 0; e < EV; ++e) {
          const int r = lane + 32 * e;
          xv[e] = r < n ? __ldcg(vp + r) : 0.0;
          yv[e] = r < n ? __ldcg(vq + r) : 0.0;
        }
        double al = 0, be = 0, ga = 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          al = __fma_rn(x[e], x[e], al);
          be = __fma_rn(y[e], y[e], be);
          ga = __fma_rn(x[e], y[e], ga);
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
              __stcg(ap + r, jrot_a(c, s, x[e], y[e]));
              __stcg(aq + r, jrot_b(c, s, x[e], y[e]));
            }
          }
          if (EV > 0) {
#pragma unroll
            for (int e = 0; e < (EV > 0 ? EV : 1); ++e) {
              const int r = lane + 32 * e;
              if (r < n) {
                __stcg(vp + r, jrot_a(c, s, xv[e], yv[e]));
                __stcg(vq + r, jrot_b(c, s, xv[e], yv[e]));
              }
            }
          } else {
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
                __stcg(vp + r, jrot_a(c, s, x[e], y[e]));
                __stcg(vq + r, jrot_b(c, s, x[e], y[e]));
              }
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
    for (int r = lane; r < m; r += 32) {
      const double v = __ldcg(A + (long long)p * m + r);
      s = __fma_rn(v, v, s);
    }
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
      s = __fma_rn(v, v, s);
    }
    s = warp_sum(s);
    if (lane == 0) T.sig[p] = sqrt(s);
  }
  if (crank == 0 && tid == 0) *T.rank_out = cnt;
  cluster_sync_all();  // no CTA leaves while its shared memory may still be addressed
}

template <int E, int EV, int NT, int CL>
static void launch_wide(SvdTask* d_tasks, int ntask, cudaStream_t st) {
  static bool once = [] {
    if (CL > 8)
      cudaFuncSetAttribute(jacobi_wide_kernel<E, EV, NT, CL>,
                           cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return true;
  }();
  (void)once;
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((unsigned)(ntask * CL));
  lc.blockDim = dim3(NT);
  lc.dynamicSmemBytes = 0;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  TLRG_CUDA(cudaLaunchKernelEx(&lc, jacobi_wide_kernel<E, EV, NT, CL>, d_tasks));
}

void jacobi_svd_wide(SvdTask* d_tasks, int ntask, int max_n, cudaStream_t st, int max_m) {
  if (ntask <= 0) return;
  const int mm = std::max(max_m, max_n);
  if (mm <= 256) launch_wide<8, 8, 512, 8>(d_tasks, ntask, st);
  else if (mm <= 512) launch_wide<16, 0, 512, 8>(d_tasks, ntask, st);
  else if (mm <= 1024 && max_n <= 288) launch_wide<32, 9, 256, 16>(d_tasks, ntask, st);
  else if (mm <= 1024) launch_wide<32, 0, 256, 16>(d_tasks, ntask, st);
  else throw CudaError("jacobi_svd_wide: more than 1024 rows");
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
// H[r, c] = sum_p U[r, p] G[p, c] for one block (rows x kij times kij x kkj).
// Each thread owns HP_R rows (stride HP_T) and eight output columns at a time;
// G is staged in shared memory 256 rows x 8 columns at a time, so every U
// element is loaded once per eight columns (the one-row-per-thread loop loaded
// it kkj times and ran the largest near-diagonal blocks, 1024 x 170 x 170 at
// cfg4, for ~20 ms on one CTA).  The p-sum runs in the same order as before,
// so the result is bitwise unchanged.  Rows [r0, r1) let several CTAs share a
// tall block.
constexpr int HP_T = 128, HP_R = 4, HP_P = 256;
__device__ __forceinline__ void hblock_product(const double* U, const double* G, long long ldg,
                                               double* H, long long ldh, int rows, int r0, int r1,
                                               int kij, int kkj, double (*sG)[8]) {
  const int tid = threadIdx.x;
  for (int c0 = 0; c0 < kkj; c0 += 8) {
    double acc[HP_R][8];
#pragma unroll
    for (int rr = 0; rr < HP_R; ++rr)
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) acc[rr][cc] = 0.0;
    for (int p0 = 0; p0 < kij; p0 += HP_P) {
      const int np = min(HP_P, kij - p0);
      __syncthreads();
      for (int e = tid; e < np * 8; e += HP_T) {
        const int pp = e >> 3, cc = e & 7;
        sG[pp][cc] = c0 + cc < kkj ? G[(p0 + pp) + (long long)(c0 + cc) * ldg] : 0.0;
      }
      __syncthreads();
      for (int pp = 0; pp < np; ++pp) {
        const double* up = U + (long long)(p0 + pp) * rows;
        double u[HP_R];
#pragma unroll
        for (int rr = 0; rr < HP_R; ++rr) {
          const int r = r0 + tid + rr * HP_T;
          u[rr] = r < r1 ? up[r] : 0.0;
        }
        const double2* g2 = reinterpret_cast<const double2*>(sG[pp]);
        double g[8];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const double2 v = g2[h];
          g[2 * h] = v.x;
          g[2 * h + 1] = v.y;
        }
#pragma unroll
        for (int rr = 0; rr < HP_R; ++rr)
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) acc[rr][cc] += u[rr] * g[cc];
      }
    }
#pragma unroll
    for (int rr = 0; rr < HP_R; ++rr) {
      const int r = r0 + tid + rr * HP_T;
      if (r < r1)
#pragma unroll
        for (int cc = 0; cc < 8; ++cc)
          if (c0 + cc < kkj) H[r + (long long)(c0 + cc) * ldh] = acc[rr][cc];
    }
  }
}
// row chunk of CTA y out of ny for a block of `rows` rows (HP_T * HP_R rows max)
__device__ __forceinline__ void hp_rows(int rows, int y, int ny, int* r0, int* r1) {
  const int per = (rows + ny - 1) / ny;
  *r0 = min(rows, y * per);
  *r1 = min(rows, *r0 + per);
}

__global__ void __launch_bounds__(HP_T) block_products_kernel(const BlockItem* items) {
  __shared__ __align__(16) double sG[HP_P][8];
  const BlockItem& B = items[blockIdx.x];
  int r0, r1;
  hp_rows(B.rows, blockIdx.y, gridDim.y, &r0, &r1);
  hblock_product(B.U, B.G, B.ldg, B.H, B.ldh, B.rows, r0, r1, B.kij, B.kkj, sG);
}

static int hp_chunks(int rows) { return std::max(1, (rows + HP_T * HP_R - 1) / (HP_T * HP_R)); }

void block_products(BlockItem* d_items, int nitems, int max_rows, cudaStream_t st) {
  if (nitems <= 0) return;
  block_products_kernel<<<dim3(nitems, hp_chunks(max_rows)), HP_T, 0, st>>>(d_items);
  TLRG_CUDA(cudaGetLastError());
}

__global__ void __launch_bounds__(HP_T) h_products_kernel(HProductArgs a) {
  __shared__ __align__(16) double sG[HP_P][8];
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
  int r0, r1;
  hp_rows(rows, blockIdx.y, gridDim.y, &r0, &r1);
  hblock_product(U, G, ldg, H, rows, rows, r0, r1, kij, kkj, sG);
}

void h_products(const HProductArgs& a, cudaStream_t st) {
  if (a.T <= 0 || a.nJ <= 0) return;
  h_products_kernel<<<dim3(a.T * a.nJ, hp_chunks(a.b)), HP_T, 0, st>>>(a);
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

// eight loads in flight per thread (restrict operands: the loads of a group
// are issued before its stores)
__global__ void __launch_bounds__(256) batched_copy_kernel(const CopyItem* items) {
  constexpr int U = 8;
  const CopyItem& C = items[blockIdx.x];
  const double* __restrict__ src = C.src;
  double* __restrict__ dst = C.dst;
  const int rows = C.rows;
  const long long n = (long long)rows * C.cols;
  for (long long e0 = threadIdx.x; e0 < n; e0 += (long long)U * blockDim.x) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long e = e0 + (long long)u * blockDim.x;
      if (e < n) {
        const int r = (int)(e % rows), c = (int)(e / rows);
        v[u] = src[r + c * C.lds];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long e = e0 + (long long)u * blockDim.x;
      if (e < n) {
        const int r = (int)(e % rows), c = (int)(e / rows);
        dst[r + c * C.ldd] = v[u];
      }
    }
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
