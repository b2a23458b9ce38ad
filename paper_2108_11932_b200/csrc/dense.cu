// Single-tile dense kernels on the factorization's critical path:
//   * Cholesky (dense_kernels.cpp:66-82, LAPACKE_dpotrf)  -- left-looking,
//     32-column panels; the trailing update runs on the grouped DMMA GEMM.
//   * Bunch-Kaufman LDL^T (dense_kernels.cpp:236-281, LAPACKE_dsytrf) with the
//     reference's unpacking into unit-lower L, D and perm.
//   * panel TRSM X = L^{-1} B (dense_kernels.cpp:311-322) shared by all tiles of
//     a column, with the LDL row permutation and D^{-1} fused (factor.cpp:257-262).
//   * small helpers: symmetrize, diagonal combine, pivot traces, D apply.
#include <algorithm>
#include <cfloat>

#include <cooperative_groups.h>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace tlrg {

// ---------------------------------------------------------------- POTRF ---
// Right-looking blocked Cholesky in ONE cooperative kernel over a small
// persistent grid (the diagonal path shares the GPU with the column's ARA).
// Per 32-column panel p:
//   phase 1: every CTA with panel rows factors A_pp redundantly in one warp's
//            REGISTERS (lane i owns row i, column broadcasts by shuffle), then
//            solves its rows of L_rp = A_rp L_pp^{-T} one warp per row;  grid.sync
//   phase 2: CTA 0 stores L_pp; rank-32 update of every trailing lower 32x32
//            tile A_rc -= L_rp L_cp^T spread over all CTAs;               grid.sync
constexpr int PB = 32;
constexpr int PO_T = 256;

// unblocked Cholesky of the pw x pw block (pw <= 32) held one row per lane;
// returns the failing column or -1.  v[j] = L(lane, j) on exit (j <= lane).
__device__ __forceinline__ int chol32_reg(double (&v)[PB], int pw) {
  const int lane = threadIdx.x & 31;
  int fail = -1;
#pragma unroll
  for (int j = 0; j < PB; ++j) {
    if (j < pw && fail < 0) {
      const double d = __shfl_sync(0xffffffffu, v[j], j);
      if (!(d > 0.0)) {
        fail = j;
      } else {
        const double rs = rsqrt(d);
        if (lane == j) v[j] = d * rs;
        else if (lane > j) v[j] *= rs;
        const double lij = v[j];
#pragma unroll
        for (int k = j + 1; k < PB; ++k) {
          const double lkj = __shfl_sync(0xffffffffu, lij, k);
          if (lane >= k) v[k] -= lij * lkj;
        }
      }
    }
  }
  return fail;
}

__global__ void __launch_bounds__(PO_T) potrf_coop_kernel(double* A, int n, int* info) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double Lp[PB][PB + 1];
  __shared__ double Xp[PB][PB + 1];
  __shared__ double Ar[PB][PB + 1];
  __shared__ double Lb[PB][PB + 1];
  __shared__ int s_fail;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nt = (n + PB - 1) / PB;
  auto bw = [&](int t) { return min(PB, n - t * PB); };
  for (int p = 0; p < nt; ++p) {
    const int p0 = p * PB, pw = bw(p);
    const int below = n - (p0 + pw);
    const bool mine = blockIdx.x == 0 || (int)blockIdx.x * PO_T < below;
    // ---- phase 1 -------------------------------------------------------------
    if (mine) {
      if (warp == 0) {
        double v[PB];
#pragma unroll
        for (int j = 0; j < PB; ++j)
          v[j] = (lane < pw && j < pw && j <= lane) ? A[(p0 + lane) + (long long)(p0 + j) * n] : 0.0;
        const int fa = chol32_reg(v, pw);
#pragma unroll
        for (int j = 0; j < PB; ++j) Lp[lane][j] = (j <= lane) ? v[j] : 0.0;
        if (lane == 0) s_fail = fa;
      }
      __syncthreads();
      if (s_fail >= 0) {
        if (tid == 0) atomicCAS(info, -1, p0 + s_fail);
      } else {
        // L_rp = A_rp L_pp^{-T}: one thread per row, forward substitution in
        // registers against L_pp in shared memory, reciprocal pivots precomputed
        if (tid < pw) Xp[0][tid] = 1.0 / Lp[tid][tid];
        __syncthreads();
        for (int r = p0 + pw + blockIdx.x * PO_T + tid; r < n; r += gridDim.x * PO_T) {
          double x[PB];
#pragma unroll
          for (int t = 0; t < PB; ++t) x[t] = t < pw ? A[r + (long long)(p0 + t) * n] : 0.0;
#pragma unroll
          for (int j = 0; j < PB; ++j) {
            double s0 = x[j], s1 = 0.0;
#pragma unroll
            for (int t = 0; t + 1 < j; t += 2) {
              s0 -= x[t] * Lp[j][t];
              s1 -= x[t + 1] * Lp[j][t + 1];
            }
            if (j & 1) s0 -= x[j - 1] * Lp[j][j - 1];
            x[j] = j < pw ? (s0 + s1) * Xp[0][j] : 0.0;
          }
#pragma unroll
          for (int t = 0; t < PB; ++t)
            if (t < pw) A[r + (long long)(p0 + t) * n] = x[t];
        }
      }
    }
    grid.sync();
    if (*(volatile int*)info >= 0) break;
    if (blockIdx.x == 0) {
      for (int e = tid; e < pw * pw; e += PO_T) {
        const int i = e % pw, j = e / pw;
        A[(p0 + i) + (long long)(p0 + j) * n] = i >= j ? Lp[i][j] : 0.0;
      }
    }
    // ---- phase 2: trailing lower tiles (r, c), p < c <= r ------------------------
    const int ntr = nt - p - 1;
    const int ntiles = ntr * (ntr + 1) / 2;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int rr = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
      while (rr * (rr + 1) / 2 > t) --rr;
      while ((rr + 1) * (rr + 2) / 2 <= t) ++rr;
      const int cc = t - rr * (rr + 1) / 2;
      const int r = p + 1 + rr, c = p + 1 + cc;
      const int r0 = r * PB, c0 = c * PB, rw = bw(r), cw = bw(c);
      __syncthreads();
      for (int e = tid; e < PB * PB; e += PO_T) {
        const int i = e % PB, k = e / PB;
        Ar[i][k] = (i < rw && k < pw) ? A[(r0 + i) + (long long)(p0 + k) * n] : 0.0;
        Lb[i][k] = (i < cw && k < pw) ? A[(c0 + i) + (long long)(p0 + k) * n] : 0.0;
      }
      __syncthreads();
      const int ci = tid & 31, rj = tid >> 5;  // 8 row groups x 32 columns
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
      for (int k = 0; k < PB; ++k) {
        const double bv = Lb[ci][k];
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] += Ar[rj + 8 * u][k] * bv;
      }
      if (ci < cw)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = rj + 8 * u;
          if (i < rw) A[(r0 + i) + (long long)(c0 + ci) * n] -= acc[u];
        }
    }
    grid.sync();
  }
  // zero the strict upper triangle (dense_kernels.cpp:79-80)
  for (long long e = blockIdx.x * (long long)PO_T + tid; e < (long long)n * n;
       e += (long long)gridDim.x * PO_T) {
    const int i = (int)(e % n), j = (int)(e / n);
    if (i < j) A[e] = 0.0;
  }
}

__global__ void set_int_kernel(int* p, int v) { *p = v; }

static int coop_grid(const void* kernel, int threads, int want) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, 0);
  int cap = sms * (per > 0 ? per : 1);
  // these kernels are latency-bound and share the GPU with the concurrent ARA
  // stream: a modest persistent grid keeps grid.sync cheap
  if (cap > 64) cap = 64;
  return want < cap ? (want > 0 ? want : 1) : cap;
}

void potrf_impl(double* A, int n, int* info, DescArena& desc, cudaStream_t st) {
  (void)desc;
  set_int_kernel<<<1, 1, 0, st>>>(info, -1);
  int nt = (n + PB - 1) / PB;
  int grid = coop_grid((const void*)potrf_coop_kernel, PO_T, std::max(nt, nt * (nt - 1) / 2));
  if (grid > 48) grid = 48;
  void* args[] = {&A, &n, &info};
  TLRG_CUDA(cudaLaunchCooperativeKernel((void*)potrf_coop_kernel, dim3(grid), dim3(PO_T), args, 0,
                                        st));
}

// ------------------------------------------------------------ CHOLQR -----
// One pass of (shifted) Cholesky QR for a sketch Y (n x p) with G = Y^T Y:
// R^T R = G + s I,  Rinv = R^{-1}  (s = 11 (n p + p (p + 1)) eps_mach tr(G) when
// shift != 0, the shifted-CholQR3 bound).  Directions with a vanishing pivot
// are dropped (zero column of Rinv), so a rank-deficient sketch yields zero
// basis columns instead of a breakdown.  One CTA, p <= 160.
__global__ void __launch_bounds__(1024) cholqr_kernel(const double* G, int p, int n, int shift,
                                                      double* Rinv, int x_in_smem) {
  extern __shared__ double csm[];
  double* R = csm;              // p x p (row-major, ld p+1)
  const int ld = p + 1;
  __shared__ double s_tr;
  __shared__ int s_dead[160];
  const int tid = threadIdx.x;
  for (int e = tid; e < p * p; e += blockDim.x) {
    const int i = e % p, j = e / p;
    R[i * ld + j] = G[i + (long long)j * p];
  }
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int i = 0; i < p; ++i) t += R[i * ld + i];
    s_tr = t;
  }
  __syncthreads();
  const double tr = s_tr;
  if (shift) {
    const double sh = 11.0 * ((double)n * p + (double)p * (p + 1)) * 2.220446049250313e-16 * tr;
    for (int i = tid; i < p; i += blockDim.x) R[i * ld + i] += sh;
  }
  const double tol = 1e-24 * (tr > 0.0 ? tr : 1.0) / p;
  __syncthreads();
  // right-looking Cholesky, upper factor in place.  2-D thread map (32 x 32):
  // thread (ty, tx) owns trailing entries (j+1+ty+32u, j+1+tx+32v) — no index
  // division in the update loop (the kernel is issue-bound otherwise)
  const int tx = tid & 31, ty = tid >> 5;
  for (int j = 0; j < p; ++j) {
    const double d = R[j * ld + j];
    const bool dead = !(d > tol);
    if (tid == 0) s_dead[j] = dead;
    if (dead) {
      __syncthreads();
      for (int k = tid; k < p; k += blockDim.x) {
        R[j * ld + k] = 0.0;
        R[k * ld + j] = 0.0;
      }
      __syncthreads();
      continue;
    }
    const double rr = rsqrt(d);
    __syncthreads();  // every thread has read R[j][j]
    for (int k = j + 1 + tid; k < p; k += blockDim.x) R[j * ld + k] *= rr;
    if (tid == 0) R[j * ld + j] = d * rr;
    __syncthreads();
    for (int a2 = j + 1 + ty; a2 < p; a2 += 32) {
      const double ra = R[j * ld + a2];
      for (int b2 = j + 1 + tx; b2 < p; b2 += 32)
        if (b2 >= a2) R[a2 * ld + b2] -= ra * R[j * ld + b2];
    }
    __syncthreads();
  }
  // R^{-1} (upper): one warp per column j, the lanes split each back-substitution
  // sum (shared-memory column, written out at the end); a dropped pivot leaves a
  // zero row/column, i.e. a zero basis column
  {
    // p x p scratch after R when it fits in shared memory, else the output itself
    double* X = x_in_smem ? R + p * ld : Rinv;
    const int lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
    for (int j = w; j < p; j += nw) {
      double* x = X + j * p;
      for (int i = lane; i < p; i += 32) x[i] = 0.0;
      __syncwarp();
      const double rjj = R[j * ld + j];
      if (lane == 0) x[j] = rjj != 0.0 ? 1.0 / rjj : 0.0;
      __syncwarp();
      for (int i = j - 1; i >= 0; --i) {
        double s0 = 0.0;
        for (int l = i + 1 + lane; l <= j; l += 32) s0 += R[i * ld + l] * x[l];
        s0 = warp_sum(s0);
        const double rii = R[i * ld + i];
        if (lane == 0) x[i] = rii != 0.0 ? -s0 / rii : 0.0;
        __syncwarp();
      }
      if (x_in_smem)
        for (int i = lane; i < p; i += 32) Rinv[(long long)j * p + i] = x[i];
    }
  }
}

// Y <- Y R^{-1} (upper R^{-1} from cholqr_kernel): a CTA owns 16 rows, stages
// them in shared memory and writes the products back in place; every output
// y_rj = sum_{i <= j} y_ri Rinv_ij is one thread's short dot product
constexpr int CQ_ROWS = 16;
__global__ void __launch_bounds__(256) cholqr_apply_kernel(double* Y, int n, int p,
                                                           const double* Rinv) {
  extern __shared__ double ys[];  // CQ_ROWS x p
  const int r0 = blockIdx.x * CQ_ROWS, nr = min(CQ_ROWS, n - r0);
  for (int e = threadIdx.x; e < CQ_ROWS * p; e += blockDim.x) {
    const int r = e % CQ_ROWS, j = e / CQ_ROWS;
    ys[e] = r < nr ? Y[r0 + r + (long long)j * n] : 0.0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < CQ_ROWS * p; e += blockDim.x) {
    const int r = e % CQ_ROWS, j = e / CQ_ROWS;
    const double* x = Rinv + (long long)j * p;
    double s0 = 0.0, s1 = 0.0;
    int i = 0;
    for (; i + 1 <= j; i += 2) {
      s0 += ys[r + i * CQ_ROWS] * __ldg(x + i);
      s1 += ys[r + (i + 1) * CQ_ROWS] * __ldg(x + i + 1);
    }
    if (i <= j) s0 += ys[r + i * CQ_ROWS] * __ldg(x + i);
    if (r < nr) Y[r0 + r + (long long)j * n] = s0 + s1;
  }
}
void cholqr_apply(double* Y, int n, int p, const double* Rinv, cudaStream_t st) {
  static size_t lim = enable_max_dyn_smem(cholqr_apply_kernel);
  (void)lim;
  cholqr_apply_kernel<<<(n + CQ_ROWS - 1) / CQ_ROWS, 256, (size_t)CQ_ROWS * p * 8, st>>>(Y, n, p,
                                                                                      Rinv);
  TLRG_CUDA(cudaGetLastError());
}


void cholqr_factor(const double* G, int p, int n, int shift, double* Rinv, cudaStream_t st) {
  static size_t lim = enable_max_dyn_smem(cholqr_kernel);
  (void)lim;
  size_t bytes = ((size_t)p * (p + 1) + (size_t)p * p) * 8;  // R + R^{-1} scratch
  int x_in_smem = 1;
  if (bytes > lim) {
    bytes = (size_t)p * (p + 1) * 8;
    x_in_smem = 0;
  }
  cholqr_kernel<<<1, 1024, bytes, st>>>(G, p, n, shift, Rinv, x_in_smem);
  TLRG_CUDA(cudaGetLastError());
}

// ------------------------------------------------------- TRTRI (base) -----
// X_bb = L_bb^{-1} for a list of diagonal blocks (<= 32 x 32), one CTA per
// block, one warp per right-hand-side column (lane i owns row i).
__global__ void __launch_bounds__(256) trtri_base_kernel(const double* L, int n, double* X,
                                                         const int* offs, const int* lens) {
  __shared__ double Ls[32][33];
  const int o = offs[blockIdx.x], len = lens[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < 32 * 32; e += 256) {
    const int i = e % 32, k = e / 32;
    Ls[i][k] = (i < len && k <= i) ? L[(o + i) + (long long)(o + k) * n] : 0.0;
  }
  __syncthreads();
  for (int j = warp; j < len; j += 8) {
    double x = lane == j ? 1.0 : 0.0;
    for (int k = j; k < len; ++k) {
      const double xk = __shfl_sync(0xffffffffu, x, k) / Ls[k][k];
      if (lane == k) x = xk;
      if (lane > k) x -= Ls[lane][k] * xk;
    }
    if (lane < len && lane >= j) X[(o + lane) + (long long)(o + j) * n] = x;
  }
}
void trtri_base(const double* L, int n, double* X, const int* d_offs, const int* d_lens,
                int nblocks, cudaStream_t st) {
  if (nblocks <= 0) return;
  trtri_base_kernel<<<nblocks, 256, 0, st>>>(L, n, X, d_offs, d_lens);
  TLRG_CUDA(cudaGetLastError());
}

// ------------------------------------------------------ BUNCH-KAUFMAN -----
// LAPACK dsytf2 (UPLO = 'L') executed by one CTA on an n x n tile in global
// memory.  Interchanges are applied to the whole rows (including the already
// computed multipliers), which yields exactly the reference's unpacked form
// (dense_kernels.cpp:253-279): P A P^T = L D L^T with perm[i] = original row.
constexpr int BK_T = 1024;

__global__ void __launch_bounds__(BK_T) sytrf_bk_kernel(double* A, int n, double* d, double* e,
                                                        uint8_t* s2, int* perm, int* info) {
  __shared__ double rv[32];
  __shared__ int ri[32];
  __shared__ int s_imax, s_kp, s_kstep;
  __shared__ double s_colmax;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = BK_T / 32;
  const double alpha = (1.0 + sqrt(17.0)) / 8.0;
  auto a = [&](int i, int j) -> double& { return A[i + (long long)j * n]; };
  for (int i = tid; i < n; i += BK_T) {
    perm[i] = i;
    d[i] = 0.0;
    if (i < n - 1) e[i] = 0.0;
    s2[i] = 0;
  }
  if (tid == 0) *info = -1;
  __syncthreads();
  // block argmax of |x_i| (first index on ties, like idamax)
  auto argmax = [&](auto getv, int lo, int hi, double& vmax, int& imax) {
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int i = lo + tid; i < hi; i += BK_T) {
      double v = fabs(getv(i));
      if (v > bv || (v == bv && i < bi)) {
        bv = v;
        bi = i;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    __syncthreads();
    if (lane == 0) {
      rv[warp] = bv;
      ri[warp] = bi;
    }
    __syncthreads();
    bv = -1.0;
    bi = 0x7fffffff;
    for (int w = 0; w < nw; ++w)
      if (rv[w] > bv || (rv[w] == bv && ri[w] < bi)) {
        bv = rv[w];
        bi = ri[w];
      }
    vmax = bv < 0 ? 0.0 : bv;
    imax = bi;
  };

  int k = 0;
  while (k < n) {
    int kstep = 1, kp = k;
    double absakk = fabs(a(k, k));
    double colmax = 0.0;
    int imax = k;
    if (k < n - 1) argmax([&](int i) { return a(i, k); }, k + 1, n, colmax, imax);
    if (tid == 0) {
      if (fmax(absakk, colmax) == 0.0) {
        if (*info < 0) *info = k;  // zero pivot: record, keep going
        kp = k;
      } else if (absakk >= alpha * colmax) {
        kp = k;
      } else {
        s_imax = imax;
      }
      s_kp = kp;
      s_kstep = 1;
      s_colmax = colmax;
    }
    __syncthreads();
    if (!(fmax(absakk, colmax) == 0.0) && !(absakk >= alpha * colmax)) {
      // rowmax: off-diagonal max of row imax in the trailing matrix
      double rm1 = 0.0, rm2 = 0.0;
      int i1, i2;
      argmax([&](int j) { return a(imax, j); }, k, imax, rm1, i1);
      if (imax < n - 1) argmax([&](int j) { return a(j, imax); }, imax + 1, n, rm2, i2);
      double rowmax = fmax(rm1, rm2);
      if (tid == 0) {
        if (absakk >= alpha * colmax * (colmax / rowmax)) {
          kp = k;
        } else if (fabs(a(imax, imax)) >= alpha * rowmax) {
          kp = imax;
        } else {
          kp = imax;
          kstep = 2;
        }
        s_kp = kp;
        s_kstep = kstep;
      }
      __syncthreads();
      kp = s_kp;
      kstep = s_kstep;
    } else {
      kp = s_kp;
    }
    __syncthreads();
    const int kk = k + kstep - 1;
    if (kp != kk) {
      // symmetric interchange of rows/columns kk and kp in the trailing matrix,
      // plus the full-row swap of the earlier multipliers (columns < k)
      for (int i = kp + 1 + tid; i < n; i += BK_T) {
        double t = a(i, kk);
        a(i, kk) = a(i, kp);
        a(i, kp) = t;
      }
      for (int j = kk + 1 + tid; j < kp; j += BK_T) {
        double t = a(j, kk);
        a(j, kk) = a(kp, j);
        a(kp, j) = t;
      }
      for (int j = tid; j < k; j += BK_T) {
        double t = a(kk, j);
        a(kk, j) = a(kp, j);
        a(kp, j) = t;
      }
      if (tid == 0) {
        double t = a(kk, kk);
        a(kk, kk) = a(kp, kp);
        a(kp, kp) = t;
        if (kstep == 2) {
          t = a(k + 1, k);
          a(k + 1, k) = a(kp, k);
          a(kp, k) = t;
        }
        int pt = perm[kk];
        perm[kk] = perm[kp];
        perm[kp] = pt;
      }
    }
    __syncthreads();
    if (kstep == 1) {
      double akk = a(k, k);
      if (akk != 0.0) {
        double r1 = 1.0 / akk;
        // trailing rank-1 update (dsyr, lower) then scale the column: one warp
        // per column j, lanes over rows i >= j (coalesced, no index arithmetic)
        for (int j = k + 1 + warp; j < n; j += nw) {
          const double ajk = r1 * a(j, k);
          for (int i = j + lane; i < n; i += 32) a(i, j) -= a(i, k) * ajk;
        }
        __syncthreads();
        for (int i = k + 1 + tid; i < n; i += BK_T) a(i, k) *= r1;
      }
      if (tid == 0) d[k] = a(k, k);
    } else {
      if (k < n - 2) {
        double d21 = a(k + 1, k);
        double d11 = a(k + 1, k + 1) / d21;
        double d22 = a(k, k) / d21;
        double t = 1.0 / (d11 * d22 - 1.0);
        d21 = t / d21;
        for (int j = k + 2 + warp; j < n; j += nw) {
          const double wkj = d21 * (d11 * a(j, k) - a(j, k + 1));
          const double wkp1j = d21 * (d22 * a(j, k + 1) - a(j, k));
          for (int i = j + lane; i < n; i += 32) a(i, j) -= a(i, k) * wkj + a(i, k + 1) * wkp1j;
        }
        __syncthreads();
        for (int j = k + 2 + tid; j < n; j += BK_T) {
          double wk = d21 * (d11 * a(j, k) - a(j, k + 1));
          double wkp1 = d21 * (d22 * a(j, k + 1) - a(j, k));
          a(j, k) = wk;
          a(j, k + 1) = wkp1;
        }
      }
      if (tid == 0) {
        d[k] = a(k, k);
        d[k + 1] = a(k + 1, k + 1);
        e[k] = a(k + 1, k);
        s2[k] = 1;
      }
    }
    __syncthreads();
    k += kstep;
  }
  __syncthreads();
  // unpack: unit lower L (2x2 block off-diagonals belong to D)
  for (long long t = tid; t < (long long)n * n; t += BK_T) {
    int i = (int)(t % n), j = (int)(t / n);
    if (i == j) a(i, j) = 1.0;
    else if (i < j) a(i, j) = 0.0;
    else if (i == j + 1 && s2[j]) a(i, j) = 0.0;
  }
}

void sytrf_bk(double* A, int n, double* d, double* e, uint8_t* s2, int* perm, int* info,
              cudaStream_t st) {
  sytrf_bk_kernel<<<1, BK_T, 0, st>>>(A, n, d, e, s2, perm, info);
  TLRG_CUDA(cudaGetLastError());
}

// ----------------------------------------------------------------- TRSM ---
// X = L^{-1} B for the whole column panel (all tiles share L_kk), right-looking
// over 32-row blocks in one cooperative kernel; 32 x 32 (row block, column
// chunk) tiles are spread over a persistent grid.  Per block row p:
//   phase 1: X_p <- L_pp^{-1} X_p       (warp-parallel substitution)  grid.sync
//   phase 2: X_r -= L_rp X_p, r > p     (32^3 tile products)          grid.sync
// LDL mode (perm != null): X = P B gathered first, L unit lower, D^{-1} applied
// last (factor.cpp:257-262, dense_kernels.cpp:126-144).
constexpr int TR_T = 128;

__global__ void __launch_bounds__(TR_T) trsm_coop_kernel(const double* L, int n, double* B,
                                                         long long nrhs, const int* perm,
                                                         const double* d, const double* e,
                                                         const uint8_t* s2, int* info,
                                                         double* W) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double Ls[32][33];
  __shared__ double Xs[32][33];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool ldl = perm != nullptr;
  double* X = ldl ? W : B;
  const int nt = (n + 31) / 32;
  const long long ncc = (nrhs + 31) / 32;
  if (ldl) {
    for (long long t = blockIdx.x * (long long)TR_T + tid; t < (long long)n * nrhs;
         t += (long long)gridDim.x * TR_T) {
      int i = (int)(t % n);
      long long c = t / n;
      X[t] = B[perm[i] + c * n];
    }
    grid.sync();
  }
  for (int p = 0; p < nt; ++p) {
    const int p0 = p * 32, pw = min(32, n - p0);
    for (long long cc = blockIdx.x; cc < ncc; cc += gridDim.x) {
      const long long c0 = cc * 32;
      const int cw = (int)min(32LL, nrhs - c0);
      __syncthreads();
      for (int t = tid; t < 32 * 32; t += TR_T) {
        int i = t % 32, k = t / 32;
        Ls[i][k] = (i < pw && k < pw) ? L[(p0 + i) + (long long)(p0 + k) * n] : 0.0;
        Xs[i][k] = (i < pw && k < cw) ? X[(p0 + i) + (c0 + k) * n] : 0.0;
      }
      __syncthreads();
      for (int c = warp; c < cw; c += TR_T / 32) {
        double xi = Xs[lane][c];
        for (int j = 0; j < pw; ++j) {
          double xj = __shfl_sync(0xffffffffu, xi, j);
          if (!ldl) xj /= Ls[j][j];
          if (lane == j) xi = xj;
          if (lane > j) xi -= Ls[lane][j] * xj;
        }
        if (lane < pw) X[(p0 + lane) + (c0 + c) * n] = xi;
      }
    }
    grid.sync();
    const long long ntiles = (long long)(nt - p - 1) * ncc;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int r = p + 1 + (int)(t / ncc);
      const long long c0 = (t % ncc) * 32;
      const int r0 = r * 32, rw = min(32, n - r0), cw = (int)min(32LL, nrhs - c0);
      __syncthreads();
      for (int q = tid; q < 32 * 32; q += TR_T) {
        int i = q % 32, k = q / 32;
        Ls[i][k] = (i < rw && k < pw) ? L[(r0 + i) + (long long)(p0 + k) * n] : 0.0;
        Xs[i][k] = (i < pw && k < cw) ? X[(p0 + i) + (c0 + k) * n] : 0.0;
      }
      __syncthreads();
      const int ci = tid & 31, rj = tid >> 5;
      double acc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] = 0.0;
#pragma unroll 8
      for (int k = 0; k < 32; ++k) {
        double xv = Xs[k][ci];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] += Ls[rj + 4 * u][k] * xv;
      }
      if (ci < cw)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          int i = rj + 4 * u;
          if (i < rw) X[(r0 + i) + (c0 + ci) * n] -= acc[u];
        }
    }
    grid.sync();
  }
  if (ldl) {
    // D^{-1} per column, then scatter back into B
    for (long long c = blockIdx.x * (long long)TR_T + tid; c < nrhs;
         c += (long long)gridDim.x * TR_T) {
      double* xc = X + c * n;
      int k = 0;
      while (k < n) {
        if (s2[k]) {
          double det = d[k] * d[k + 1] - e[k] * e[k];
          if (det == 0.0) {
            atomicCAS(info, -1, k);
            break;
          }
          double a = xc[k], b = xc[k + 1];
          xc[k] = (d[k + 1] * a - e[k] * b) / det;
          xc[k + 1] = (d[k] * b - e[k] * a) / det;
          k += 2;
        } else {
          if (d[k] == 0.0) {
            atomicCAS(info, -1, k);
            break;
          }
          xc[k] /= d[k];
          k += 1;
        }
      }
    }
    grid.sync();
    for (long long t = blockIdx.x * (long long)TR_T + tid; t < (long long)n * nrhs;
         t += (long long)gridDim.x * TR_T)
      B[t] = X[t];
  }
}

static double* trsm_scratch(size_t n) {
  static double* p = nullptr;
  static size_t cap = 0;
  if (n > cap) {
    if (p) cudaFree(p);
    TLRG_CUDA(cudaMalloc(&p, n * sizeof(double)));
    cap = n;
  }
  return p;
}

void trsm_panel(const double* L, int n, double* B, long long nrhs, const int* perm,
                const double* d, const double* e, const uint8_t* s2, int* info,
                cudaStream_t st, double* work) {
  if (nrhs <= 0 || n <= 0) return;
  double* W = perm ? (work ? work : trsm_scratch((size_t)n * nrhs)) : nullptr;
  const int nt = (n + 31) / 32;
  const long long ncc = (nrhs + 31) / 32;
  long long want = std::max<long long>(ncc, (long long)(nt - 1) * ncc);
  int grid = coop_grid((const void*)trsm_coop_kernel, TR_T, (int)std::min<long long>(want, 1 << 20));
  void* args[] = {&L, &n, &B, &nrhs, &perm, &d, &e, &s2, &info, &W};
  TLRG_CUDA(cudaLaunchCooperativeKernel((void*)trsm_coop_kernel, dim3(grid), dim3(TR_T), args, 0,
                                        st));
}

// -------------------------------------------------------------- HELPERS ---
__global__ void symmetrize_kernel(double* D, int n) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long tot = (long long)n * n;
  if (t >= tot) return;
  int i = (int)(t % n), j = (int)(t / n);
  if (i <= j) return;
  double v = 0.5 * (D[i + (long long)j * n] + D[j + (long long)i * n]);  // factor.cpp:32-39
  D[i + (long long)j * n] = v;
  D[j + (long long)i * n] = v;
}
void symmetrize(double* D, int n, cudaStream_t st) {
  long long tot = (long long)n * n;
  symmetrize_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(D, n);
  TLRG_CUDA(cudaGetLastError());
}

__global__ void diag_combine_kernel(const double* A, const double* D, const double* corr,
                                    double shift, double* out, int n) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long tot = (long long)n * n;
  if (t >= tot) return;
  int i = (int)(t % n), j = (int)(t / n);
  double v = A[t];
  if (D) v -= D[t];  // factor.cpp:217-218
  if (i == j) {
    if (corr) v += corr[i];  // factor.cpp:219-223
    if (shift > 0) v += shift;  // factor.cpp:224
  }
  out[t] = v;
}
void diag_combine(const double* A, const double* D, const double* corr, double shift,
                  double* out, int n, cudaStream_t st) {
  long long tot = (long long)n * n;
  diag_combine_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(A, D, corr, shift, out, n);
  TLRG_CUDA(cudaGetLastError());
}

__global__ void min_diag_sq_kernel(const double* L, int n, double* out) {
  __shared__ double red[32];
  double m = INFINITY;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double v = L[i + (long long)i * n];
    m = fmin(m, v * v);
  }
  for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = INFINITY;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmin(r, red[w]);
    *out = r;
  }
}
void min_diag_sq(const double* L, int n, double* out, cudaStream_t st) {
  min_diag_sq_kernel<<<1, 256, 0, st>>>(L, n, out);
  TLRG_CUDA(cudaGetLastError());
}

__global__ void min_block_pivot_kernel(const double* d, const double* e, const uint8_t* s2, int n,
                                       double* out) {
  // factor.cpp:87-102 (sequential scan; n <= a few thousand)
  double m = INFINITY;
  int k = 0;
  while (k < n) {
    if (s2[k]) {
      double mean = 0.5 * (d[k] + d[k + 1]);
      double rad = hypot(0.5 * (d[k] - d[k + 1]), e[k]);
      m = fmin(m, fmin(fabs(mean - rad), fabs(mean + rad)));
      k += 2;
    } else {
      m = fmin(m, fabs(d[k]));
      k += 1;
    }
  }
  *out = m;
}
void min_block_pivot(const double* d, const double* e, const uint8_t* s2, int n, double* out,
                     cudaStream_t st) {
  min_block_pivot_kernel<<<1, 1, 0, st>>>(d, e, s2, n, out);
  TLRG_CUDA(cudaGetLastError());
}

// W <- D W  (dense_kernels.cpp:97-116): one thread per (row, column); the
// thread of a 2x2 block's first row updates both rows (BlockDiagonal marks
// block starts only, so the second row of a 2x2 never starts a block)
__device__ __forceinline__ void bd_apply_row(const double* d, const double* e, const uint8_t* s2,
                                             int n, double* x, int r) {
  if (s2[r] && r + 1 < n) {
    const double a = x[r], b = x[r + 1];
    x[r] = d[r] * a + e[r] * b;
    x[r + 1] = e[r] * a + d[r + 1] * b;
  } else if (!(r > 0 && s2[r - 1])) {
    x[r] *= d[r];
  }
}
__global__ void bd_apply_kernel(const double* d, const double* e, const uint8_t* s2, int n,
                                double* W, long long ld, int cols) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int c = blockIdx.y; c < cols; c += gridDim.y) bd_apply_row(d, e, s2, n, W + (long long)c * ld, r);
}
void bd_apply(const double* d, const double* e, const uint8_t* s2, int n, double* W, long long ld,
              int cols, cudaStream_t st) {
  if (cols <= 0 || n <= 0) return;
  dim3 grid((n + 127) / 128, std::min(cols, 1024));
  bd_apply_kernel<<<grid, 128, 0, st>>>(d, e, s2, n, W, ld, cols);
  TLRG_CUDA(cudaGetLastError());
}
// one launch for a list of (D block, column block) items
__global__ void bd_apply_batched_kernel(const BdItem* items, int n, long long ld) {
  const BdItem it = items[blockIdx.y];
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int c = 0; c < it.cols; ++c) bd_apply_row(it.d, it.e, it.s2, n, it.W + (long long)c * ld, r);
}
void bd_apply_batched(const BdItem* d_items, int nitems, int n, long long ld, cudaStream_t st) {
  if (nitems <= 0 || n <= 0) return;
  bd_apply_batched_kernel<<<dim3((n + 127) / 128, nitems), 128, 0, st>>>(d_items, n, ld);
  TLRG_CUDA(cudaGetLastError());
}

__global__ void frob_sq_kernel(const double* p, long long n, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (long long t = threadIdx.x; t < n; t += blockDim.x) s += p[t] * p[t];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}
__global__ void vec_sum_kernel(const double* p, int n, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int t = threadIdx.x; t < n; t += blockDim.x) s += p[t];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}
void block_sum_device(const double* p, int n, double* out, cudaStream_t st) {
  vec_sum_kernel<<<1, 256, 0, st>>>(p, n, out);
  TLRG_CUDA(cudaGetLastError());
}
void frob_sq(const double* p, long long n, double* out, cudaStream_t st) {
  frob_sq_kernel<<<1, 1024, 0, st>>>(p, n, out);
  TLRG_CUDA(cudaGetLastError());
}

// counter-based Gaussian fill (splitmix64 + Box-Muller); used for the Schur
// compensation sketch, whose randomness is not part of the reference's streams.
__global__ void gaussian_fill_kernel(double* out, long long n, uint64_t seed) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long pairs = (n + 1) / 2;
  if (t >= pairs) return;
  uint64_t a = mix64(seed ^ mix64((uint64_t)t * 2 + 1));
  uint64_t b = mix64(a ^ 0x5851f42d4c957f2dULL);
  double u1 = ((double)(a >> 11) + 1.0) * 0x1.0p-53;
  double u2 = (double)(b >> 11) * 0x1.0p-53;
  double r = sqrt(-2.0 * log(u1));
  double s, c;
  sincospi(2.0 * u2, &s, &c);
  out[2 * t] = r * c;
  if (2 * t + 1 < n) out[2 * t + 1] = r * s;
}
void fill_gaussian_philox(double* out, long long n, uint64_t seed, cudaStream_t st) {
  if (n <= 0) return;
  long long pairs = (n + 1) / 2;
  gaussian_fill_kernel<<<(unsigned)((pairs + 255) / 256), 256, 0, st>>>(out, n, seed);
  TLRG_CUDA(cudaGetLastError());
}

// corr[i] = sum_j |D_ij - (Xl Xr^T)_ij| is computed after the GEMM R = D - Xl Xr^T;
// this kernel takes R directly.
// corr_i = sum_j |R_ij| and the row's sum of squares: a CTA owns 32 rows, its
// 16 thread groups split the columns, partials combined in a fixed order
constexpr int RS_G = 16;
__global__ void __launch_bounds__(32 * RS_G) rowsum_abs_kernel(const double* R, int n, double* corr,
                                                               double* frob_part) {
  __shared__ double ps[RS_G][32], pf[RS_G][32];
  const int r = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + r;
  double s = 0.0, f = 0.0;
  if (i < n)
    for (int j = g; j < n; j += RS_G) {
      const double v = R[i + (long long)j * n];
      s += fabs(v);
      f += v * v;
    }
  ps[g][r] = s;
  pf[g][r] = f;
  __syncthreads();
  if (g == 0 && i < n) {
    double a = 0.0, b = 0.0;
    for (int t = 0; t < RS_G; ++t) {
      a += ps[t][r];
      b += pf[t][r];
    }
    corr[i] = a;
    frob_part[i] = b;
  }
}
void rowsum_abs_residual(const double* R, const double*, const double*, int n, int,
                         double* corr, double* frob_part, cudaStream_t st) {
  rowsum_abs_kernel<<<(n + 31) / 32, 32 * RS_G, 0, st>>>(R, n, corr, frob_part);
  TLRG_CUDA(cudaGetLastError());
}

}  // namespace tlrg
