#include <cooperative_groups.h>
#include <cstdio>
#include <vector>
#include <random>
#include "common.cuh"
namespace cg = cooperative_groups;
using namespace tlrg;
constexpr int PB = 32;
constexpr int PO_T = 256;
constexpr int PO_W = PO_T / 32;
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

__global__ void __launch_bounds__(PO_T) potrf_x(double* A, int n, int* info, long long* tm) {
  long long t0 = clock64(), tp1 = 0, tp2 = 0, ts1 = 0, ts2 = 0;
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
    long long a1 = clock64(); tp1 += a1 - t0;
    grid.sync();
    long long a2 = clock64(); ts1 += a2 - a1; t0 = a2;
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
    long long b1 = clock64(); tp2 += b1 - t0;
    grid.sync();
    long long b2 = clock64(); ts2 += b2 - b1; t0 = b2;
  }
  if (threadIdx.x == 0) { tm[blockIdx.x*4+0] = tp1; tm[blockIdx.x*4+1] = ts1; tm[blockIdx.x*4+2] = tp2; tm[blockIdx.x*4+3] = ts2; }
  // zero the strict upper triangle (dense_kernels.cpp:79-80)
  for (long long e = blockIdx.x * (long long)PO_T + tid; e < (long long)n * n;
       e += (long long)gridDim.x * PO_T) {
    const int i = (int)(e % n), j = (int)(e / n);
    if (i < j) A[e] = 0.0;
  }
}



int main() {
  const int n = 512;
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  std::vector<double> X((size_t)n * n), A((size_t)n * n, 0.0);
  for (auto& x : X) x = nd(g);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0;
      for (int k = 0; k < n; ++k) s += X[i + k * n] * X[j + k * n];
      A[i + j * n] = s / n + (i == j ? 1.0 : 0.0);
    }
  double *dA, *dW; int* info; long long* tm;
  cudaMalloc(&dA, 8 * n * n); cudaMalloc(&dW, 8 * n * n); cudaMalloc(&info, 16); cudaMalloc(&tm, 8*2048); cudaMemset(tm, 0, 8*2048);
  cudaMemcpy(dA, A.data(), 8 * n * n, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int grid : {8, 16, 48}) for (int rep = 0; rep < 2; ++rep) {
    cudaMemcpy(dW, dA, 8 * n * n, cudaMemcpyDeviceToDevice);
    cudaMemset(info, 0xff, 4);
    int nn = n;
    void* args[] = {&dW, &nn, &info, &tm};
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)potrf_x, dim3(grid), dim3(PO_T), args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    std::vector<long long> h(4*grid); cudaMemcpy(h.data(), tm, 8*4*grid, cudaMemcpyDeviceToHost);
    printf("grid %d: %.1f us  cta0 phase1 %lld sync1 %lld phase2 %lld sync2 %lld kcyc (%s)\n", grid, ms*1e3, h[0]/1000, h[1]/1000, h[2]/1000, h[3]/1000, cudaGetErrorString(cudaGetLastError()));
  }
}
