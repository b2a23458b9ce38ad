// Grouped FP64 GEMM on the sm_100a FP64 tensor pipe (DMMA.8x8x4).
//
// One launch computes an arbitrary list of independent problems
//   C_p = alpha_p * op(A_p) * op(B_p) + beta_p * C_p
// with per-problem shapes, strides and transposes.  This is the batched,
// non-uniform GEMM the paper's GPU code obtained from MAGMA and
// the reference runs as millions of small cblas_dgemm calls
// (dense_kernels.cpp:43-57).  CTAs are mapped to (problem, tile) through a
// prefix table, so ragged batches need no padding in HBM.
//
// Tiling: BM x BN x 16 with 4 warps; operands staged through double-buffered
// shared memory by cp.async (8-byte, zero-filled at the edges); padding of the
// shared tiles (stride = 4 mod 16 doubles) keeps the 64-bit fragment reads
// bank-conflict free.
#pragma once
#include "common.cuh"

namespace tlrg {

struct GemmProblem {
  const double* A;
  const double* B;
  double* C;
  long long lda, ldb, ldc;
  int M, N, K;
  int transA, transB;
  double alpha, beta;
  int tile_start;  // exclusive prefix of CTA tiles (filled by the launcher)
  int tiles_n;     // tiles along N
  // optional device-resident controls (read at run time; M/K above are then
  // upper bounds used for tiling): skip the problem when *skip != 0, take the
  // actual M / K from *Mp / *Kp.  This keeps launches static across ARA rounds
  // so a whole round can be captured once and replayed from a device loop.
  const int* skip;
  const int* Mp;
  const int* Kp;
};

static_assert(sizeof(GemmProblem) % 8 == 0 && sizeof(GemmProblem) / 8 <= 128, "descriptor");

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int BM, int BN>
struct GemmCfg {
  static constexpr int BK = 16;
  static constexpr int SA = BM + 4;  // = 4 (mod 16) for BM multiple of 16
  static constexpr int SB = BN + 4;
  static constexpr int WM = BM / 2, WN = BN / 2;  // 2x2 warps
  static constexpr int FM = WM / 8, FN = WN / 8;  // 8x8 fragments per warp
};

template <int BM, int BN>
__global__ void __launch_bounds__(128) grouped_gemm_kernel(const GemmProblem* __restrict__ probs,
                                                           const int* __restrict__ owner) {
  using Cfg = GemmCfg<BM, BN>;
  constexpr int BK = Cfg::BK, SA = Cfg::SA, SB = Cfg::SB;
  __shared__ __align__(16) double As[2][BK * SA];
  __shared__ __align__(16) double Bs[2][BK * SB];
  __shared__ __align__(16) GemmProblem sP;
  __shared__ int s_go;

  // the problem owning this CTA comes from a per-CTA owner table; the 8-byte
  // words of its descriptor are fetched in parallel and the device-side
  // controls are resolved once
  {
    const int pidx = owner[blockIdx.x];
    const unsigned long long* src =
        reinterpret_cast<const unsigned long long*>(probs + pidx);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(&sP);
    constexpr int W = sizeof(GemmProblem) / 8;
    if (threadIdx.x < W) dst[threadIdx.x] = src[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0) {
      int go = 1;
      if (sP.skip && *sP.skip) go = 0;
      if (go && sP.Mp) sP.M = min(sP.M, *sP.Mp);
      if (go && sP.Kp) sP.K = min(sP.K, *sP.Kp);
      const int local = blockIdx.x - sP.tile_start;
      if (go && (local / sP.tiles_n) * BM >= sP.M) go = 0;
      s_go = go;
    }
    __syncthreads();
    if (!s_go) return;
  }
  const GemmProblem P = sP;
  const int local = blockIdx.x - P.tile_start;
  const int m0 = (local / P.tiles_n) * BM, n0 = (local % P.tiles_n) * BN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 1) * Cfg::WM, wn = (warp & 1) * Cfg::WN;
  const int g = lane >> 2, t4 = lane & 3;

  double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = (P.K + BK - 1) / BK;

  auto load = [&](int stage, int k0) {
    // A tile: op(A)[m0 .. m0+BM) x [k0 .. k0+BK)
    if (!P.transA) {
      for (int e = tid; e < BM * BK; e += 128) {
        int mm = e % BM, kk = e / BM;
        int gm = m0 + mm, gk = k0 + kk;
        bool v = gm < P.M && gk < P.K;
        const double* src = v ? P.A + gm + (long long)gk * P.lda : P.A;
        cp_async8(&As[stage][kk * SA + mm], src, v);
      }
    } else {
      for (int e = tid; e < BM * BK; e += 128) {
        int kk = e % BK, mm = e / BK;
        int gm = m0 + mm, gk = k0 + kk;
        bool v = gm < P.M && gk < P.K;
        const double* src = v ? P.A + gk + (long long)gm * P.lda : P.A;
        cp_async8(&As[stage][kk * SA + mm], src, v);
      }
    }
    // B tile: op(B)[k0 .. k0+BK) x [n0 .. n0+BN)
    if (!P.transB) {
      for (int e = tid; e < BK * BN; e += 128) {
        int kk = e % BK, nn = e / BK;
        int gk = k0 + kk, gn = n0 + nn;
        bool v = gk < P.K && gn < P.N;
        const double* src = v ? P.B + gk + (long long)gn * P.ldb : P.B;
        cp_async8(&Bs[stage][kk * SB + nn], src, v);
      }
    } else {
      for (int e = tid; e < BK * BN; e += 128) {
        int nn = e % BN, kk = e / BN;
        int gk = k0 + kk, gn = n0 + nn;
        bool v = gk < P.K && gn < P.N;
        const double* src = v ? P.B + gn + (long long)gk * P.ldb : P.B;
        cp_async8(&Bs[stage][kk * SB + nn], src, v);
      }
    }
    cp_async_commit();
  };

  if (nk > 0) load(0, 0);
  for (int kt = 0; kt < nk; ++kt) {
    const int cur = kt & 1;
    if (kt + 1 < nk) {
      load(cur ^ 1, (kt + 1) * BK);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* as = As[cur];
    const double* bs = Bs[cur];
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double af[Cfg::FM], bf[Cfg::FN];
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i) af[i] = as[(ks + t4) * SA + wm + i * 8 + g];
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j) bf[j] = bs[(ks + t4) * SB + wn + j * 8 + g];
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }

  // epilogue: C = alpha*acc + beta*C
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int gm = m0 + wm + i * 8 + g;
        int gn = n0 + wn + j * 8 + 2 * t4 + h;
        if (gm < P.M && gn < P.N) {
          double* c = P.C + gm + (long long)gn * P.ldc;
          double v = P.alpha * acc[i][j][h];
          if (P.beta != 0.0) v += P.beta * *c;
          *c = v;
        }
      }
}

}  // namespace tlrg
