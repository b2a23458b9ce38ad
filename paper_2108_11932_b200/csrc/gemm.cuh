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

// ---- large-tile variant: BM x BN x 16, WGM x WGN warps of 32 x (BN/WGN),
// STAGES-deep cp.async pipeline, 16-byte copies where the operand is contiguous
// along the shared tile's fast axis (A not transposed: m; B transposed: n) and
// 16-byte aligned, 8-byte copies otherwise.  Used for problem lists with large
// tiles (the diagonal SYRK D_k = H_k U_k^T, the compensation sketch products at
// m = 1024, the bs = 32 sampling products), where the 64 x 32 kernel's
// per-element copies and 2:1 load:DMMA ratio cap it well below the pipe.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
template <int N>
__device__ __forceinline__ void cp_async_wait_n() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int BM, int BN, int WGM, int WGN, int STAGES, int BK = 16>
__global__ void __launch_bounds__(32 * WGM * WGN) grouped_gemm_big_kernel(
    const GemmProblem* __restrict__ probs, const int* __restrict__ owner) {
  constexpr int NT = 32 * WGM * WGN, SA = BM + 4, SB = BN + 4;
  constexpr int WM = BM / WGM, WN = BN / WGN, FM = WM / 8, FN = WN / 8;
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;                        // STAGES x BK x SA
  double* Bs = gsm + STAGES * BK * SA;     // STAGES x BK x SB
  __shared__ __align__(16) GemmProblem sP;
  __shared__ int s_go;
  {
    const int pidx = owner[blockIdx.x];
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(probs + pidx);
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
  const int wm = (warp / WGN) * WM, wn = (warp % WGN) * WN;
  const int g = lane >> 2, t4 = lane & 3;
  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int nk = (P.K + BK - 1) / BK;
  auto load = [&](int stage, int k0) {
    double* as = As + stage * BK * SA;
    double* bs = Bs + stage * BK * SB;
    if (!P.transA) {
      // pairs (gm, gm + 1) of one k are contiguous in both
      for (int e = tid; e < BM * BK / 2; e += NT) {
        const int mm = 2 * (e % (BM / 2)), kk = e / (BM / 2);
        const int gm = m0 + mm, gk = k0 + kk;
        const double* src = P.A + gm + (long long)gk * P.lda;
        const bool v0 = gm < P.M && gk < P.K, v1 = gm + 1 < P.M && gk < P.K;
        if (v0 && v1 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
          cp_async16(&as[kk * SA + mm], src, 16);
        } else {
          cp_async8(&as[kk * SA + mm], v0 ? src : P.A, v0);
          cp_async8(&as[kk * SA + mm + 1], v1 ? src + 1 : P.A, v1);
        }
      }
    } else {
      for (int e = tid; e < BM * BK; e += NT) {
        const int kk = e % BK, mm = e / BK;
        const int gm = m0 + mm, gk = k0 + kk;
        const bool v = gm < P.M && gk < P.K;
        cp_async8(&as[kk * SA + mm], v ? P.A + gk + (long long)gm * P.lda : P.A, v);
      }
    }
    if (P.transB) {
      for (int e = tid; e < BN * BK / 2; e += NT) {
        const int nn = 2 * (e % (BN / 2)), kk = e / (BN / 2);
        const int gk = k0 + kk, gn = n0 + nn;
        const double* src = P.B + gn + (long long)gk * P.ldb;
        const bool v0 = gk < P.K && gn < P.N, v1 = gk < P.K && gn + 1 < P.N;
        if (v0 && v1 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
          cp_async16(&bs[kk * SB + nn], src, 16);
        } else {
          cp_async8(&bs[kk * SB + nn], v0 ? src : P.B, v0);
          cp_async8(&bs[kk * SB + nn + 1], v1 ? src + 1 : P.B, v1);
        }
      }
    } else {
      for (int e = tid; e < BN * BK; e += NT) {
        const int kk = e % BK, nn = e / BK;
        const int gk = k0 + kk, gn = n0 + nn;
        const bool v = gk < P.K && gn < P.N;
        cp_async8(&bs[kk * SB + nn], v ? P.B + gk + (long long)gn * P.ldb : P.B, v);
      }
    }
  };
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load(s, s * BK);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait_n<STAGES - 2>();
    __syncthreads();
    {
      const int kn = kt + STAGES - 1;
      if (kn < nk) load(kn % STAGES, kn * BK);
      cp_async_commit();
    }
    const double* as = As + (kt % STAGES) * BK * SA;
    const double* bs = Bs + (kt % STAGES) * BK * SB;
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double af[FM], bf[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i) af[i] = as[(ks + t4) * SA + wm + i * 8 + g];
#pragma unroll
      for (int j = 0; j < FN; ++j) bf[j] = bs[(ks + t4) * SB + wn + j * 8 + g];
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait_n<0>();
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gm = m0 + wm + i * 8 + g;
        const int gn = n0 + wn + j * 8 + 2 * t4 + h;
        if (gm < P.M && gn < P.N) {
          double* c = P.C + gm + (long long)gn * P.ldc;
          double v = P.alpha * acc[i][j][h];
          if (P.beta != 0.0) v += P.beta * *c;
          *c = v;
        }
      }
}

}  // namespace tlrg
