// Per-tile Gaussian streams, draw-for-draw identical to the reference's
// tlr::Rng (util.hpp:24-53): std::mt19937_64 -> uniform (0,1] -> Marsaglia
// polar method with a one-value pair cache.
//
// The stream of a tile is modelled as an infinite sequence of gaussians: every
// accepted polar attempt contributes (u*f, v*f) in that order, so a draw of n
// values simply consumes the next n sequence entries (the cache is the odd
// leftover).  One warp owns one tile stream; the 312-word MT state lives in
// shared memory while the warp works on it and in HBM between kernels.
#pragma once
#include <cstdint>

#include "common.cuh"

namespace tlrg {

constexpr int MT_N = 312, MT_M = 156;
constexpr uint64_t MT_MATRIX_A = 0xB5026F5AA96619E9ULL;
constexpr uint64_t MT_UM = 0xFFFFFFFF80000000ULL, MT_LM = 0x7FFFFFFFULL;

struct RngState {
  uint64_t mt[MT_N];
  int32_t idx;          // next raw word; MT_N means "twist first"
  int32_t have_cached;  // Marsaglia pair cache (util.hpp:33-36)
  double cached;
};

__host__ __device__ inline uint64_t mix64(uint64_t x) {  // util.hpp:10-15
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
__host__ __device__ inline uint64_t tile_seed(uint64_t root, uint64_t phase, uint64_t i,
                                              uint64_t j) {  // util.hpp:17-20
  return mix64(mix64(mix64(root ^ phase) ^ i) ^ j);
}
__host__ __device__ inline uint64_t ara_column_seed(uint64_t root, int i, int k) {
  return tile_seed(root, 0xfac7ULL, (uint64_t)i, (uint64_t)k);  // ara.cpp:19-21
}

__host__ __device__ inline void rng_seed(RngState* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = MT_N;
  s->have_cached = 0;
  s->cached = 0.0;
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}
__device__ __forceinline__ uint64_t mt_twist1(uint64_t cur, uint64_t nxt, uint64_t far) {
  uint64_t y = (cur & MT_UM) | (nxt & MT_LM);
  return far ^ (y >> 1) ^ ((y & 1ULL) ? MT_MATRIX_A : 0ULL);
}

// Warp-cooperative regeneration of the 312-word block held in shared memory.
__device__ __forceinline__ void warp_mt_twist(uint64_t* mt) {
  const int lane = threadIdx.x & 31;
  uint64_t r[5];
  // phase 1: i in [0, 156): reads old mt[i], mt[i+1], mt[i+156]
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    int i = lane + 32 * t;
    if (i < MT_N - MT_M) r[t] = mt_twist1(mt[i], mt[i + 1], mt[i + MT_M]);
  }
  __syncwarp();
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    int i = lane + 32 * t;
    if (i < MT_N - MT_M) mt[i] = r[t];
  }
  __syncwarp();
  // phase 2: i in [156, 311): reads old mt[i], mt[i+1], NEW mt[i-156]
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    int i = MT_N - MT_M + lane + 32 * t;
    if (i < MT_N - 1) r[t] = mt_twist1(mt[i], mt[i + 1], mt[i - (MT_N - MT_M)]);
  }
  __syncwarp();
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    int i = MT_N - MT_M + lane + 32 * t;
    if (i < MT_N - 1) mt[i] = r[t];
  }
  __syncwarp();
  // phase 3: i = 311 reads NEW mt[0] and NEW mt[155]
  if (lane == 0) mt[MT_N - 1] = mt_twist1(mt[MT_N - 1], mt[0], mt[MT_M - 1]);
  __syncwarp();
}

__device__ __forceinline__ double mt_uniform(uint64_t x) {  // util.hpp:28-30
  return ((double)(x >> 11) + 1.0) * 0x1.0p-53;
}

// Draw `count` gaussians from the stream whose state is staged in shared
// memory (`mt`, `idx`, `have_cached`, `cached` are warp-uniform locals kept by
// the caller).  out[p * ostride] receives the p-th value.
__device__ inline void warp_rng_draw(uint64_t* mt, int& idx, int& have_cached, double& cached,
                                     double* out, long long count, long long ostride = 1) {
  const int lane = threadIdx.x & 31;
  long long produced = 0;
  if (count <= 0) return;
  if (have_cached) {
    if (lane == 0) out[0] = cached;
    have_cached = 0;
    produced = 1;
  }
  while (produced < count) {
    if (idx >= MT_N) {
      warp_mt_twist(mt);
      idx = 0;
    }
    int n_att = (MT_N - idx) / 2;
    if (n_att > 32) n_att = 32;
    bool acc = false;
    double g0 = 0.0, g1 = 0.0;
    if (lane < n_att) {
      double u = 2.0 * mt_uniform(mt_temper(mt[idx + 2 * lane])) - 1.0;
      double v = 2.0 * mt_uniform(mt_temper(mt[idx + 2 * lane + 1])) - 1.0;
      double s = u * u + v * v;
      acc = (s < 1.0) && (s != 0.0);
      if (acc) {
        double f = sqrt(-2.0 * log(s) / s);
        g0 = u * f;
        g1 = v * f;
      }
    }
    unsigned mask = __ballot_sync(0xffffffffu, acc);
    int rank = __popc(mask & ((1u << lane) - 1u));
    long long need = count - produced;  // > 0
    // attempts needed: the accepted attempt of rank r covers values 2r, 2r+1
    int need_att = (int)((need + 1) / 2);  // accepted attempts still needed
    int n_acc = __popc(mask);
    if (n_acc >= need_att) {
      // stop at the need_att-th accepted attempt (rank need_att-1)
      unsigned m2 = mask;
      for (int t = 0; t < need_att - 1; ++t) m2 &= m2 - 1;
      int stop_lane = __ffs(m2) - 1;
      if (acc && lane <= stop_lane) {
        long long p0 = produced + 2LL * rank;
        out[p0 * ostride] = g0;
        if (p0 + 1 < count) out[(p0 + 1) * ostride] = g1;
      }
      // cache the unused second value of the last attempt
      double last_g1 = __shfl_sync(0xffffffffu, g1, stop_lane);
      if ((need & 1LL) != 0) {
        have_cached = 1;
        cached = last_g1;
      }
      idx += 2 * (stop_lane + 1);
      produced = count;
    } else {
      if (acc) {
        long long p0 = produced + 2LL * rank;
        out[p0 * ostride] = g0;
        out[(p0 + 1) * ostride] = g1;
      }
      produced += 2LL * n_acc;
      idx += 2 * n_att;
    }
  }
  __syncwarp();
}

// Stage a tile stream into shared memory (warp-cooperative) and back.
__device__ __forceinline__ void warp_rng_load(const RngState* g, uint64_t* mt, int& idx,
                                              int& hc, double& c) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < MT_N; i += 32) mt[i] = g->mt[i];
  idx = g->idx;
  hc = g->have_cached;
  c = g->cached;
  __syncwarp();
}
__device__ __forceinline__ void warp_rng_store(RngState* g, const uint64_t* mt, int idx, int hc,
                                               double c) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  for (int i = lane; i < MT_N; i += 32) g->mt[i] = mt[i];
  if (lane == 0) {
    g->idx = idx;
    g->have_cached = hc;
    g->cached = c;
  }
}

}  // namespace tlrg
