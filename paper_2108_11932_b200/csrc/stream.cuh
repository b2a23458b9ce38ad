// Per-tile gaussian stream helpers shared by the ARA kernels (device code).
// Ring buffers: absolute stream position p lives at buf[s*cap + p % cap];
// avail / cursor are absolute counts with avail - cursor <= cap.
#pragma once
#include "kernels.h"

namespace tlrg {

constexpr int RCH = 1024;    // accepted pairs staged per chunk

struct GenSmem {
  uint64_t mt[MT_N];
  double pu[RCH], pv[RCH], ps[RCH];
  int idx, chunk;
};

// CTA-cooperative: append values to slot s from `have` up to `target` (even).
__device__ inline void cta_generate(GaussStreams& G, int s, long long have, long long target, GenSmem& S) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  RngState* g = &G.st[s];
  double* buf = G.buf + (long long)s * G.cap;
  for (int i = tid; i < MT_N; i += blockDim.x) S.mt[i] = g->mt[i];
  if (tid == 0) S.idx = g->idx;
  __syncthreads();
  while (have < target) {
    const long long need_pairs = (target - have) / 2;
    if (warp == 0) {
      int chunk = (int)(need_pairs < RCH ? need_pairs : RCH);
      int got = 0, ix = S.idx;
      while (got < chunk) {
        if (ix >= MT_N) {
          warp_mt_twist(S.mt);
          ix = 0;
        }
        int n_att = (MT_N - ix) / 2;
        if (n_att > 32) n_att = 32;
        bool acc = false;
        double u = 0, v = 0, q = 0;
        if (lane < n_att) {
          u = 2.0 * mt_uniform(mt_temper(S.mt[ix + 2 * lane])) - 1.0;
          v = 2.0 * mt_uniform(mt_temper(S.mt[ix + 2 * lane + 1])) - 1.0;
          q = u * u + v * v;
          acc = (q < 1.0) && (q != 0.0);
        }
        unsigned mask = __ballot_sync(0xffffffffu, acc);
        int rank = __popc(mask & ((1u << lane) - 1u));
        int nacc = __popc(mask), left = chunk - got;
        if (acc && rank < left) {
          S.pu[got + rank] = u;
          S.pv[got + rank] = v;
          S.ps[got + rank] = q;
        }
        if (nacc >= left) {
          unsigned m2 = mask;
          for (int t = 0; t < left - 1; ++t) m2 &= m2 - 1;
          ix += 2 * __ffs(m2);
          got = chunk;
        } else {
          ix += 2 * n_att;
          got += nacc;
        }
      }
      if (lane == 0) {
        S.idx = ix;
        S.chunk = chunk;
      }
    }
    __syncthreads();
    const int chunk = S.chunk;
    const long long base = have % G.cap;  // even, cap even: a pair never wraps apart
    for (int i = tid; i < chunk; i += blockDim.x) {
      double q = S.ps[i];
      double f = sqrt(-2.0 * log(q) / q);
      long long p0 = base + 2LL * i;
      while (p0 >= G.cap) p0 -= G.cap;
      buf[p0] = S.pu[i] * f;
      buf[p0 + 1] = S.pv[i] * f;
    }
    have += 2LL * chunk;
    __syncthreads();
  }
  for (int i = tid; i < MT_N; i += blockDim.x) g->mt[i] = S.mt[i];
  if (tid == 0) {
    g->idx = S.idx;
    g->have_cached = 0;
    G.avail[s] = have;
  }
  __syncthreads();
}

// dst[0..n) <- src[0..n) with eight loads in flight per thread (the plain
// loop keeps one: without restrict the store may alias the next load)
__device__ __forceinline__ void copy_span(const double* __restrict__ src,
                                          double* __restrict__ dst, long long n, int nthreads) {
  constexpr int U = 8;
  long long e = threadIdx.x;
  for (; e + (long long)(U - 1) * nthreads < n; e += (long long)U * nthreads) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = src[e + (long long)u * nthreads];
#pragma unroll
    for (int u = 0; u < U; ++u) dst[e + (long long)u * nthreads] = v[u];
  }
  for (; e < n; e += nthreads) dst[e] = src[e];
}

// dst[0..n) <- ring[(pos + e) mod cap], without a per-element modulo
__device__ __forceinline__ void ring_copy(const double* ring, long long cap, long long pos,
                                          long long n, double* dst, int nthreads) {
  const long long start = pos % cap;
  const long long first = n < cap - start ? n : cap - start;
  copy_span(ring + start, dst, first, nthreads);
  copy_span(ring, dst + first, n - first, nthreads);
}

__device__ __forceinline__ long long ring_target(const GaussStreams& G, long long cur,
                                                 long long want) {
  long long t = want < cur + G.cap ? want : cur + G.cap;
  return t & ~1LL;
}


}  // namespace tlrg
