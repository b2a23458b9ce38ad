// Grouped FP64 DMMA GEMM launcher and the argument-table arena.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "kernels.h"

namespace tlrg {


void DescArena::reserve(size_t bytes) {
  if (bytes <= cap) return;
  if (h) retired.push_back({h, d});  // freed at the owner's next reset-safe point
  size_t c = std::max(bytes, (size_t)1 << 20);
  TLRG_CUDA(cudaMallocHost(&h, c));
  TLRG_CUDA(cudaMalloc(&d, c));
  cap = c;
  used = 0;
}

void* DescArena::push(const void* src, size_t bytes, cudaStream_t st) {
  size_t off = (used + 255) & ~(size_t)255;
  if (off + bytes > cap) {
    // Old block may still be read by in-flight kernels: retire it, never free
    // it before the owner synchronises.
    if (h) retired.push_back({h, d});
    size_t c = std::max(2 * cap, bytes + 256);
    c = std::max(c, (size_t)1 << 20);
    TLRG_CUDA(cudaMallocHost(&h, c));
    TLRG_CUDA(cudaMalloc(&d, c));
    cap = c;
    off = 0;
  }
  std::memcpy(h + off, src, bytes);
  TLRG_CUDA(cudaMemcpyAsync(d + off, h + off, bytes, cudaMemcpyHostToDevice, st));
  used = off + bytes;
  return d + off;
}

DescArena::~DescArena() {
  release_retired();
  if (h) cudaFreeHost(h);
  if (d) cudaFree(d);
}

void DescArena::release_retired() {
  for (auto& r : retired) {
    cudaFreeHost(r.h);
    cudaFree(r.d);
  }
  retired.clear();
}

template <int BM, int BN>
static GemmPlan plan_grouped(std::vector<GemmProblem>& probs, DescArena& desc, cudaStream_t st,
                             int big = 0) {
  std::vector<GemmProblem> live;
  live.reserve(probs.size());
  long long tiles = 0;
  for (auto p : probs) {
    if (p.M <= 0 || p.N <= 0) continue;
    p.tiles_n = (p.N + BN - 1) / BN;
    p.tile_start = (int)tiles;
    tiles += (long long)((p.M + BM - 1) / BM) * p.tiles_n;
    live.push_back(p);
  }
  GemmPlan plan;
  plan.bn = BN;
  plan.big = big;
  if (tiles == 0) return plan;
  if (tiles > 0x7fffffffLL) throw std::runtime_error("grouped_gemm: too many tiles");
  std::vector<int> owner((size_t)tiles);
  for (size_t p = 0; p < live.size(); ++p) {
    long long t1 = p + 1 < live.size() ? live[p + 1].tile_start : tiles;
    for (long long t = live[p].tile_start; t < t1; ++t) owner[t] = (int)p;
  }
  plan.d = (const GemmProblem*)desc.push(live.data(), live.size() * sizeof(GemmProblem), st);
  plan.owner = (const int*)desc.push(owner.data(), owner.size() * sizeof(int), st);
  plan.n = (int)live.size();
  plan.tiles = (int)tiles;
  return plan;
}

// the large-tile kernels pay off once every problem of the list is big: a
// ragged list of thin problems keeps the 64-row tiles (better load balance)
static int big_config(const std::vector<GemmProblem>& probs) {
  const char* e = std::getenv("TLRG_GEMM_BIG");  // 0: never use the large tiles (A/B)
  if (e && e[0] == '0') return 0;
  long long work = 0, t64 = 0, t32 = 0;
  int minM = 1 << 30, minN = 1 << 30, maxN = 0;
  for (auto& p : probs) {
    if (p.M <= 0 || p.N <= 0) continue;
    minM = std::min(minM, p.M);
    minN = std::min(minN, p.N);
    maxN = std::max(maxN, p.N);
    work += (long long)p.M * p.N * std::max(p.K, 1);
    t64 += (long long)((p.M + 127) / 128) * ((p.N + 63) / 64);
    t32 += (long long)((p.M + 127) / 128) * ((p.N + 31) / 32);
  }
  // large tiles only with about a wave of them (148 SMs): fewer CTAs than that
  // leave SMs idle and the 64 x 32 kernel wins
  if (work < (1LL << 24) || minM < 128) return 0;
  if (minN >= 64 && t64 >= 120) return 1;
  // the 128 x 32 tiles lost to the 64 x 32 kernel on the bs = 32 round lists once
  // the long reductions were split (cfg3 3.43 -> 3.22 s, cfg4 14.39 -> 13.60 s,
  // measured A/B on one box): opt-in only (TLRG_GEMM_BIG32=1)
  const char* e32 = std::getenv("TLRG_GEMM_BIG32");
  if (maxN <= 32 && minN >= 24 && t32 >= 120 && e32 && e32[0] == '1') return 2;
  return 0;
}

static GemmPlan plan_small(std::vector<GemmProblem>& probs, DescArena& desc, cudaStream_t st) {
  int maxN = 0;
  for (auto& p : probs)
    if (p.M > 0) maxN = std::max(maxN, p.N);
  return maxN <= 16 ? plan_grouped<64, 16>(probs, desc, st) : plan_grouped<64, 32>(probs, desc, st);
}

GemmPlan gemm_plan(std::vector<GemmProblem>& probs, DescArena& desc, cudaStream_t st) {
  const int big = big_config(probs);
  if (big == 1) return plan_grouped<128, 64>(probs, desc, st, 1);
  if (big == 2) return plan_grouped<128, 32>(probs, desc, st, 2);
  // mixed list: split off the large problems when they alone make a wave
  std::vector<GemmProblem> large, small;
  for (auto& p : probs) {
    if (p.M <= 0 || p.N <= 0) continue;
    (p.M >= 128 && p.N >= 24 ? large : small).push_back(p);
  }
  if (!large.empty() && !small.empty()) {
    const int bl = big_config(large);
    if (bl) {
      GemmPlan P = bl == 1 ? plan_grouped<128, 64>(large, desc, st, 1)
                           : plan_grouped<128, 32>(large, desc, st, 2);
      P.rest = std::make_shared<GemmPlan>(plan_small(small, desc, st));
      return P;
    }
  }
  return plan_small(probs, desc, st);
}

template <int BM, int BN, int WGM, int WGN, int ST, int BK = 16>
static void launch_big(const GemmPlan& p, cudaStream_t st) {
  constexpr size_t bytes = (size_t)ST * BK * ((BM + 4) + (BN + 4)) * sizeof(double);
  static size_t lim = enable_max_dyn_smem(grouped_gemm_big_kernel<BM, BN, WGM, WGN, ST, BK>);
  (void)lim;
  grouped_gemm_big_kernel<BM, BN, WGM, WGN, ST, BK>
      <<<(unsigned)p.tiles, 32 * WGM * WGN, bytes, st>>>(p.d, p.owner);
}

void gemm_launch(const GemmPlan& p, cudaStream_t st) {
  if (p.rest) gemm_launch(*p.rest, st);
  if (p.tiles == 0) return;
  // (BK = 32 / 4 stages and 2 x 2 warps of 64 x 32 were measured: within 10 %,
  // better only on 4096^3, worse on the cfg4 SYRK shapes)
  if (p.big == 1)
    launch_big<128, 64, 4, 2, 3>(p, st);
  else if (p.big == 2)
    launch_big<128, 32, 4, 1, 3>(p, st);
  else if (p.bn == 16)
    grouped_gemm_kernel<64, 16><<<(unsigned)p.tiles, 128, 0, st>>>(p.d, p.owner);
  else
    grouped_gemm_kernel<64, 32><<<(unsigned)p.tiles, 128, 0, st>>>(p.d, p.owner);
  TLRG_CUDA(cudaGetLastError());
}

void grouped_gemm(std::vector<GemmProblem>& probs, DescArena& desc, cudaStream_t st) {
  gemm_launch(gemm_plan(probs, desc, st), st);
}

}  // namespace tlrg
