// Grouped FP64 DMMA GEMM launcher and the argument-table arena.
#include <algorithm>
#include <cstring>
#include <vector>

#include "kernels.h"

namespace tlrg {

namespace {
struct Retired {
  char* h;
  char* d;
};
std::vector<Retired>& retired() {
  static std::vector<Retired> r;
  return r;
}
}  // namespace

void DescArena::reserve(size_t bytes) {
  if (bytes <= cap) return;
  if (h) retired().push_back({h, d});  // freed at the next reset-safe point
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
    if (h) retired().push_back({h, d});
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
  if (h) cudaFreeHost(h);
  if (d) cudaFree(d);
}

void release_retired_arenas() {
  for (auto& r : retired()) {
    cudaFreeHost(r.h);
    cudaFree(r.d);
  }
  retired().clear();
}

template <int BM, int BN>
static void launch_grouped(std::vector<GemmProblem>& probs, DescArena& desc, cudaStream_t st) {
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
  if (tiles == 0) return;
  if (tiles > 0x7fffffffLL) throw std::runtime_error("grouped_gemm: too many tiles");
  auto* d = (const GemmProblem*)desc.push(live.data(), live.size() * sizeof(GemmProblem), st);
  grouped_gemm_kernel<BM, BN><<<(unsigned)tiles, 128, 0, st>>>(d, (int)live.size());
  TLRG_CUDA(cudaGetLastError());
}

void grouped_gemm(std::vector<GemmProblem>& probs, DescArena& desc, cudaStream_t st) {
  int maxN = 0;
  for (auto& p : probs)
    if (p.M > 0) maxN = std::max(maxN, p.N);
  if (maxN <= 16)
    launch_grouped<64, 16>(probs, desc, st);
  else
    launch_grouped<64, 32>(probs, desc, st);
}

}  // namespace tlrg
