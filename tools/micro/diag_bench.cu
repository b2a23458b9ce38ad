// Dev microbenchmark: latency of the diagonal-path kernels on one 512 x 512 tile.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I../../paper_2108_11932_b200/csrc
//        diag_bench.cu -L../../paper_2108_11932_b200/lib -ltlrg -Xlinker -rpath=...
#include <cstdio>
#include <vector>
#include <random>
#include "kernels.h"
using namespace tlrg;
namespace tlrg { void potrf_impl(double* A, int n, int* info, DescArena& desc, cudaStream_t st); }
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
  double *dA, *dW;
  int* info;
  cudaMalloc(&dA, 8 * n * n);
  cudaMalloc(&dW, 8 * n * n);
  cudaMalloc(&info, 16);
  cudaMemcpy(dA, A.data(), 8 * n * n, cudaMemcpyHostToDevice);
  cudaStream_t st;
  cudaStreamCreate(&st);
  DescArena desc;
  desc.reserve(1 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpyAsync(dW, dA, 8 * n * n, cudaMemcpyDeviceToDevice, st);
    cudaEventRecord(a, st);
    potrf_impl(dW, n, info, desc, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    int hi = 0;
    cudaMemcpy(&hi, info, 4, cudaMemcpyDeviceToHost);
    printf("potrf %d: %.1f us (info %d) %s\n", n, ms * 1e3, hi, cudaGetErrorString(cudaGetLastError()));
  }
  // cholqr on a 64 x 64 Gram
  for (int p : {32, 48, 64}) {
    std::vector<double> G((size_t)p * p);
    for (int i = 0; i < p; ++i)
      for (int j = 0; j < p; ++j) G[i + j * p] = A[i + j * n];
    double *dG, *dR;
    cudaMalloc(&dG, 8 * p * p);
    cudaMalloc(&dR, 8 * p * p);
    cudaMemcpy(dG, G.data(), 8 * p * p, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a, st);
      cholqr_factor(dG, p, n, 1, dR, st);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("cholqr p=%d: %.1f us %s\n", p, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
    }
    // jacobi on the p x p Gram (SPD)
    SvdTask t{};
    double *dV, *dS, *dWk;
    int* rk;
    cudaMalloc(&dV, 8 * p * p);
    cudaMalloc(&dS, 8 * p);
    cudaMalloc(&dWk, 16 * p * p);
    cudaMalloc(&rk, 4);
    t.A = dG; t.V = dV; t.sig = dS; t.work = dWk; t.rank_out = rk; t.n = p; t.cut = 1e-2; t.tol = 1e-14;
    SvdTask* dt;
    cudaMalloc(&dt, sizeof(SvdTask));
    cudaMemcpy(dt, &t, sizeof t, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemcpy(dG, G.data(), 8 * p * p, cudaMemcpyHostToDevice);
      cudaEventRecord(a, st);
      if (p <= 64) sym_jacobi(dt, 1, p, st); else jacobi_svd(dt, 1, p, st);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("jacobi p=%d: %.1f us %s\n", p, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
