// Microbenchmark: cost of cooperative grid.sync() and of the chol32 register kernel.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void syncs(int n, int* out) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < n; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = n;
}
__global__ void empty_k() {}
int main() {
  int* d; cudaMalloc(&d, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int grid : {8, 16, 48, 148}) for (int threads : {128, 256}) {
    int n = 1000;
    void* args[] = {&n, &d};
    cudaLaunchCooperativeKernel((void*)syncs, grid, threads, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)syncs, grid, threads, args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("grid %3d x %3d: %.3f us per grid.sync  (%s)\n", grid, threads, ms * 1e3 / n, cudaGetErrorString(cudaGetLastError()));
  }
  cudaEventRecord(a);
  for (int i = 0; i < 1000; ++i) empty_k<<<1, 32>>>();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("empty launch: %.3f us\n", ms);
  int n = 1; void* args[] = {&n, &d};
  cudaEventRecord(a);
  for (int i = 0; i < 100; ++i) cudaLaunchCooperativeKernel((void*)syncs, 48, 256, args, 0, 0);
  cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("coop launch (48x256, 1 sync): %.3f us\n", ms * 10);
  return 0;
}
