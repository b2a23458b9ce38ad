// Dev microbenchmark: FP64 latency / throughput of scalar ops on this GPU.
#include <cstdio>
__global__ void lat(double* out, long long* cyc, double x0, int n) {
  double x = x0, y = 1.0000001;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-9);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = x / (y + x * 1e-12);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 1.0);
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x + 1.0);
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1e-9;
  long long t5 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
__global__ void thr(double* out, long long* cyc, int n) {
  double a[8];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x + k;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], 1.0000001, 1e-9);
  long long t1 = clock64();
  double s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[5] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1 << 24); cudaMalloc(&c, 64);
  const int n = 4096;
  lat<<<1, 32>>>(o, c, 1.0, n);
  long long h[6]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
  printf("dependent latency (cycles/op): dfma %.1f  ddiv %.1f  dsqrt %.1f  drsqrt %.1f  shfl64+add %.1f\n",
         (double)h[0] / n, (double)h[1] / n, (double)h[2] / n, (double)h[3] / n, (double)h[4] / n);
  for (int threads : {256, 1024}) {
    thr<<<148, threads>>>(o, c, n);
    cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
    double fma_per_clk_sm = (double)threads * 8 * n / h[5];
    printf("throughput %d threads/SM: %.1f DFMA/clk/SM (%s)\n", threads, fma_per_clk_sm, cudaGetErrorString(cudaGetLastError()));
  }
}
