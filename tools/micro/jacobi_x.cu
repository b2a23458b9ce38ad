#include <cstdio>
#include <vector>
#include <random>
#include "kernels.h"
using namespace tlrg;
constexpr int JT = 1024;

__global__ void __launch_bounds__(JT) jacobi_x(SvdTask* tasks, int staged, long long* tm) {
  long long c0 = clock64(), cdot = 0, crot = 0, cbar = 0; int nsw = 0;
  extern __shared__ double jsm[];
  SvdTask& T = tasks[blockIdx.x];
  const int n = T.n, m = T.m > 0 ? T.m : T.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = JT / 32;
  if (n == 0) {
    if (tid == 0) *T.rank_out = 0;
    return;
  }
  double* A = staged ? jsm : T.work;       // m x n
  double* V = A + (long long)m * n;        // n x n
  for (long long e = tid; e < (long long)m * n; e += JT) A[e] = T.A[e];
  for (long long e = tid; e < (long long)n * n; e += JT) V[e] = (e % n == e / n) ? 1.0 : 0.0;
  __shared__ int rotated;
  __shared__ double s_tiny;
  {
    __shared__ double red[32];
    double f = 0.0;
    for (long long e = tid; e < (long long)m * n; e += JT) f += A[e] * A[e];
    f = block_sum(f, red);
    if (tid == 0) s_tiny = f * 1e-34;  // (1e-17 ||A||_F)^2: below rounding of any column
  }
  __syncthreads();
  const double tiny2 = s_tiny;
  // rotation threshold: rounding level of an m-term dot product (dgesvj style)
  // rotation threshold: rounding level of an m-term dot product (m eps); a
  // stricter one only makes the final sweeps chase rounding noise
  const double tol = fmax(1e-15, (double)m * 2.220446049250313e-16);
  const int nn = n + (n & 1);
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    ++nsw;
    for (int step = 0; step < nn - 1; ++step) {
      long long s0 = clock64();
      for (int pi = warp; pi < nn / 2; pi += nw) {
        int p = (step + pi) % (nn - 1);
        int q = pi == 0 ? nn - 1 : (step - pi + nn - 1) % (nn - 1);
        if (p >= n || q >= n) continue;
        double* ap = A + (long long)p * m;
        double* aq = A + (long long)q * m;
        double al = 0, be = 0, ga = 0;
        for (int r = lane; r < m; r += 32) {
          al += ap[r] * ap[r];
          be += aq[r] * aq[r];
          ga += ap[r] * aq[r];
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (threadIdx.x == 0) cdot += clock64() - s0;
        if (al > tiny2 && be > tiny2 && ga * ga > tol * tol * (al * be)) {
          // t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = (be - al) / (2 ga),
          // rewritten with one sqrt, one division and one rsqrt
          const double dl = be - al;
          double t = (dl >= 0 ? 2.0 * ga : -2.0 * ga) / (fabs(dl) + sqrt(dl * dl + 4.0 * ga * ga));
          double c = rsqrt(1.0 + t * t), s = c * t;
          for (int r = lane; r < m; r += 32) {
            double x = ap[r], y = aq[r];
            ap[r] = c * x - s * y;
            aq[r] = s * x + c * y;
          }
          double* vp = V + (long long)p * n;
          double* vq = V + (long long)q * n;
          for (int r = lane; r < n; r += 32) {
            double x = vp[r], y = vq[r];
            vp[r] = c * x - s * y;
            vq[r] = s * x + c * y;
          }
          if (lane == 0) rotated = 1;
        }
      }
      long long s1 = clock64();
      __syncthreads();
      if (threadIdx.x == 0) { crot += s1 - s0; cbar += clock64() - s1; }
    }
    if (!rotated) break;
    __syncthreads();
  }
  // singular values = column norms of A
  for (int p = warp; p < n; p += nw) {
    double s = 0.0;
    for (int r = lane; r < m; r += 32) s += A[(long long)p * m + r] * A[(long long)p * m + r];
    s = warp_sum(s);
    if (lane == 0) T.sig[p] = sqrt(s);
  }
  __syncthreads();
  __shared__ int cnt;
  if (tid == 0) cnt = 0;
  __syncthreads();
  for (int p = warp; p < n; p += nw) {
    double sp = T.sig[p];
    int rk = 0;
    for (int q = lane; q < n; q += 32) {
      double sq = T.sig[q];
      rk += (sq > sp || (sq == sp && q < p)) ? 1 : 0;
    }
    rk = warp_sum_int(rk);
    if (lane == 0 && sp > T.cut) atomicAdd(&cnt, 1);
    for (int r = lane; r < m; r += 32) T.A[(long long)rk * m + r] = A[(long long)p * m + r];
    for (int r = lane; r < n; r += 32) T.V[(long long)rk * n + r] = V[(long long)p * n + r];
  }
  __syncthreads();
  // sigma in descending order
  for (int p = warp; p < n; p += nw) {
    double s = 0.0;
    for (int r = lane; r < m; r += 32) s += T.A[(long long)p * m + r] * T.A[(long long)p * m + r];
    s = warp_sum(s);
    if (lane == 0) T.sig[p] = sqrt(s);
  }
  if (tid == 0) *T.rank_out = cnt;
  if (tid == 0) { tm[0] = nsw; tm[1] = cdot; tm[2] = crot; tm[3] = cbar; tm[4] = clock64() - c0; }
}


int main() {
  for (int p : {32, 48, 64}) {
    std::mt19937_64 g(p); std::normal_distribution<double> nd;
    std::vector<double> X(p * 2 * p), G(p * p);
    for (auto& x : X) x = nd(g);
    for (int i = 0; i < p; ++i) for (int j = 0; j < p; ++j) { double s = 0; for (int k = 0; k < 2 * p; ++k) s += X[i + k * p] * X[j + k * p]; G[i + j * p] = s; }
    double *dG, *dV, *dS, *dW; int* rk; long long* tm;
    cudaMalloc(&dG, 8 * p * p); cudaMalloc(&dV, 8 * p * p); cudaMalloc(&dS, 8 * p); cudaMalloc(&dW, 16 * p * p); cudaMalloc(&rk, 4); cudaMalloc(&tm, 64);
    SvdTask t{}; t.A = dG; t.V = dV; t.sig = dS; t.work = dW; t.rank_out = rk; t.n = p; t.cut = 1e-2;
    SvdTask* dt; cudaMalloc(&dt, sizeof t); cudaMemcpy(dt, &t, sizeof t, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(jacobi_x, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemcpy(dG, G.data(), 8 * p * p, cudaMemcpyHostToDevice);
      jacobi_x<<<1, JT, 2 * p * p * 8>>>(dt, 1, tm);
      long long h[5]; cudaMemcpy(h, tm, 40, cudaMemcpyDeviceToHost);
      printf("p=%d sweeps %lld dot %lld rot %lld bar %lld total %lld kcyc (%s)\n", p, h[0], h[1] / 1000, h[2] / 1000, h[3] / 1000, h[4] / 1000, cudaGetErrorString(cudaGetLastError()));
    }
  }
}
