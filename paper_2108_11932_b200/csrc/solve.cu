// Solve-side operators on the device (K17/K18 of SURVEY.md 2.3):
//   tlr_matvec (tlr_matrix.cpp:182-227), factor_apply (solve.cpp:157-214),
//   factor_solve = tile sweeps (solve.cpp:69-155), dot / nrm2 helpers.
// All reductions use a fixed order (no atomics), so results are deterministic.
#include <algorithm>
#include <cmath>

#include "core.h"

namespace tlrg {

namespace {

// out[woff + c] = sum_r A[r + c*rows] * x[xoff + r] for c < rank   (CTA per item)
struct DotItem {
  const double* A;
  long long woff, xoff;
  int rows, rank;
};
__global__ void __launch_bounds__(256) tile_dots_kernel(const DotItem* items, const double* x,
                                                        double* w) {
  const DotItem& D = items[blockIdx.x];
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = warp; c < D.rank; c += 8) {
    const double* a = D.A + (long long)c * D.rows;
    double s = 0.0;
    for (int r = lane; r < D.rows; r += 32) s += a[r] * x[D.xoff + r];
    s = warp_sum(s);
    if (lane == 0) w[D.woff + c] = s;
  }
}

// One CTA per block row: y_i = [P_out](diag-term) + sum_contrib P[r,c] w[c]
struct RowItem {
  const double* diag;  // rows x rows (ld rows) or null
  const int* in_perm;  // gather x through perm (or null)
  const int* out_perm; // scatter the diag term through perm (or null)
  long long yoff;
  int rows, diag_trans;
  int c_begin, c_end;  // range in the contribution list
};
struct Contrib {
  const double* P;  // rows x rank
  long long woff;
  int rank;
};
__global__ void __launch_bounds__(256) block_rows_kernel(const RowItem* items, const Contrib* cl,
                                                         const double* x, const double* w,
                                                         double* y, int accumulate) {
  extern __shared__ double sm[];
  const RowItem& R = items[blockIdx.x];
  double* xin = sm;
  double* val = sm + R.rows;
  const int n = R.rows;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    xin[r] = R.diag ? x[R.yoff + (R.in_perm ? R.in_perm[r] : r)] : 0.0;
    val[r] = 0.0;
  }
  __syncthreads();
  if (R.diag) {
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
      double s = 0.0;
      if (!R.diag_trans)
        for (int c = 0; c < n; ++c) s += R.diag[r + (long long)c * n] * xin[c];
      else
        for (int c = 0; c < n; ++c) s += R.diag[c + (long long)r * n] * xin[c];
      val[R.out_perm ? R.out_perm[r] : r] = s;
    }
  }
  __syncthreads();
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    double s = val[r];
    for (int t = R.c_begin; t < R.c_end; ++t) {
      const Contrib& C = cl[t];
      for (int c = 0; c < C.rank; ++c) s += C.P[r + (long long)c * n] * w[C.woff + c];
    }
    if (accumulate) y[R.yoff + r] += s;
    else y[R.yoff + r] = s;
  }
}

__global__ void bd_vec_kernel(const double* d, const double* e, const uint8_t* s2, int b, int nb,
                              long long n, double* x, int solve) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nb) return;
  long long rem = n - (long long)k * b;
  int rows = (int)(rem < b ? rem : b);
  const double* dk = d + (long long)k * b;
  const double* ek = e + (long long)k * b;
  const uint8_t* sk = s2 + (long long)k * b;
  double* xk = x + (long long)k * b;
  int i = 0;
  while (i < rows) {
    if (sk[i]) {
      double a = xk[i], c = xk[i + 1];
      if (!solve) {
        xk[i] = dk[i] * a + ek[i] * c;
        xk[i + 1] = ek[i] * a + dk[i + 1] * c;
      } else {
        double det = dk[i] * dk[i + 1] - ek[i] * ek[i];
        xk[i] = (dk[i + 1] * a - ek[i] * c) / det;
        xk[i + 1] = (dk[i] * c - ek[i] * a) / det;
      }
      i += 2;
    } else {
      xk[i] = solve ? xk[i] / dk[i] : xk[i] * dk[i];
      i += 1;
    }
  }
}

// forward/backward substitution on one diagonal tile (single CTA, x in smem)
__global__ void __launch_bounds__(256) trsv_tile_kernel(const double* L, int n, double* x,
                                                        const int* perm, int unit, int trans) {
  extern __shared__ double xs[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int r = tid; r < n; r += 256) xs[r] = (perm && !trans) ? x[perm[r]] : x[r];
  __syncthreads();
  if (!trans) {
    for (int p0 = 0; p0 < n; p0 += 32) {
      int pw = min(32, n - p0);
      if (warp == 0) {
        double xi = lane < pw ? xs[p0 + lane] : 0.0;
        for (int j = 0; j < pw; ++j) {
          double xj = __shfl_sync(0xffffffffu, xi, j);
          if (!unit) xj /= L[(p0 + j) + (long long)(p0 + j) * n];
          if (lane == j) xi = xj;
          if (lane > j && lane < pw) xi -= L[(p0 + lane) + (long long)(p0 + j) * n] * xj;
        }
        if (lane < pw) xs[p0 + lane] = xi;
      }
      __syncthreads();
      for (int r = p0 + pw + tid; r < n; r += 256) {
        double s = 0.0;
        for (int c = 0; c < pw; ++c) s += L[r + (long long)(p0 + c) * n] * xs[p0 + c];
        xs[r] -= s;
      }
      __syncthreads();
    }
  } else {
    // solve L^T x = y  (backward)
    int nblk = (n + 31) / 32;
    for (int bi = nblk - 1; bi >= 0; --bi) {
      int p0 = bi * 32, pw = min(32, n - p0);
      // x_p -= L[p0+pw:, p]^T x[p0+pw:]
      for (int c = warp; c < pw; c += 8) {
        double s = 0.0;
        for (int r = p0 + pw + lane; r < n; r += 32) s += L[r + (long long)(p0 + c) * n] * xs[r];
        s = warp_sum(s);
        if (lane == 0) xs[p0 + c] -= s;
      }
      __syncthreads();
      if (warp == 0) {
        double xi = lane < pw ? xs[p0 + lane] : 0.0;
        for (int j = pw - 1; j >= 0; --j) {
          double xj = __shfl_sync(0xffffffffu, xi, j);
          if (!unit) xj /= L[(p0 + j) + (long long)(p0 + j) * n];
          if (lane == j) xi = xj;
          if (lane < j) xi -= L[(p0 + j) + (long long)(p0 + lane) * n] * xj;
        }
        if (lane < pw) xs[p0 + lane] = xi;
      }
      __syncthreads();
    }
  }
  for (int r = tid; r < n; r += 256) {
    if (perm && trans) x[perm[r]] = xs[r];
    else x[r] = xs[r];
  }
}

// x_i -= U_ik (V_ik^T x_k) for the listed tiles (CTA per tile)
struct UpdItem {
  const double* U;
  const double* V;
  long long xi_off, xk_off;
  int rows_i, rows_k, rank;
};
__global__ void __launch_bounds__(256) lower_update_kernel(const UpdItem* items, double* x) {
  __shared__ double w[1024];
  const UpdItem& I = items[blockIdx.x];
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = warp; c < I.rank; c += 8) {
    double s = 0.0;
    for (int r = lane; r < I.rows_k; r += 32) s += I.V[r + (long long)c * I.rows_k] * x[I.xk_off + r];
    s = warp_sum(s);
    if (lane == 0) w[c] = s;
  }
  __syncthreads();
  for (int r = threadIdx.x; r < I.rows_i; r += 256) {
    double s = 0.0;
    for (int c = 0; c < I.rank; ++c) s += I.U[r + (long long)c * I.rows_i] * w[c];
    x[I.xi_off + r] -= s;
  }
}

// x_k -= sum_{i>k} V_ik (U_ik^T x_i), fixed i order (single CTA)
__global__ void __launch_bounds__(256) upper_gather_kernel(const UpdItem* items, int nitems,
                                                           double* x, int rows_k, long long xk_off) {
  __shared__ double w[1024];
  extern __shared__ double acc[];
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = threadIdx.x; r < rows_k; r += 256) acc[r] = 0.0;
  for (int t = 0; t < nitems; ++t) {
    const UpdItem& I = items[t];
    __syncthreads();
    for (int c = warp; c < I.rank; c += 8) {
      double s = 0.0;
      for (int r = lane; r < I.rows_i; r += 32)
        s += I.U[r + (long long)c * I.rows_i] * x[I.xi_off + r];
      s = warp_sum(s);
      if (lane == 0) w[c] = s;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < rows_k; r += 256) {
      double s = 0.0;
      for (int c = 0; c < I.rank; ++c) s += I.V[r + (long long)c * rows_k] * w[c];
      acc[r] += s;
    }
  }
  __syncthreads();
  for (int r = threadIdx.x; r < rows_k; r += 256) x[xk_off + r] -= acc[r];
}

__global__ void dot_partial_kernel(const double* a, const double* b, long long n, double* part) {
  __shared__ double red[32];
  double s = 0.0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x)
    s += a[t] * b[t];
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__global__ void sum_kernel(const double* part, int n, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += part[i];
    *out = s;
  }
}

void launch_block_rows(Ctx& C, const std::vector<RowItem>& rows,
                       const std::vector<Contrib>& cl, const double* x, const double* w,
                       double* y, int b, int accumulate) {
  if (rows.empty()) return;
  RowItem* dr = C.push(rows);
  Contrib* dc = cl.empty() ? nullptr : C.push(cl);
  block_rows_kernel<<<(unsigned)rows.size(), 256, 2 * b * sizeof(double), C.st>>>(
      dr, dc, x, w, y, accumulate);
  TLRG_CUDA(cudaGetLastError());
  ++C.launches;
}

void launch_dots(Ctx& C, const std::vector<DotItem>& it, const double* x, double* w) {
  if (it.empty()) return;
  tile_dots_kernel<<<(unsigned)it.size(), 256, 0, C.st>>>(C.push(it), x, w);
  TLRG_CUDA(cudaGetLastError());
  ++C.launches;
}

}  // namespace

namespace {
__global__ void axpby_kernel(double a, const double* x, double b, double* y, long long n) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x)
    y[t] = (a != 0.0 ? a * x[t] : 0.0) + b * y[t];
}
}  // namespace

void axpby_device(Ctx& C, double a, const double* x, double b, double* y, long long n) {
  int blocks = (int)std::min<long long>((n + 255) / 256, 148 * 8);
  axpby_kernel<<<blocks, 256, 0, C.st>>>(a, x, b, y, n);
  TLRG_CUDA(cudaGetLastError());
}

double dot_device(Ctx& C, const double* a, const double* b, long long n) {
  int blocks = (int)std::min<long long>((n + 255) / 256, 296);
  double* part = C.buf<double>("dot_part", 300);
  double* out = C.buf<double>("dot_out", 1);
  dot_partial_kernel<<<blocks, 256, 0, C.st>>>(a, b, n, part);
  sum_kernel<<<1, 32, 0, C.st>>>(part, blocks, out);
  double* h = C.pinned_dbl(1);
  TLRG_CUDA(cudaMemcpyAsync(h, out, sizeof(double), cudaMemcpyDeviceToHost, C.st));
  C.sync();
  return h[0];
}

namespace {
// ||U V^T||_F^2 = sum_{p,q} (U^T U)_pq (V^T V)_pq, one CTA per low-rank tile,
// one warp per (p <= q) pair, fixed-order reductions
struct FrobItem {
  const double* U;
  const double* V;
  int ru, rv, r;
};
__global__ void __launch_bounds__(256) lowrank_frob_kernel(const FrobItem* items, double* part) {
  const FrobItem it = items[blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ double red[8];
  double acc = 0.0;
  const int npairs = it.r * (it.r + 1) / 2;
  for (int e = warp; e < npairs; e += 8) {
    int q = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
    while (q * (q + 1) / 2 > e) --q;
    while ((q + 1) * (q + 2) / 2 <= e) ++q;
    const int p = e - q * (q + 1) / 2;
    const double* up = it.U + (long long)p * it.ru;
    const double* uq = it.U + (long long)q * it.ru;
    const double* vp = it.V + (long long)p * it.rv;
    const double* vq = it.V + (long long)q * it.rv;
    double gu = 0.0, gv = 0.0;
    for (int i = lane; i < it.ru; i += 32) gu += up[i] * uq[i];
    for (int i = lane; i < it.rv; i += 32) gv += vp[i] * vq[i];
    gu = warp_sum(gu);
    gv = warp_sum(gv);
    acc += (p == q ? 1.0 : 2.0) * gu * gv;
  }
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w];
    part[blockIdx.x] = s;
  }
}
}  // namespace

double frob_norm_device(Ctx& C, const Matrix& A) {
  const int nb = A.nb, b = A.b;
  double* out = C.buf<double>("fn_out", (size_t)nb + 2);
  for (int k = 0; k < nb; ++k) frob_sq(A.diag + (size_t)k * b * b, (long long)A.rows(k) * A.rows(k),
                                       out + k, C.st);
  std::vector<FrobItem> items;
  for (int i = 1; i < nb; ++i)
    for (int j = 0; j < i; ++j) {
      long long t = A.t(i, j);
      if (A.rank[t]) items.push_back({A.U[t], A.V[t], A.rows(i), A.rows(j), A.rank[t]});
    }
  double* part = C.buf<double>("fn_part", items.size() + 1);
  double* lr = out + nb;
  if (!items.empty()) {
    lowrank_frob_kernel<<<(unsigned)items.size(), 256, 0, C.st>>>(C.push(items), part);
    TLRG_CUDA(cudaGetLastError());
    sum_kernel<<<1, 32, 0, C.st>>>(part, (int)items.size(), lr);
  } else {
    fill_zero(lr, 1, C.st);
  }
  C.launches += nb + 2;
  double* h = C.pinned_dbl((size_t)nb + 1);
  TLRG_CUDA(cudaMemcpyAsync(h, out, sizeof(double) * (nb + 1), cudaMemcpyDeviceToHost, C.st));
  C.sync();
  double s = 0.0;
  for (int k = 0; k < nb; ++k) s += h[k];
  return std::sqrt(s + 2.0 * h[nb]);
}

void difference_apply_device(Ctx& C, const Matrix& A, const Factor& F, const double* v, double* w,
                             double* t) {
  if (!F.perm.empty()) {
    // (P A P^T - L L^T) v in the factor frame (solve.cpp:283-297)
    double* pv = C.buf<double>("da_pv", (size_t)A.n);
    tile_perm_device(C, F, v, pv, true);
    matvec_device(C, A, pv, t);
    tile_perm_device(C, F, t, w, false);
  } else {
    matvec_device(C, A, v, w);
  }
  factor_apply_device(C, F, v, t);
  axpby_device(C, -1.0, t, 1.0, w, A.n);  // w = A v - L L^T v
}

// Hutchinson estimate of ||P A P^T - L L^T||_F: probe t
// is the first n draws of tlr::Rng(tile_seed(seed, 0xF20B, t, 0)), E g as the
// reference's difference_apply (solve.cpp:283-297); identical estimator to the
// oracle's ref_estimate_frob_diff, so both sides see the same probes.
double estimate_frob_diff_device(Ctx& C, const Matrix& A, const Factor& F, int probes,
                                 uint64_t seed) {
  const int64_t n = A.n;
  double* g = C.buf<double>("fr_g", (size_t)n);
  double* w = C.buf<double>("fr_w", (size_t)n);
  double* t = C.buf<double>("fr_t", (size_t)n);
  RngState* rs = C.buf<RngState>("fr_rng", 1);
  double acc = 0.0;
  for (int p = 0; p < probes; ++p) {
    std::vector<uint64_t> s1{tile_seed(seed, 0xF20BULL, (uint64_t)p, 0)};
    rng_seed(rs, C.push(s1), 1, C.st);
    rng_draw(rs, nullptr, 1, g, n, n, C.st);
    difference_apply_device(C, A, F, g, w, t);
    acc += dot_device(C, w, w, n);
  }
  return std::sqrt(acc / probes);
}

void matvec_device(Ctx& C, const Matrix& A, const double* x, double* y) {
  const int nb = A.nb, b = A.b;
  std::vector<DotItem> d1, d2;
  std::vector<long long> w1(A.rank.size()), w2(A.rank.size());
  long long wtot = 0;
  for (int i = 1; i < nb; ++i)
    for (int j = 0; j < i; ++j) {
      long long t = A.t(i, j);
      int r = A.rank[t];
      if (!r) continue;
      w1[t] = wtot;
      d1.push_back({A.V[t], wtot, (long long)j * b, A.rows(j), r});  // V^T x_j
      wtot += r;
      w2[t] = wtot;
      d2.push_back({A.U[t], wtot, (long long)i * b, A.rows(i), r});  // U^T x_i
      wtot += r;
    }
  double* w = C.buf<double>("mv_w", (size_t)std::max(wtot, 1LL));
  std::vector<DotItem> all(d1);
  all.insert(all.end(), d2.begin(), d2.end());
  launch_dots(C, all, x, w);
  std::vector<RowItem> rows;
  std::vector<Contrib> cl;
  for (int i = 0; i < nb; ++i) {
    RowItem R{};
    R.diag = A.diag + (size_t)i * b * b;
    R.yoff = (long long)i * b;
    R.rows = A.rows(i);
    R.c_begin = (int)cl.size();
    for (int j = 0; j < i; ++j) {
      long long t = A.t(i, j);
      if (A.rank[t]) cl.push_back({A.U[t], w1[t], A.rank[t]});
    }
    for (int l = i + 1; l < nb; ++l) {
      long long t = A.t(l, i);
      if (A.rank[t]) cl.push_back({A.V[t], w2[t], A.rank[t]});
    }
    R.c_end = (int)cl.size();
    rows.push_back(R);
  }
  launch_block_rows(C, rows, cl, x, w, y, b, 0);
}

void factor_apply_device(Ctx& C, const Factor& F, const double* x, double* y) {
  const Matrix& L = *F.L;
  const int nb = L.nb, b = L.b;
  const bool ldl = F.mode == 1;
  double* t = C.buf<double>("fa_t", (size_t)L.n);
  // t = L^T x :  t_k = L_kk^T (P x_k) + sum_{i>k} V_ik (U_ik^T x_i)
  std::vector<DotItem> d;
  std::vector<long long> wo(L.rank.size());
  long long wtot = 0;
  for (int i = 1; i < nb; ++i)
    for (int k = 0; k < i; ++k) {
      long long q = L.t(i, k);
      if (!L.rank[q]) continue;
      wo[q] = wtot;
      d.push_back({L.U[q], wtot, (long long)i * b, L.rows(i), L.rank[q]});
      wtot += L.rank[q];
    }
  double* w = C.buf<double>("fa_w", (size_t)std::max(wtot, 1LL));
  launch_dots(C, d, x, w);
  std::vector<RowItem> rows;
  std::vector<Contrib> cl;
  for (int k = 0; k < nb; ++k) {
    RowItem R{};
    R.diag = L.diag + (size_t)k * b * b;
    R.diag_trans = 1;
    R.in_perm = ldl ? F.D.perm + (size_t)k * b : nullptr;
    R.yoff = (long long)k * b;
    R.rows = L.rows(k);
    R.c_begin = (int)cl.size();
    for (int i = k + 1; i < nb; ++i) {
      long long q = L.t(i, k);
      if (L.rank[q]) cl.push_back({L.V[q], wo[q], L.rank[q]});
    }
    R.c_end = (int)cl.size();
    rows.push_back(R);
  }
  launch_block_rows(C, rows, cl, x, w, t, b, 0);
  if (ldl) {
    bd_vec_kernel<<<(nb + 127) / 128, 128, 0, C.st>>>(F.D.d, F.D.e, F.D.s2, b, nb, L.n, t, 0);
    ++C.launches;
  }
  // y = L t :  y_k = P^T(L_kk t_k) + sum_{j<k} U_kj (V_kj^T t_j)
  d.clear();
  wtot = 0;
  for (int k = 1; k < nb; ++k)
    for (int j = 0; j < k; ++j) {
      long long q = L.t(k, j);
      if (!L.rank[q]) continue;
      wo[q] = wtot;
      d.push_back({L.V[q], wtot, (long long)j * b, L.rows(j), L.rank[q]});
      wtot += L.rank[q];
    }
  w = C.buf<double>("fa_w2", (size_t)std::max(wtot, 1LL));
  launch_dots(C, d, t, w);
  rows.clear();
  cl.clear();
  for (int k = 0; k < nb; ++k) {
    RowItem R{};
    R.diag = L.diag + (size_t)k * b * b;
    R.out_perm = ldl ? F.D.perm + (size_t)k * b : nullptr;
    R.yoff = (long long)k * b;
    R.rows = L.rows(k);
    R.c_begin = (int)cl.size();
    for (int j = 0; j < k; ++j) {
      long long q = L.t(k, j);
      if (L.rank[q]) cl.push_back({L.U[q], wo[q], L.rank[q]});
    }
    R.c_end = (int)cl.size();
    rows.push_back(R);
  }
  launch_block_rows(C, rows, cl, t, w, y, b, 0);
}

void factor_solve_device(Ctx& C, const Factor& F, double* x) {
  const Matrix& L = *F.L;
  const int nb = L.nb, b = L.b;
  const bool ldl = F.mode == 1;
  double* xp = nullptr;
  if (!F.perm.empty()) {  // z = P b (solve.cpp:144-155)
    xp = C.buf<double>("solve_perm", (size_t)L.n);
    TLRG_CUDA(cudaMemcpyAsync(xp, x, sizeof(double) * L.n, cudaMemcpyDeviceToDevice, C.st));
    tile_perm_device(C, F, xp, x, false);
  }
  // forward sweep (solve.cpp:69-90)
  for (int k = 0; k < nb; ++k) {
    int rk = L.rows(k);
    const int* perm = ldl ? F.D.perm + (size_t)k * b : nullptr;
    trsv_tile_kernel<<<1, 256, rk * sizeof(double), C.st>>>(L.diag + (size_t)k * b * b, rk,
                                                           x + (long long)k * b, perm, ldl, 0);
    std::vector<UpdItem> it;
    for (int i = k + 1; i < nb; ++i) {
      long long q = L.t(i, k);
      if (!L.rank[q]) continue;
      it.push_back({L.U[q], L.V[q], (long long)i * b, (long long)k * b, L.rows(i), rk, L.rank[q]});
    }
    if (!it.empty()) lower_update_kernel<<<(unsigned)it.size(), 256, 0, C.st>>>(C.push(it), x);
    C.launches += 2;
  }
  if (ldl) {
    bd_vec_kernel<<<(nb + 127) / 128, 128, 0, C.st>>>(F.D.d, F.D.e, F.D.s2, b, nb, L.n, x, 1);
    ++C.launches;
  }
  // backward sweep (solve.cpp:92-120)
  for (int k = nb - 1; k >= 0; --k) {
    int rk = L.rows(k);
    std::vector<UpdItem> it;
    for (int i = k + 1; i < nb; ++i) {
      long long q = L.t(i, k);
      if (!L.rank[q]) continue;
      it.push_back({L.U[q], L.V[q], (long long)i * b, (long long)k * b, L.rows(i), rk, L.rank[q]});
    }
    if (!it.empty())
      upper_gather_kernel<<<1, 256, rk * sizeof(double), C.st>>>(C.push(it), (int)it.size(), x, rk,
                                                                 (long long)k * b);
    const int* perm = ldl ? F.D.perm + (size_t)k * b : nullptr;
    trsv_tile_kernel<<<1, 256, rk * sizeof(double), C.st>>>(L.diag + (size_t)k * b * b, rk,
                                                           x + (long long)k * b, perm, ldl, 1);
    C.launches += 2;
    if ((k & 31) == 0) C.sync();  // bound the argument arena between syncs
  }
  if (xp) {  // x = P^T z
    TLRG_CUDA(cudaMemcpyAsync(xp, x, sizeof(double) * L.n, cudaMemcpyDeviceToDevice, C.st));
    tile_perm_device(C, F, xp, x, true);
  }
  C.sync();
}

// ------------------------------------------------------------- Ctx bits ---
int* Ctx::pinned_ints(size_t n) {
  if (n > h_ints_cap) {
    if (h_ints) cudaFreeHost(h_ints);
    TLRG_CUDA(cudaMallocHost(&h_ints, n * sizeof(int)));
    h_ints_cap = n;
  }
  return h_ints;
}
double* Ctx::pinned_dbl(size_t n) {
  if (n > h_dbl_cap) {
    if (h_dbl) cudaFreeHost(h_dbl);
    TLRG_CUDA(cudaMallocHost(&h_dbl, n * sizeof(double)));
    h_dbl_cap = n;
  }
  return h_dbl;
}
Ctx::~Ctx() {
  ctx_register(this, false);
  if (st_main) cudaStreamSynchronize(st_main);
  chunk_cache_release(this);
  if (h_ints) cudaFreeHost(h_ints);
  if (h_dbl) cudaFreeHost(h_dbl);
  bufs.clear();
  if (st) cudaStreamDestroy(st);
  if (st2) cudaStreamDestroy(st2);
  if (sd) cudaStreamDestroy(sd);
  for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
}
void Matrix::free_all() {
  if (diag) stream_free(ctx, ctx_alive(ctx) ? ctx->st_main : nullptr, diag);
  diag = nullptr;
  stores.clear();
}

}  // namespace tlrg
