// Per-tile latency kernels of an ARA round:
//   * rng_draw  : tlr::Rng gaussian blocks.  Warp 0 walks the mt19937_64
//                 stream and the polar accept/reject decisions (integer work,
//                 one ballot per 32 attempts); all warps then evaluate
//                 sqrt(-2 log s / s) for the accepted pairs in parallel.
//   * panel_tau : tau = 100 * eps_mach * ||Y_raw||_F (dense_kernels.cpp:391-392)
//   * panel_mgs : one sweep of the reference's panel MGS2 with deficiency
//                 replacement (dense_kernels.cpp:331-375) + R <- Rp R and the
//                 finalisation of orthog (dense_kernels.cpp:397-417).
//                 Every thread owns a fixed set of rows, so the only
//                 synchronisations are the three block reductions per column
//                 (two re-orthogonalisation passes + the norm).
#include <cfloat>

#include "kernels.h"
#include "stream.cuh"

namespace tlrg {

// ------------------------------------------------------------------ RNG ---
__global__ void rng_seed_kernel(RngState* states, const uint64_t* seeds, int n) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) rng_seed(&states[t], seeds[t]);
}

constexpr int RT = 128;      // threads per draw CTA

__global__ void __launch_bounds__(RT) rng_draw_kernel(RngState* states, const int* idx,
                                                      double* out, long long count,
                                                      long long out_stride) {
  __shared__ uint64_t mt[MT_N];
  __shared__ double pu[RCH], pv[RCH], ps[RCH];
  __shared__ int s_idx, s_hc, s_target;
  __shared__ double s_c;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  RngState* g = &states[idx ? idx[blockIdx.x] : blockIdx.x];
  double* o = out + (long long)blockIdx.x * out_stride;
  for (int i = tid; i < MT_N; i += RT) mt[i] = g->mt[i];
  if (tid == 0) {
    s_idx = g->idx;
    s_hc = g->have_cached;
    s_c = g->cached;
  }
  __syncthreads();
  long long produced = 0;
  if (s_hc && count > 0) {
    if (tid == 0) o[0] = s_c;
    produced = 1;
    __syncthreads();
    if (tid == 0) s_hc = 0;
  }
  while (produced < count) {
    const long long need = count - produced;
    const long long need_att = (need + 1) / 2;
    if (warp == 0) {
      int target = (int)(need_att < RCH ? need_att : RCH);
      int got = 0, ix = s_idx;
      while (got < target) {
        if (ix >= MT_N) {
          warp_mt_twist(mt);
          ix = 0;
        }
        int n_att = (MT_N - ix) / 2;
        if (n_att > 32) n_att = 32;
        bool acc = false;
        double u = 0, v = 0, s = 0;
        if (lane < n_att) {
          u = 2.0 * mt_uniform(mt_temper(mt[ix + 2 * lane])) - 1.0;
          v = 2.0 * mt_uniform(mt_temper(mt[ix + 2 * lane + 1])) - 1.0;
          s = u * u + v * v;
          acc = (s < 1.0) && (s != 0.0);
        }
        unsigned mask = __ballot_sync(0xffffffffu, acc);
        int rank = __popc(mask & ((1u << lane) - 1u));
        int nacc = __popc(mask), left = target - got;
        if (acc && rank < left) {
          pu[got + rank] = u;
          pv[got + rank] = v;
          ps[got + rank] = s;
        }
        if (nacc >= left) {
          unsigned m2 = mask;
          for (int t = 0; t < left - 1; ++t) m2 &= m2 - 1;
          ix += 2 * (__ffs(m2) - 1 + 1);
          got = target;
        } else {
          ix += 2 * n_att;
          got += nacc;
        }
      }
      if (lane == 0) {
        s_idx = ix;
        s_target = target;
      }
    }
    __syncthreads();
    const int target = s_target;
    for (int i = tid; i < target; i += RT) {
      double s = ps[i];
      double f = sqrt(-2.0 * log(s) / s);
      long long p0 = produced + 2LL * i;
      o[p0] = pu[i] * f;
      if (p0 + 1 < count) {
        o[p0 + 1] = pv[i] * f;
      } else {
        s_hc = 1;  // odd tail: cache the second value (util.hpp:43-45)
        s_c = pv[i] * f;
      }
    }
    produced += 2LL * target;
    __syncthreads();
  }
  for (int i = tid; i < MT_N; i += RT) g->mt[i] = mt[i];
  if (tid == 0) {
    g->idx = s_idx;
    g->have_cached = s_hc;
    g->cached = s_c;
  }
}

void rng_seed(RngState* states, const uint64_t* d_seeds, int n, cudaStream_t st) {
  if (n <= 0) return;
  rng_seed_kernel<<<(n + 127) / 128, 128, 0, st>>>(states, d_seeds, n);
  TLRG_CUDA(cudaGetLastError());
}
void rng_draw(RngState* states, const int* d_idx, int ntiles, double* out, long long count,
              long long out_stride, cudaStream_t st) {
  if (ntiles <= 0 || count <= 0) return;
  rng_draw_kernel<<<ntiles, RT, 0, st>>>(states, d_idx, out, count, out_stride);
  TLRG_CUDA(cudaGetLastError());
}

__global__ void __launch_bounds__(RT) gauss_generate_kernel(GaussStreams G, const int* slots,
                                                            const long long* want) {
  __shared__ GenSmem S;
  const int s = slots[blockIdx.x];
  const long long have = G.avail[s];
  const long long target = ring_target(G, G.cursor[s], want[blockIdx.x]);
  if (have >= target) return;
  cta_generate(G, s, have, target, S);
}

__global__ void __launch_bounds__(RT) gauss_round_kernel(GaussStreams G, const int* done,
                                                         const int* rows, int cols, int bs,
                                                         double* Om) {
  __shared__ GenSmem S;
  const int s = blockIdx.x;
  if (done[s]) return;
  const long long need = (long long)cols * bs + 2LL * bs * rows[s];
  const long long chunk = 2LL * cols * bs;
  const long long cur = G.cursor[s], av = G.avail[s];
  if (av - cur < need) cta_generate(G, s, av, ring_target(G, cur, cur + need + chunk), S);
  const double* b = G.buf + (long long)s * G.cap;
  double* dst = Om + (long long)s * cols * bs;
  const long long n = (long long)cols * bs;
  ring_copy(b, G.cap, cur, n, dst, RT);
  __syncthreads();
  if (threadIdx.x == 0) G.cursor[s] = cur + n;
}

// Ring top-up off the round's critical path: generate the slot's stream until
// the ring is full again (ring_target caps at cursor + cap, so only consumed
// positions are overwritten).  Runs concurrently with the round's products and
// panel sweeps, which only read the ring and advance the cursor: a cursor read
// here that is already stale only under-estimates the free space.
__global__ void __launch_bounds__(RT) gauss_topup_kernel(GaussStreams G, const int* done,
                                                         long long low) {
  __shared__ GenSmem S;
  const int s = blockIdx.x;
  if (done[s]) return;
  const long long cur = *reinterpret_cast<volatile long long*>(G.cursor + s), av = G.avail[s];
  if (av - cur >= low) return;
  cta_generate(G, s, av, ring_target(G, cur, cur + G.cap), S);
}

__global__ void __launch_bounds__(256) gauss_gather_kernel(GaussStreams G, const int* slots,
                                                           double* out, long long count,
                                                           long long out_stride) {
  const int s = slots[blockIdx.x];
  const long long c0 = G.cursor[s];
  const double* b = G.buf + (long long)s * G.cap;
  double* dst = out + (long long)blockIdx.x * out_stride;
  ring_copy(b, G.cap, c0, count, dst, 256);
  __syncthreads();
  if (threadIdx.x == 0) G.cursor[s] = c0 + count;
}

void gauss_generate(const GaussStreams& G, const int* d_slots, const long long* d_want, int n,
                    cudaStream_t st) {
  if (n <= 0) return;
  gauss_generate_kernel<<<n, RT, 0, st>>>(G, d_slots, d_want);
  TLRG_CUDA(cudaGetLastError());
}
void gauss_gather(const GaussStreams& G, const int* d_slots, int n, double* out, long long count,
                  long long out_stride, cudaStream_t st) {
  if (n <= 0 || count <= 0) return;
  gauss_gather_kernel<<<n, 256, 0, st>>>(G, d_slots, out, count, out_stride);
  TLRG_CUDA(cudaGetLastError());
}
void gauss_round(const GaussStreams& G, const int* done, const int* rows, int nslots, int cols,
                 int bs, double* Om, cudaStream_t st) {
  if (nslots <= 0) return;
  gauss_round_kernel<<<nslots, RT, 0, st>>>(G, done, rows, cols, bs, Om);
  TLRG_CUDA(cudaGetLastError());
}

void gauss_topup(const GaussStreams& G, const int* done, int nslots, long long low,
                 cudaStream_t st) {
  if (nslots <= 0) return;
  gauss_topup_kernel<<<nslots, RT, 0, st>>>(G, done, low);
  TLRG_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------- PANEL TAU ---
__global__ void __launch_bounds__(256) panel_tau_kernel(PanelTask* tasks) {
  __shared__ double red[32];
  PanelTask& T = tasks[blockIdx.x];
  if (T.done && *T.done) return;
  long long n = (long long)T.rows * T.width;
  double s = 0.0;
  for (long long e = threadIdx.x; e < n; e += 256) s += T.Y[e] * T.Y[e];
  s = block_sum(s, red);
  if (threadIdx.x == 0) {
    double tau = 100.0 * DBL_EPSILON * sqrt(s);
    T.tau = tau == 0.0 ? DBL_MIN : tau;
  }
}
void panel_tau(PanelTask* d_tasks, int ntask, cudaStream_t st) {
  if (ntask <= 0) return;
  panel_tau_kernel<<<ntask, 256, 0, st>>>(d_tasks);
  TLRG_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------- PANEL MGS ---
constexpr int PT = 512;
constexpr int PW = PT / 32;

struct PanelSmem {
  double* part;  // [2][PW][part_len]
  double* cbuf;  // [max(part_len, rows)]
  int cbuf_len;  // = part_len (stride of the partial buffers)
  int buf;
};

// Lane-strided dot product over the panel rows with four independent partial
// sums (summed (a0 + a1) + (a2 + a3)): the per-step dot lists are the column
// sweep's critical path and a single FMA chain serializes on every load.
__device__ __forceinline__ double panel_dot(const double* __restrict__ a,
                                            const double* __restrict__ b, int rows, int lane) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int r = lane;
  for (; r + 96 < rows; r += 128) {
    a0 += a[r] * b[r];
    a1 += a[r + 32] * b[r + 32];
    a2 += a[r + 64] * b[r + 64];
    a3 += a[r + 96] * b[r + 96];
  }
  for (; r < rows; r += 32) a0 += a[r] * b[r];
  return (a0 + a1) + (a2 + a3);
}

// Block-reduce `nv` per-thread partial values (already warp-summed into lane 0)
// -> cbuf[0..nv).  One __syncthreads.
__device__ __forceinline__ void reduce_to(PanelSmem& S, int nv) {
  __syncthreads();
  double* P = S.part + (size_t)S.buf * PW * S.cbuf_len;
  for (int p = threadIdx.x; p < nv; p += PT) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < PW; ++w) s += P[w * S.cbuf_len + p];
    S.cbuf[p] = s;
  }
  S.buf ^= 1;
  __syncthreads();
}

// one classical re-orthogonalisation pass of column j against columns < j;
// coefficients are returned in S.cbuf
__device__ __forceinline__ void cgs_pass(double* Y, int rows, int j, PanelSmem& S) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* yj = Y + (long long)j * rows;
  // warps split the coefficients; each dot runs over all rows (one warp sum)
  __syncthreads();  // y_j (and cbuf readers of the previous pass) are settled
  int p = warp;
  for (; p + PW < j; p += 2 * PW) {
    const double* ya = Y + (long long)p * rows;
    const double* yb = Y + (long long)(p + PW) * rows;
    double sa = 0.0, sb = 0.0;
    for (int r = lane; r < rows; r += 32) {
      double y = yj[r];
      sa += ya[r] * y;
      sb += yb[r] * y;
    }
    sa = warp_sum(sa);
    sb = warp_sum(sb);
    if (lane == 0) {
      S.cbuf[p] = sa;
      S.cbuf[p + PW] = sb;
    }
  }
  if (p < j) {
    const double* ya = Y + (long long)p * rows;
    double sa = 0.0;
    for (int r = lane; r < rows; r += 32) sa += ya[r] * yj[r];
    sa = warp_sum(sa);
    if (lane == 0) S.cbuf[p] = sa;
  }
  __syncthreads();
  // y_j -= sum_p c_p y_p over this thread's rows (independent accumulators per row)
  double* yw = Y + (long long)j * rows;
  constexpr int RPT = 8;
  for (int r0 = 0; r0 < rows; r0 += RPT * PT) {
    double acc[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) acc[u] = 0.0;
    for (int p = 0; p < j; ++p) {
      const double c = S.cbuf[p];
      const double* yp = Y + (long long)p * rows + r0 + threadIdx.x;
#pragma unroll
      for (int u = 0; u < RPT; ++u)
        if (r0 + threadIdx.x + u * PT < rows) acc[u] += c * yp[u * PT];
    }
#pragma unroll
    for (int u = 0; u < RPT; ++u)
      if (r0 + threadIdx.x + u * PT < rows) yw[r0 + threadIdx.x + u * PT] -= acc[u];
  }
}

__device__ __forceinline__ double col_norm(const double* y, int rows, PanelSmem& S) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double s = 0.0;
  for (int r = threadIdx.x; r < rows; r += PT) s += y[r] * y[r];
  s = warp_sum(s);
  if (lane == 0) S.part[(size_t)S.buf * PW * S.cbuf_len + warp * S.cbuf_len] = s;
  reduce_to(S, 1);
  return sqrt(S.cbuf[0]);
}

__global__ void __launch_bounds__(PT) panel_mgs_kernel(PanelTask* tasks, int sweep, int finalize,
                                                       int ys_in_smem, int rp_in_smem,
                                                       int part_len, int cbuf_len) {
  extern __shared__ double smem[];
  PanelSmem S;
  S.part = smem;
  S.cbuf = S.part + 2 * PW * part_len;
  S.cbuf_len = part_len;
  S.buf = 0;
  uint64_t* smt = reinterpret_cast<uint64_t*>(S.cbuf + cbuf_len);
  double* dyn = reinterpret_cast<double*>(smt + MT_N);

  PanelTask& T = tasks[blockIdx.x];
  if (T.done && *T.done) return;
  const int rows = T.rows, w = T.width, q = T.qdev ? *T.qdev : T.q;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* Rp = rp_in_smem ? dyn : T.Rp;
  size_t yoff = rp_in_smem ? (size_t)w * w : 0;
  yoff += (smem_u32(dyn + yoff) & 15) ? 1 : 0;  // 16-byte aligned panel
  double* Y = ys_in_smem ? dyn + yoff : T.Y;
  const unsigned ybytes = (unsigned)((size_t)rows * w * 8);
  const bool bulk = ys_in_smem && (ybytes % 16 == 0) && (((size_t)T.Y & 15) == 0);
  __shared__ __align__(8) uint64_t s_bar;
  if (ys_in_smem) {
    if (bulk) {
      // one TMA bulk copy stages the whole panel (UBLKCP)
      if (tid == 0) {
        mbar_init(&s_bar, 1);
        mbar_arrive_expect_tx(&s_bar, ybytes);
        bulk_g2s(Y, T.Y, ybytes, &s_bar);
      }
      __syncthreads();
      mbar_wait(&s_bar, 0);
    } else {
      for (long long e = tid; e < (long long)rows * w; e += PT) Y[e] = T.Y[e];
    }
  }
  for (long long e = tid; e < (long long)w * w; e += PT) Rp[e] = 0.0;
  if (sweep == 0)
    for (int j = tid; j < w; j += PT) {
      T.deficient[j] = 0;
      T.tiny[j] = 0.0;
    }
  __syncthreads();
  const double tau = T.tau;
  int rep_n = 0, rep_used = 0;  // batch of projected replacement vectors
  long long rep_base = 0;
  __shared__ int s_fast;

  // deficient column j (norm below tau after its two passes): record the first
  // tiny norm, restart from a fresh direction of the tile's own stream, project
  // out Q and the earlier panel columns (dense_kernels.cpp:348-372); returns the
  // norm the column is then divided by
  auto replace_col = [&](int j, double nj) -> double {
    double* yj = Y + (long long)j * rows;
    if (tid == 0 && !T.deficient[j]) {
      T.deficient[j] = 1;
      T.tiny[j] = isfinite(nj) ? nj : 0.0;
    }
    if (rep_used == rep_n) {
      // Project the next (w - j) vectors of the tile's stream against Q in
      // one batch: replacement vector u is stream[c0 + u*rows, ...) with
      // y <- y - Q (Q^T y) (dense_kernels.cpp:351-358); the cursor only
      // advances over the vectors actually consumed.
      __syncthreads();
      const long long c0 = *T.gcursor;
      rep_base = c0;
      rep_used = 0;
      rep_n = w - j;
      __syncthreads();
      ring_copy(T.gbuf, T.gcap, c0, (long long)rows * rep_n, T.rep, PT);
      __syncthreads();
      if (q > 0) {
        for (int pi = warp; pi < q * rep_n; pi += PW) {
          const int t = pi % q, c = pi / q;
          const double* qt = T.Q + (long long)t * rows;
          const double* rc = T.rep + (long long)c * rows;
          double sacc = 0.0;
          for (int r = lane; r < rows; r += 32) sacc += qt[r] * rc[r];
          sacc = warp_sum(sacc);
          if (lane == 0) T.repC[t + (long long)c * q] = sacc;
        }
        __syncthreads();
        // rep -= Q (Q^T rep): each Q element is loaded once per row and
        // applied to up to 16 replacement vectors held in registers
        for (int c0 = 0; c0 < rep_n; c0 += 16) {
          const int nc = min(16, rep_n - c0);
          for (int r = tid; r < rows; r += PT) {
            double acc[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) acc[c] = 0.0;
            for (int t = 0; t < q; ++t) {
              const double qv = T.Q[(long long)t * rows + r];
              const double* rc = T.repC + t + (long long)c0 * q;
#pragma unroll
              for (int c = 0; c < 16; ++c)
                if (c < nc) acc[c] += qv * rc[(long long)c * q];
            }
#pragma unroll
            for (int c = 0; c < 16; ++c)
              if (c < nc) T.rep[r + (long long)(c0 + c) * rows] -= acc[c];
          }
        }
        __syncthreads();
      }
    }
    for (int r = tid; r < rows; r += PT) yj[r] = T.rep[r + (long long)rep_used * rows];
    ++rep_used;
    if (tid == 0) *T.gcursor = rep_base + (long long)rep_used * rows;
    if (j > 0)
      for (int pass = 0; pass < 2; ++pass) cgs_pass(Y, rows, j, S);
    nj = col_norm(yj, rows, S);
    if (nj == 0.0) {
      // pathological: unit coordinate direction, written by the row's owner
      if (tid == (j % rows) % PT) yj[j % rows] = 1.0;
      nj = 1.0;
    }
    if (tid == 0) Rp[j + (long long)j * w] = 0.0;
    return nj;
  };

  // ---- second sweep as one Gram product (see ara_fused.cu sweep2_gram): the
  // panel is orthonormal to O(eps) after sweep 1 and the caller's BGS, so
  // R2 = I + striu(F) + diag(F)/2 with F = Y^T Y - I, and Y <- Y R2^{-1} with
  // R2^{-1} = I - striu(F) - diag(F)/2 (dropped terms O(|F|^2)).  Taken when no
  // column can deflate (tau < 1/4) and |F| <= 1e-6 everywhere; otherwise the
  // column sweep below runs.
  bool gram_done = false;
  if (sweep == 1 && w <= 32 && tau < 0.25) {
    double* F = T.Rp + (long long)w * w;  // w x w scratch (the R-update buffer)
    if (tid == 0) s_fast = 1;
    __syncthreads();
    for (int e = warp; e < w * (w + 1) / 2; e += PW) {
      int jj = (int)((sqrtf(8.0f * e + 1.0f) - 1.0f) * 0.5f);
      while (jj * (jj + 1) / 2 > e) --jj;
      while ((jj + 1) * (jj + 2) / 2 <= e) ++jj;
      const int ii = e - jj * (jj + 1) / 2;
      const double* xa = Y + (long long)ii * rows;
      const double* xb = Y + (long long)jj * rows;
      double sacc = panel_dot(xa, xb, rows, lane);
      sacc = warp_sum(sacc);
      if (lane == 0) {
        const double f = sacc - (ii == jj ? 1.0 : 0.0);
        F[ii + (long long)jj * w] = f;
        if (!(fabs(f) <= 1e-6)) s_fast = 0;
      }
    }
    __syncthreads();
    if (s_fast) {
      for (long long e = tid; e < (long long)w * w; e += PT) {
        const int ii = (int)(e % w), jj = (int)(e / w);
        const double f = ii <= jj ? F[ii + (long long)jj * w] : 0.0;
        Rp[e] = ii < jj ? f : ii == jj ? 1.0 + 0.5 * f : 0.0;
      }
      // y_row <- y_row R2^{-1}, one row per thread
      for (int r = tid; r < rows; r += PT) {
        double yr[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) yr[c] = c < w ? Y[r + (long long)c * rows] : 0.0;
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          if (c < w) {
            double v = yr[c] * (1.0 - 0.5 * F[c + (long long)c * w]);
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (i < c) v -= yr[i] * F[i + (long long)c * w];
            Y[r + (long long)c * rows] = v;
          }
        }
      }
      __syncthreads();
      gram_done = true;
    }
  }

  // ---- column sweep: two-pass Gram-Schmidt with ONE block reduction per
  // column (delayed second pass; see ara_fused.cu dcgs_step).  Step s
  // finalizes column s-1 and runs the first pass of column s:
  //   a = Y_{<s-1}^T v, d = v^T v, b = Y_{<s-1}^T y_s, c = v^T y_s
  //   v <- v - Y a, n^2 = d - |a|^2, u = v / n
  //   y_s <- y_s - Y_{<s-1} b - u (c - a^T b) / n
  for (int st = 1; st <= w && !gram_done; ++st) {
    const int JA = st - 1;
    const bool hasb = st < w;
    double* v = Y + (long long)JA * rows;
    double* ys = hasb ? Y + (long long)st * rows : nullptr;
    const int nd = hasb ? 2 * JA + 2 : JA + 1;
    __syncthreads();
    for (int t = warp; t < nd; t += PW) {
      const double *xa, *xb;
      if (t < JA) {
        xa = Y + (long long)t * rows;
        xb = v;
      } else if (t == JA) {
        xa = v;
        xb = v;
      } else if (t < 2 * JA + 1) {
        xa = Y + (long long)(t - JA - 1) * rows;
        xb = ys;
      } else {
        xa = v;
        xb = ys;
      }
      double sacc = panel_dot(xa, xb, rows, lane);
      sacc = warp_sum(sacc);
      if (lane == 0) S.cbuf[t] = sacc;
    }
    __syncthreads();
    const double* cf = S.cbuf;
    double asq = 0.0;
    for (int p = 0; p < JA; ++p) asq += cf[p] * cf[p];
    const double nj = sqrt(fmax(cf[JA] - asq, 0.0));
    if (tid == 0)
      for (int p = 0; p < JA; ++p) Rp[p + (long long)JA * w] += cf[p];
    if (!(nj >= tau)) {
      const double nr = replace_col(JA, nj);
      const double inv = 1.0 / nr;
      for (int r = tid; r < rows; r += PT) v[r] *= inv;
      if (hasb) {
        cgs_pass(Y, rows, st, S);  // first pass of column s against the final columns
        if (tid == 0)
          for (int p = 0; p < st; ++p) Rp[p + (long long)st * w] += S.cbuf[p];
      }
      continue;
    }
    if (tid == 0) Rp[JA + (long long)JA * w] = nj;
    const double inv = 1.0 / nj;
    double beta = 0.0;
    if (hasb) {
      double ab = 0.0;
      for (int p = 0; p < JA; ++p) ab += cf[p] * cf[JA + 1 + p];
      beta = (cf[2 * JA + 1] - ab) * inv;
      if (tid == 0) {
        for (int p = 0; p < JA; ++p) Rp[p + (long long)st * w] += cf[JA + 1 + p];
        Rp[JA + (long long)st * w] += beta;
      }
    }
    for (int r = tid; r < rows; r += PT) {
      double sa = 0.0, sb = 0.0;
      for (int p = 0; p < JA; ++p) {
        const double yv = Y[(long long)p * rows + r];
        sa += cf[p] * yv;
        if (hasb) sb += cf[JA + 1 + p] * yv;
      }
      const double u = (v[r] - sa) * inv;
      v[r] = u;
      if (hasb) ys[r] -= sb + beta * u;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // smem writes -> async proxy
  __syncthreads();
  if (ys_in_smem && !(finalize && T.qcols)) {
    if (bulk) {
      if (tid == 0) {
        bulk_s2g(T.Y, Y, ybytes);
        bulk_wait_all();
      }
    } else {
      for (long long e = tid; e < (long long)rows * w; e += PT) T.Y[e] = Y[e];
    }
  }

  // R <- Rp * R  (R = I before the first sweep)
  double* R = T.R;
  if (sweep == 0) {
    for (long long e = tid; e < (long long)w * w; e += PT) R[e] = Rp[e];
  } else {
    double* Rt = T.Rp + (long long)w * w;
    for (long long e = tid; e < (long long)w * w; e += PT) {
      int p = (int)(e % w), jj = (int)(e / w);
      double s = 0.0;
      for (int t = p; t <= jj; ++t) s += Rp[p + (long long)t * w] * R[t + (long long)jj * w];
      Rt[e] = p <= jj ? s : 0.0;
    }
    __syncthreads();
    for (long long e = tid; e < (long long)w * w; e += PT) R[e] = Rt[e];
  }
  __syncthreads();
  if (finalize) {
    for (int jj = tid; jj < w; jj += PT) {
      if (T.deficient[jj]) {
        for (int i = 0; i < w; ++i) R[i + (long long)jj * w] = 0.0;
        R[jj + (long long)jj * w] = T.tiny[jj];
        T.col_norms[jj] = T.tiny[jj];
        T.new_mass[jj] = T.tiny[jj];
      } else {
        double s = 0.0;
        for (int i = 0; i <= jj; ++i) s += R[i + (long long)jj * w] * R[i + (long long)jj * w];
        T.col_norms[jj] = sqrt(s);
        T.new_mass[jj] = fabs(R[jj + (long long)jj * w]);
      }
    }
    if (T.qcols) {
      // absorb (ara.cpp:171-195): window of post-deflation norms, keep filter,
      // basis append, convergence / done flags
      __shared__ int keep[64];
      __shared__ int s_nkeep, s_q0;
      __syncthreads();
      if (tid == 0) {
        int qc = *T.qcols;
        *T.rounds += 1;
        int cnt = *T.rcount, pos = *T.rpos;
        for (int j = 0; j < w; ++j) {
          T.recent[pos] = T.col_norms[j];
          pos = (pos + 1) % T.window;
          if (cnt < T.window) ++cnt;
        }
        *T.rcount = cnt;
        *T.rpos = pos;
        int room = T.cap - qc, nk = 0;
        for (int j = 0; j < w && nk < room && nk < 64; ++j)
          if (T.new_mass[j] * T.eta > T.eps) keep[nk++] = j;
        double e = 0.0;
        for (int t = 0; t < cnt; ++t) e = fmax(e, T.recent[t]);
        int conv = e * T.eta <= T.eps;
        *T.conv = conv;
        *T.qcols = qc + nk;
        int dn = conv || (qc + nk) >= T.cap;
        *T.donew = dn;
        if (dn) atomicSub(T.active, 1);
        s_nkeep = nk;
        s_q0 = qc;
      }
      __syncthreads();
      const int nk = s_nkeep, q0 = s_q0;
      for (long long e = tid; e < (long long)nk * rows; e += PT) {
        int c = (int)(e / rows), r = (int)(e % rows);
        T.Qw[(long long)(q0 + c) * rows + r] = Y[(long long)keep[c] * rows + r];
      }
    }
  }
}

void panel_mgs(PanelTask* d_tasks, int ntask, int sweep, int finalize, int max_width,
               int max_rows, cudaStream_t st) {
  static size_t lim = enable_max_dyn_smem(panel_mgs_kernel);
  if (ntask <= 0) return;
  int part_len = max_width;
  int cbuf_len = std::max(2 * max_width + 2, max_rows);  // DCGS2 dot list <= 2 w + 2
  size_t base = ((size_t)2 * PW * part_len + cbuf_len + MT_N) * 8;
  size_t rp = (size_t)max_width * max_width * 8;
  size_t ys = (size_t)max_rows * max_width * 8;
  int rp_in = base + rp <= lim;
  int ys_in = base + (rp_in ? rp : 0) + ys + 16 <= lim;
  size_t bytes = base + (rp_in ? rp : 0) + (ys_in ? ys + 16 : 0);
  panel_mgs_kernel<<<ntask, PT, bytes, st>>>(d_tasks, sweep, finalize, ys_in, rp_in, part_len,
                                             cbuf_len);
  TLRG_CUDA(cudaGetLastError());
}

}  // namespace tlrg
