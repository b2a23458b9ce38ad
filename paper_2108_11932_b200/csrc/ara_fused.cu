// Fused per-tile ARA: ONE launch runs every round of every tile of a batch.
//
// One CTA owns one tile (slot) for its whole adaptive life, so a round costs no
// kernel boundaries and converged tiles free their SM immediately.  Per round
// (TileState::draw/absorb, ara.cpp:155-195, with the reference's orthog,
// dense_kernels.cpp:331-420):
//   draw    Omega_s = next cols x bs values of the tile's exact tlr::Rng stream
//           (pre-generated ring; topped up in-CTA when it runs dry)
//   sample  W = [V^A | -U_k,:]^T Omega   ((kA+K) x bs, FP64 DMMA, split-k)
//           Y = [U^A | H_s] W             (rows x bs, FP64 DMMA, into smem)
//           = A(i,k) Omega - sum_j U_ij G_ij U_kj^T Omega   (Eq. 1, re-associated)
//   orthog  tau = 100 eps_mach ||Y||_F; 2 sweeps of {C = Q^T Y, Y -= Q C (DMMA),
//           column CGS2 panel in smem with deficient-column replacement}
//   absorb  window of post-deflation norms, keep filter, basis append,
//           convergence / done.
// Dense mode (build_tlr's DenseSampler, ara.hpp:43-57): Y = A_tile Omega.
#include <cfloat>

#include "kernels.h"
#include "stream.cuh"

namespace tlrg {

namespace {

constexpr int FT = 256;         // threads per CTA
constexpr int FW = FT / 32;     // warps
constexpr int RED = 2048;       // doubles of split-k partial buffer (8 warps x 64 x NT<=4)

struct FSmem {
  double* Y;      // ldy x bs
  double* R;      // bs x bs
  double* Rp;     // bs x bs
  double* Rt;     // bs x bs
  double* part;   // RED
  double* stg;    // 2 x stg_half (GEMM staging)
  double* cbuf;   // bs (coefficients)
  double* wred;   // FW
  double* tiny;   // bs
  double* cn;     // bs
  double* nm;     // bs
  double* recent; // window
  uint8_t* defi;  // bs
  int* keep;      // bs
  GenSmem* gen;   // aliases Y
};

__device__ __forceinline__ double cta_sum(double v, double* wred) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) wred[warp] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < FW; ++w) s += wred[w];
  return s;
}

// ---- CTA GEMMs with cp.async-staged operands (double-buffered) -----------
// Global operands are streamed through shared memory in chunks so that each
// thread keeps many loads in flight; the FP64 tensor pipe (DMMA.8x8x4) reads
// bank-conflict-free fragments (row strides = 4 mod 16 doubles).
constexpr int KC = 32;           // TN: k-chunk (reduction rows per stage)
constexpr int MB = 64;           // TN: output rows per block (8 warps x 8)
constexpr int LAT = KC + 4;      // TN: smem row stride
constexpr int KN = 8;            // NN: A columns per stage
constexpr int MAXROWS = 512;     // NN: output rows (8 m-tiles per warp)

__device__ __forceinline__ int nn_ld(int rows) { return ((rows + 15) / 16) * 16 + 4; }

// out(m, n, v): v = sgn(m) * sum_{k<Kd} acol(m)[k] * B(k, n),  m < M, n < NT*8.
// B is global (staged, ld ldb) or, with B_SMEM, read directly from shared memory.
template <int NT, bool B_SMEM, class ACol, class Sgn, class Out>
__device__ void gemm_tn(int M, int Kd, ACol acol, const double* B, long long ldb, Sgn sgn,
                        Out out, double* stg, long long stg_half, double* part) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int nmb = (M + MB - 1) / MB, nkc = (Kd + KC - 1) / KC;
  const int total = nmb * nkc;
  if (total == 0) return;
  auto issue = [&](int c) {
    const int mb = c / nkc, kc = c % nkc;
    double* sA = stg + (c & 1) * stg_half;
    double* sB = sA + MB * LAT;
    for (int e = tid; e < MB * KC; e += FT) {
      const int mm = e / KC, kk = e % KC;
      const int m = mb * MB + mm, k = kc * KC + kk;
      const bool v = m < M && k < Kd;
      cp_async8(&sA[mm * LAT + kk], v ? acol(m) + k : acol(0), v);
    }
    if (!B_SMEM)
      for (int e = tid; e < NT * 8 * KC; e += FT) {
        const int n = e / KC, kk = e % KC, k = kc * KC + kk;
        const bool v = k < Kd;
        cp_async8(&sB[n * LAT + kk], v ? B + k + (long long)n * ldb : B, v);
      }
    cp_async_commit();
  };
  double acc[NT][2];
#pragma unroll
  for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = 0.0;
  issue(0);
  for (int c = 0; c < total; ++c) {
    if (c + 1 < total) {
      issue(c + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int mb = c / nkc, kc = c % nkc;
    const int mtb = min(8, (M - mb * MB + 7) / 8);
#ifdef TLRG_FUSED_NOSPLIT
    const int ksp = 1;
    const int mt = warp, kp = warp < mtb ? 0 : 1;
#else
    const int ksp = 8 / mtb;
    const int mt = warp % mtb, kp = warp / mtb;
#endif
    const double* sA = stg + (c & 1) * stg_half;
    const double* sB = sA + MB * LAT;
    if (kp < ksp) {
      for (int st = kp; st < KC / 4; st += ksp) {
        const double a = sA[(mt * 8 + g) * LAT + st * 4 + t];
        double b[NT];
        if (B_SMEM) {
          const int k = kc * KC + st * 4 + t;
#pragma unroll
          for (int j = 0; j < NT; ++j) b[j] = k < Kd ? B[k + (long long)(j * 8 + g) * ldb] : 0.0;
        } else {
#pragma unroll
          for (int j = 0; j < NT; ++j) b[j] = sB[(j * 8 + g) * LAT + st * 4 + t];
        }
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma_8x8x4(acc[j][0], acc[j][1], a, b[j]);
      }
    }
    __syncthreads();
    if (kc == nkc - 1) {
      // block epilogue: reduce the split-k partials in a fixed order
      if (ksp > 1) {
        double* P = part + warp * 64 * NT;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          P[g * 8 * NT + j * 8 + 2 * t] = acc[j][0];
          P[g * 8 * NT + j * 8 + 2 * t + 1] = acc[j][1];
        }
        __syncthreads();
        for (int e = tid; e < mtb * 64 * NT; e += FT) {
          const int mt2 = e / (64 * NT), r = e % (64 * NT);
          const int gi = r / (8 * NT), n = r % (8 * NT);
          const int m = mb * MB + mt2 * 8 + gi;
          if (m >= M) continue;
          double sum = 0.0;
          for (int k2 = 0; k2 < ksp; ++k2) sum += part[(k2 * mtb + mt2) * 64 * NT + r];
          out(m, n, sgn(m) * sum);
        }
        __syncthreads();
      } else if (kp < ksp) {  // idle warps (mtb does not divide 8) hold zeros
        const int m = mb * MB + mt * 8 + g;
        if (m < M) {
          const double sg = sgn(m);
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            out(m, j * 8 + 2 * t, sg * acc[j][0]);
            out(m, j * 8 + 2 * t + 1, sg * acc[j][1]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = 0.0;
    }
  }
  __syncthreads();
}

// epi(m, n, v): v = sum_{k<Kd} acol(k)[m] * B[k + n*ldb],  m < rows (<= 512), n < NT*8.
template <int NT, class ACol, class Epi>
__device__ void gemm_nn(int rows, int Kd, ACol acol, const double* B, long long ldb, Epi epi,
                        double* stg, long long stg_half) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int lda = nn_ld(rows);
  const int nch = (Kd + KN - 1) / KN;
  if (nch == 0) return;
  auto issue = [&](int c) {
    double* sA = stg + (c & 1) * stg_half;
    double* sB = sA + KN * lda;
    for (int e = tid; e < KN * rows; e += FT) {
      const int kk = e / rows, r = e % rows, k = c * KN + kk;
      const bool v = k < Kd;
      cp_async8(&sA[kk * lda + r], v ? acol(k) + r : B, v);
    }
    for (int e = tid; e < NT * 8 * KN; e += FT) {
      const int n = e / KN, kk = e % KN, k = c * KN + kk;
      const bool v = k < Kd;
      cp_async8(&sB[n * (KN + 4) + kk], v ? B + k + (long long)n * ldb : B, v);
    }
    cp_async_commit();
  };
  constexpr int MTW = MAXROWS / 64;
  double acc[MTW][NT][2];
#pragma unroll
  for (int i = 0; i < MTW; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  issue(0);
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) {
      issue(c + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* sA = stg + (c & 1) * stg_half;
    const double* sB = sA + KN * lda;
#pragma unroll
    for (int st = 0; st < KN / 4; ++st) {
      double b[NT];
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = sB[(j * 8 + g) * (KN + 4) + st * 4 + t];
#pragma unroll
      for (int i = 0; i < MTW; ++i) {
        const int m = (warp + 8 * i) * 8 + g;
        if ((warp + 8 * i) * 8 < rows) {
          const double a = sA[(st * 4 + t) * lda + m];
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a, b[j]);
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < MTW; ++i) {
    const int m = (warp + 8 * i) * 8 + g;
    if (m < rows) {
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        epi(m, j * 8 + 2 * t, acc[i][j][0]);
        epi(m, j * 8 + 2 * t + 1, acc[i][j][1]);
      }
    }
  }
  __syncthreads();
}

// one classical pass of column j against the panel columns p < j; the
// coefficients land in S.cbuf (and are added to Rp(:, j) when rp != null)
__device__ void cgs_pass(double* Y, int ldy, int rows, int j, FSmem& S, double* rp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* yj = Y + (long long)j * ldy;
  for (int p = warp; p < j; p += FW) {
    const double* yp = Y + (long long)p * ldy;
    double s = 0.0;
    for (int r = lane; r < rows; r += 32) s += yp[r] * yj[r];
    s = warp_sum(s);
    if (lane == 0) S.cbuf[p] = s;
  }
  __syncthreads();
  if (rp && threadIdx.x < j) rp[threadIdx.x] += S.cbuf[threadIdx.x];
  double* yw = Y + (long long)j * ldy;
  for (int r = threadIdx.x; r < rows; r += FT) {
    double acc = 0.0;
    for (int p = 0; p < j; ++p) acc += S.cbuf[p] * Y[(long long)p * ldy + r];
    yw[r] -= acc;
  }
  __syncthreads();
}

__device__ double col_norm(const double* y, int rows, FSmem& S) {
  double s = 0.0;
  for (int r = threadIdx.x; r < rows; r += FT) s += y[r] * y[r];
  return sqrt(cta_sum(s, S.wred));
}

struct TileCtx {
  const FusedSlot* sl;
  GaussStreams G;
  int s, rows, cols, bs, ldy, q;
  long long* cur;  // smem cursor (absolute stream position)
};

// panel MGS2 of one sweep (dense_kernels.cpp:331-375) on the smem panel; Rp is
// accumulated, deficient columns are replaced from the tile's stream and
// projected against Q and the earlier panel columns.
template <int NT>
__device__ void panel_sweep(TileCtx& T, FSmem& S, int sweep, double tau) {
  const int rows = T.rows, w = T.bs, ldy = T.ldy, q = T.q;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* Y = S.Y;
  for (int e = threadIdx.x; e < w * w; e += FT) S.Rp[e] = 0.0;
  if (sweep == 0)
    for (int j = threadIdx.x; j < w; j += FT) {
      S.defi[j] = 0;
      S.tiny[j] = 0.0;
    }
  __syncthreads();
  const FusedSlot& sl = *T.sl;
  const double* gb = T.G.buf + (long long)T.s * T.G.cap;
  for (int j = 0; j < w; ++j) {
    double* yj = Y + (long long)j * ldy;
    if (j > 0)
      for (int pass = 0; pass < 2; ++pass) cgs_pass(Y, ldy, rows, j, S, S.Rp + (long long)j * w);
    double nj = col_norm(yj, rows, S);
    if (!(nj >= tau)) {
      if (threadIdx.x == 0 && !S.defi[j]) {
        S.defi[j] = 1;
        S.tiny[j] = isfinite(nj) ? nj : 0.0;
      }
      // fresh direction from the tile's own stream: y <- g - Q (Q^T g)
      const long long c0 = *T.cur;
      __syncthreads();
      if (threadIdx.x == 0) *T.cur = c0 + rows;
      ring_copy(gb, T.G.cap, c0, rows, yj, FT);
      __syncthreads();
      if (q > 0) {
        double* rc = sl.repC;
        for (int tq = warp; tq < q; tq += FW) {
          const double* qt = sl.Q + (long long)tq * rows;
          double s = 0.0;
          for (int r = lane; r < rows; r += 32) s += qt[r] * yj[r];
          s = warp_sum(s);
          if (lane == 0) rc[tq] = s;
        }
        __syncthreads();
        for (int r = threadIdx.x; r < rows; r += FT) {
          double s = 0.0;
          for (int tq = 0; tq < q; ++tq) s += sl.Q[(long long)tq * rows + r] * rc[tq];
          yj[r] -= s;
        }
        __syncthreads();
      }
      if (j > 0)
        for (int pass = 0; pass < 2; ++pass) cgs_pass(Y, ldy, rows, j, S, nullptr);
      nj = col_norm(yj, rows, S);
      if (nj == 0.0) {
        if (threadIdx.x == 0) yj[j % rows] = 1.0;
        nj = 1.0;
      }
      if (threadIdx.x == 0) S.Rp[j + (long long)j * w] = 0.0;
    } else {
      if (threadIdx.x == 0) S.Rp[j + (long long)j * w] = nj;
    }
    const double inv = 1.0 / nj;
    for (int r = threadIdx.x; r < rows; r += FT) yj[r] *= inv;
    __syncthreads();
  }
  // R <- Rp R   (R = I before the first sweep)
  if (sweep == 0) {
    for (int e = threadIdx.x; e < w * w; e += FT) S.R[e] = S.Rp[e];
  } else {
    for (int e = threadIdx.x; e < w * w; e += FT) {
      const int p = e % w, jj = e / w;
      double s = 0.0;
      for (int tt = p; tt <= jj; ++tt) s += S.Rp[p + tt * w] * S.R[tt + jj * w];
      S.Rt[e] = p <= jj ? s : 0.0;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < w * w; e += FT) S.R[e] = S.Rt[e];
  }
  __syncthreads();
}

template <int NT>
__global__ void __launch_bounds__(FT) ara_fused_kernel(FusedArgs A) {
  extern __shared__ __align__(16) double fsm[];
  const int s = blockIdx.x;
  const FusedSlot& sl = A.slots[s];
  const int rows = sl.rows, cols = A.cols, bs = NT * 8;
  const int ldy = A.ldy;
  FSmem S;
  {
    double* p = fsm;
    S.Y = p;
    p += A.ysz;
    S.gen = reinterpret_cast<GenSmem*>(S.Y);
    S.R = p; p += bs * bs;
    S.Rp = p; p += bs * bs;
    S.Rt = p; p += bs * bs;
    S.part = p; p += RED;
    S.stg = p; p += 2 * A.stg_half;
    S.cbuf = p; p += bs;
    S.wred = p; p += FW;
    S.tiny = p; p += bs;
    S.cn = p; p += bs;
    S.nm = p; p += bs;
    S.recent = p; p += A.window;
    S.keep = reinterpret_cast<int*>(p); p += bs;
    S.defi = reinterpret_cast<uint8_t*>(p);
  }
  __shared__ long long s_cur, s_av;
  __shared__ int s_q, s_done, s_nkeep, s_rounds, s_conv, s_rcount, s_rpos;
  __shared__ double s_tau;
  if (threadIdx.x == 0) {
    s_cur = A.G.cursor[s];
    s_av = A.G.avail[s];
    s_q = 0;
    s_done = sl.cap <= 0;
    s_rounds = 0;
    s_conv = 0;
    s_rcount = 0;
    s_rpos = 0;
  }
  __syncthreads();
  TileCtx T{&sl, A.G, s, rows, cols, bs, ldy, 0, &s_cur};
  const double* gb = A.G.buf + (long long)s * A.G.cap;
  const int kA = sl.kA, K = A.K, KW = kA + K;

  while (!s_done && s_rounds < A.max_rounds) {
    // ---- draw: make sure Omega and every possible replacement are available
    {
      const long long need = (long long)cols * bs + 2LL * bs * rows;
      if (s_av - s_cur < need) {
        long long want = s_cur + need + 2LL * cols * bs;
        long long tgt = want < s_cur + A.G.cap ? want : s_cur + A.G.cap;
        tgt &= ~1LL;
        GaussStreams G = A.G;
        cta_generate(G, s, s_av, tgt, *S.gen);
        if (threadIdx.x == 0) s_av = A.G.avail[s];
        __syncthreads();
      }
      ring_copy(gb, A.G.cap, s_cur, (long long)cols * bs, sl.Om, FT);
      __syncthreads();
      if (threadIdx.x == 0) s_cur += (long long)cols * bs;
    }
    // ---- sample -------------------------------------------------------------
    if (sl.Ad) {
      // dense operator: Y = A_tile Omega
      gemm_nn<NT>(
          rows, cols, [&](int k) { return sl.Ad + (long long)k * sl.ldad; }, sl.Om, cols,
          [&](int m, int n, double v) { S.Y[m + n * ldy] = v; }, S.stg, A.stg_half);
    } else {
      // W = [V^A | -U_k,:]^T Omega
      gemm_tn<NT, false>(
          KW, cols,
          [&](int m) { return m < kA ? sl.VA + (long long)m * cols : A.Ucat + (long long)(m - kA) * cols; },
          sl.Om, cols, [&](int m) { return m < kA ? 1.0 : -1.0; },
          [&](int m, int n, double v) { sl.W[m + (long long)n * KW] = v; }, S.stg, A.stg_half,
          S.part);
      // Y = [U^A | H] W
      gemm_nn<NT>(
          rows, KW,
          [&](int k) { return k < kA ? sl.UA + (long long)k * rows : sl.H + (long long)(k - kA) * rows; },
          sl.W, KW, [&](int m, int n, double v) { S.Y[m + n * ldy] = v; }, S.stg, A.stg_half);
    }
    // ---- orthog (dense_kernels.cpp:379-420) ------------------------------------
    {
      double f = 0.0;
      for (int e = threadIdx.x; e < rows * bs; e += FT) {
        const double y = S.Y[(e % rows) + (e / rows) * ldy];
        f += y * y;
      }
      f = cta_sum(f, S.wred);
      if (threadIdx.x == 0) {
        double tau = 100.0 * DBL_EPSILON * sqrt(f);
        s_tau = tau == 0.0 ? DBL_MIN : tau;
      }
      __syncthreads();
    }
    T.q = s_q;
    for (int sweep = 0; sweep < 2; ++sweep) {
      if (T.q > 0) {
        const int q = T.q;
        // C = Q^T Y
        gemm_tn<NT, true>(
            q, rows, [&](int m) { return sl.Q + (long long)m * rows; }, S.Y, ldy,
            [](int) { return 1.0; }, [&](int m, int n, double v) { sl.Cq[m + (long long)n * q] = v; },
            S.stg, A.stg_half, S.part);
        // Y -= Q C
        gemm_nn<NT>(
            rows, q, [&](int k) { return sl.Q + (long long)k * rows; }, sl.Cq, q,
            [&](int m, int n, double v) { S.Y[m + n * ldy] -= v; }, S.stg, A.stg_half);
      }
      panel_sweep<NT>(T, S, sweep, s_tau);
    }
    // ---- finalize + absorb (ara.cpp:171-195) -----------------------------------
    for (int jj = threadIdx.x; jj < bs; jj += FT) {
      if (S.defi[jj]) {
        S.cn[jj] = S.tiny[jj];
        S.nm[jj] = S.tiny[jj];
      } else {
        double v = 0.0;
        for (int i = 0; i <= jj; ++i) v += S.R[i + jj * bs] * S.R[i + jj * bs];
        S.cn[jj] = sqrt(v);
        S.nm[jj] = fabs(S.R[jj + jj * bs]);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int qc = s_q;
      int cnt = s_rcount, pos = s_rpos;
      for (int j = 0; j < bs; ++j) {
        S.recent[pos] = S.cn[j];
        pos = (pos + 1) % A.window;
        if (cnt < A.window) ++cnt;
      }
      s_rcount = cnt;
      s_rpos = pos;
      const int room = sl.cap - qc;
      int nk = 0;
      for (int j = 0; j < bs && nk < room; ++j)
        if (S.nm[j] * A.eta > A.eps) S.keep[nk++] = j;
      double e = 0.0;
      for (int t2 = 0; t2 < cnt; ++t2) e = fmax(e, S.recent[t2]);
      s_conv = e * A.eta <= A.eps;
      s_q = qc + nk;
      s_nkeep = nk;
      s_done = s_conv || (qc + nk) >= sl.cap;
      ++s_rounds;
    }
    __syncthreads();
    {
      const int nk = s_nkeep, q0 = s_q - s_nkeep;
      for (int e = threadIdx.x; e < nk * rows; e += FT) {
        const int c = e / rows, r = e % rows;
        sl.Q[(long long)(q0 + c) * rows + r] = S.Y[r + S.keep[c] * ldy];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    A.qcols[s] = s_q;
    A.rounds[s] = s_rounds;
    A.conv[s] = s_conv;
    A.G.cursor[s] = s_cur;
    A.G.avail[s] = s_av;
  }
}

long long fused_stg_half(int maxrows, int bs) {
  long long tn = (long long)(MB + bs) * LAT;
  long long nn = (long long)KN * (((maxrows + 15) / 16) * 16 + 4) + (long long)bs * (KN + 4);
  long long h = tn > nn ? tn : nn;
  return (h + 1) & ~1LL;
}
size_t fused_smem_bytes(int maxrows, int bs, int window, int* ldy, long long* ysz) {
  int l = ((maxrows + 15) / 16) * 16 + 4;
  long long y = (long long)l * bs;
  long long gen = (sizeof(GenSmem) + 7) / 8;
  if (y < gen) y = gen;
  y = (y + 1) & ~1LL;
  *ldy = l;
  *ysz = y;
  long long d = y + 3LL * bs * bs + RED + 2 * fused_stg_half(maxrows, bs) + bs + FW + 3LL * bs + window + bs /*keep ints*/ + bs;
  return (size_t)d * 8 + 64;
}

}  // namespace

bool ara_fused_supported(int maxrows, int bs, int window) {
  if (maxrows > MAXROWS) return false;
  if (bs != 8 && bs != 16 && bs != 24 && bs != 32) return false;
  int ldy;
  long long ysz;
  size_t bytes = fused_smem_bytes(maxrows, bs, window, &ldy, &ysz);
  static int optin = 0;
  if (!optin) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  return bytes + 1024 <= (size_t)optin;
}

void ara_fused(FusedArgs args, int T, int maxrows, cudaStream_t st) {
  if (T <= 0) return;
  const int bs = args.bs;
  long long ysz;
  size_t bytes = fused_smem_bytes(maxrows, bs, args.window, &args.ldy, &ysz);
  args.ysz = ysz;
  args.stg_half = fused_stg_half(maxrows, bs);
  switch (bs) {
#define TLRG_FUSED_CASE(NT)                                                                 \
  case NT * 8: {                                                                            \
    static size_t lim = enable_max_dyn_smem(ara_fused_kernel<NT>);                          \
    if (bytes > lim) throw CudaError("ara_fused: shared memory budget exceeded");           \
    ara_fused_kernel<NT><<<T, FT, bytes, st>>>(args);                                       \
    break;                                                                                  \
  }
    TLRG_FUSED_CASE(1)
    TLRG_FUSED_CASE(2)
    TLRG_FUSED_CASE(3)
    TLRG_FUSED_CASE(4)
#undef TLRG_FUSED_CASE
    default:
      throw CudaError("ara_fused: unsupported block size");
  }
  TLRG_CUDA(cudaGetLastError());
}

}  // namespace tlrg
