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
#include <cstdlib>

#include "kernels.h"
#include "stream.cuh"

namespace tlrg {

namespace {

constexpr int FT = 256;         // consumer threads per CTA
constexpr int FW = FT / 32;     // consumer warps
constexpr int FTP = FT + 32;    // + one producer warp (gaussian stream)

// barrier among the consumer warps only (the producer warp runs free)
__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, %0;" ::"n"(FT) : "memory"); }
constexpr int MAXROWS = 512;
constexpr int RPT = MAXROWS / FT;  // tile rows per consumer thread (r = tid + i*FT)
constexpr int PART_UNITS = 16;  // split-k partial tiles kept in shared memory

struct FSmem {
  double* Y;      // ldy x bs
  double* R;      // bs x bs
  double* Rp;     // bs x bs
  double* Rt;     // bs x bs
  double* part;   // PART_UNITS x 64 x NT
  double* cbuf;   // bs (coefficients)
  double* wpart;  // 2 x FW x 32 per-warp partial coefficient vectors
  double* wred;   // FW
  double* tiny;   // bs
  double* cn;     // bs
  double* nm;     // bs
  double* recent; // window
  uint8_t* defi;  // bs
  int* keep;      // bs
  double* sig;    // FUSED_QMAX
  int* perm;      // FUSED_QMAX
};

__device__ __forceinline__ double cta_sum(double v, double* wred) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  cbar();
  if (lane == 0) wred[warp] = v;
  cbar();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < FW; ++w) s += wred[w];
  return s;
}

__device__ __forceinline__ double2 ld2(const double* p) {
  return *reinterpret_cast<const double2*>(p);
}

// ---- CTA GEMMs on the FP64 tensor pipe with direct 16-byte fragment loads --
// Every lane owns a PAIR of consecutive reduction indices per 8-k block and
// feeds them to two DMMA.8x8x4 (the k order inside a block is immaterial as
// long as both operands agree), so each fragment load is one 128-bit access.
// Operands live in L2 (streamed once per round) or shared memory.

// out(m, n, v): v = sgn(m) * sum_{k<Kd} acol(m)[k] * bcol(n)[k],  m < M, n < NT*8.
// Kd even; acol/bcol columns 16-byte aligned.  Split-k over warps when M is
// small, partial tiles reduced in a fixed order (deterministic).
template <int NT, class ACol, class BCol, class Sgn, class Out>
__device__ void tn16(int M, int Kd, ACol acol, BCol bcol, Sgn sgn, Out out, double* part) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int mtiles = (M + 7) / 8;
  if (mtiles == 0 || Kd <= 0) return;
  if (mtiles >= FW) {
    // wide: k-outer, MTW m-tiles per warp share each B fragment (more loads in flight)
    constexpr int MTW = 4;
    const int k8 = (Kd + 7) / 8;
    const double* bp[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) bp[j] = bcol(j * 8 + g);
    for (int base = 0; base < mtiles; base += FW * MTW) {
      const double* ap[MTW];
      bool mv[MTW];
#pragma unroll
      for (int i = 0; i < MTW; ++i) {
        const int m = (base + warp + FW * i) * 8 + g;
        mv[i] = m < M;
        ap[i] = mv[i] ? acol(m) : nullptr;
      }
      double acc[MTW][NT][2];
#pragma unroll
      for (int i = 0; i < MTW; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 4
      for (int kb = 0; kb < k8; ++kb) {
        const int kk = kb * 8 + 2 * t;
        const bool kv = kk < Kd;
        double2 b[NT], a[MTW];
#pragma unroll
        for (int j = 0; j < NT; ++j) b[j] = kv ? ld2(bp[j] + kk) : make_double2(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < MTW; ++i) a[i] = (mv[i] && kv) ? ld2(ap[i] + kk) : make_double2(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < MTW; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i].x, b[j].x);
            dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i].y, b[j].y);
          }
      }
#pragma unroll
      for (int i = 0; i < MTW; ++i) {
        const int m = (base + warp + FW * i) * 8 + g;
        if (m < M) {
          const double sg = sgn(m);
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            out(m, j * 8 + 2 * t, sg * acc[i][j][0]);
            out(m, j * 8 + 2 * t + 1, sg * acc[i][j][1]);
          }
        }
      }
    }
    cbar();
    return;
  }
  int ks = FW / mtiles;
  if (ks < 1) ks = 1;
  if (ks * mtiles > PART_UNITS) ks = PART_UNITS / mtiles > 0 ? PART_UNITS / mtiles : 1;
  const int k8 = (Kd + 7) / 8;
  const int per = (k8 + ks - 1) / ks;
  const int units = mtiles * ks;
  for (int u = warp; u < units; u += FW) {
    const int mt = u % mtiles, kc = u / mtiles;
    const int m = mt * 8 + g;
    const bool mv = m < M;
    const double* ap = mv ? acol(m) : nullptr;
    const double* bp[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) bp[j] = bcol(j * 8 + g);
    const int b_lo = kc * per, b_hi = min(k8, b_lo + per);
    double acc[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll 2
    for (int kb = b_lo; kb < b_hi; ++kb) {
      const int kk = kb * 8 + 2 * t;
      const bool kv = kk < Kd;
      const double2 a = (mv && kv) ? ld2(ap + kk) : make_double2(0.0, 0.0);
      double2 b[NT];
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = kv ? ld2(bp[j] + kk) : make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        dmma_8x8x4(acc[j][0], acc[j][1], a.x, b[j].x);
        dmma_8x8x4(acc[j][0], acc[j][1], a.y, b[j].y);
      }
    }
    if (ks == 1) {
      if (mv) {
        const double sg = sgn(m);
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          out(m, j * 8 + 2 * t, sg * acc[j][0]);
          out(m, j * 8 + 2 * t + 1, sg * acc[j][1]);
        }
      }
    } else {
      double* P = part + (long long)u * 64 * NT;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        P[g * 8 * NT + j * 8 + 2 * t] = acc[j][0];
        P[g * 8 * NT + j * 8 + 2 * t + 1] = acc[j][1];
      }
    }
  }
  if (ks > 1) {
    cbar();
    for (int e = threadIdx.x; e < mtiles * 64 * NT; e += FT) {
      const int mt = e / (64 * NT), r = e % (64 * NT);
      const int m = mt * 8 + r / (8 * NT), n = r % (8 * NT);
      if (m >= M) continue;
      double sum = 0.0;
      for (int kc = 0; kc < ks; ++kc) sum += part[((long long)kc * mtiles + mt) * 64 * NT + r];
      out(m, n, sgn(m) * sum);
    }
  }
  cbar();
}

// epi(r, c, v): v = sum_{k<Kd} acol(k)[r] * B[k + c*ldb],  r < rows (even, <= 512),
// c < NT*8.  Computed as (B^T A^T): the small operand B is the DMMA "A" side and
// every lane loads two consecutive tile rows (even/odd 8-row DMMA tiles) with
// one 128-bit access (ldb even, 16-byte aligned columns).
template <int NT, class ACol, class Epi>
__device__ void nn16(int rows, int Kd, ACol acol, const double* B, int ldb, Epi epi) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  constexpr int GPW = MAXROWS / 16 / FW;  // 16-row groups per warp
  const int ngr = (rows + 15) / 16;
  double acc[GPW][NT][2][2];
#pragma unroll
  for (int i = 0; i < GPW; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0][0] = acc[i][j][0][1] = acc[i][j][1][0] = acc[i][j][1][1] = 0.0;
  const int k8 = (Kd + 7) / 8;
#pragma unroll 4
  for (int kb = 0; kb < k8; ++kb) {
    const int kk = kb * 8 + 2 * t;
    double2 aw[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const double* bj = B + kk + (long long)(j * 8 + g) * ldb;
      aw[j] = kk + 1 < Kd ? ld2(bj) : make_double2(kk < Kd ? bj[0] : 0.0, 0.0);
    }
    const double* c0 = kk < Kd ? acol(kk) : nullptr;
    const double* c1 = kk + 1 < Kd ? acol(kk + 1) : nullptr;
#pragma unroll
    for (int i = 0; i < GPW; ++i) {
      const int gr = warp + FW * i;
      const int r = gr * 16 + 2 * g;
      double2 b0 = make_double2(0.0, 0.0), b1 = make_double2(0.0, 0.0);
      if (gr < ngr && r < rows) {
        if (c0) b0 = ld2(c0 + r);
        if (c1) b1 = ld2(c1 + r);
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        dmma_8x8x4(acc[i][j][0][0], acc[i][j][0][1], aw[j].x, b0.x);
        dmma_8x8x4(acc[i][j][1][0], acc[i][j][1][1], aw[j].x, b0.y);
        dmma_8x8x4(acc[i][j][0][0], acc[i][j][0][1], aw[j].y, b1.x);
        dmma_8x8x4(acc[i][j][1][0], acc[i][j][1][1], aw[j].y, b1.y);
      }
    }
  }
  // a warp reads and writes only its own row groups: once every lane's reads
  // are done the epilogue may overwrite an operand in place
  __syncwarp();
#pragma unroll
  for (int i = 0; i < GPW; ++i) {
    const int gr = warp + FW * i;
    if (gr >= ngr) continue;
    const int r0 = gr * 16 + 4 * t;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int c = j * 8 + g;
      // even tile: rows r0, r0 + 2; odd tile: rows r0 + 1, r0 + 3
      if (r0 < rows) {
        epi(r0, c, acc[i][j][0][0]);
        epi(r0 + 1, c, acc[i][j][1][0]);
      }
      if (r0 + 2 < rows) {
        epi(r0 + 2, c, acc[i][j][0][1]);
        epi(r0 + 3, c, acc[i][j][1][1]);
      }
    }
  }
  cbar();
}

struct TileCtx {
  const FusedSlot* sl;
  GaussStreams G;
  int s, rows, cols, bs, ldy, q;
  long long* cur;  // smem cursor (absolute stream position)
  long long* av;   // smem count of values produced (producer warp)
  int wlim;        // panel columns actually present (<= BS)
  int passes;      // Gram-Schmidt passes per column and sweep (reference: 2)
  int dcgs;        // one reduction per column (delayed second pass)
};

// Reduce-scatter of N (16 or 32) values over a warp: afterwards every lane
// holds the full warp sum of index (lane >> 1) (N = 16) or lane (N = 32).
// Reduce-scatter of N (a power of two <= 32) values over a warp: afterwards
// every lane holds the full warp sum of index lane >> (5 - log2 N).  N halving
// levels (N-1 shuffles) plus one full xor level per remaining lane bit.
template <int N>
__device__ __forceinline__ double warp_reduce_scatter(double (&v)[N]) {
  const int lane = threadIdx.x & 31;
  double w[N];
#pragma unroll
  for (int i = 0; i < N; ++i) w[i] = v[i];
#pragma unroll
  for (int half = N / 2, bit = 16; half >= 1; half >>= 1, bit >>= 1) {
    const bool hi = (lane & bit) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double send = hi ? w[i] : w[i + half];
      const double keep = hi ? w[i + half] : w[i];
      w[i] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
    }
  }
  double r = w[0];
#pragma unroll
  for (int bit = 16 / N; bit >= 1; bit >>= 1) r += __shfl_xor_sync(0xffffffffu, r, bit);
  return r;
}

// ---- TMA-staged streaming of the big operand (sampling products) ----------
// The A operands of the two sampling products ([V^A | U_k,:] and [U^A | H_i],
// 4 KB columns) stream through shared memory by bulk copies (cp.async.bulk,
// mbarrier completion, two stages of SCOL columns, padded stride so the
// 16-byte fragment loads are bank-conflict free); compute on one stage
// overlaps the copy of the next.
constexpr int SCOL = 8;
constexpr int SPAD = 520;
struct Stager {
  double* buf;    // 2 x SCOL x SPAD
  uint64_t* bar;  // 2 mbarriers
};
template <class ACol>
__device__ __forceinline__ void stage_issue(const Stager& st, int s, int c, int ncol, int len,
                                            ACol acol) {
  if (threadIdx.x == 0) {
    const int c0 = c * SCOL, nc = min(SCOL, ncol - c0);
    mbar_arrive_expect_tx(&st.bar[s], (unsigned)(nc * len * 8));
    for (int j = 0; j < nc; ++j)
      bulk_g2s(st.buf + (s * SCOL + j) * SPAD, acol(c0 + j), (unsigned)(len * 8), &st.bar[s]);
  }
}

// out(m, n, v) for m < M: v = sgn(m) * sum_{k<Kd} acol(m)[k] * bcol(n)[k]; the M
// columns are staged 8 at a time, the warps split k, partials reduced in a
// fixed order.  Kd even, <= 8 * 64 * FW.
template <int NT, class ACol, class BCol, class Sgn, class Out>
__device__ void tn16_tma(int M, int Kd, ACol acol, BCol bcol, Sgn sgn, Out out, double* part,
                         const Stager& st, unsigned& ph) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int nch = (M + SCOL - 1) / SCOL;
  if (nch == 0 || Kd <= 0) return;
  const int k8 = (Kd + 7) / 8, per = (k8 + FW - 1) / FW;
  const int kb0 = warp * per, kb1 = min(k8, kb0 + per);
  const double* bp[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) bp[j] = bcol(j * 8 + g);
  stage_issue(st, 0, 0, M, Kd, acol);
  if (nch > 1) stage_issue(st, 1, 1, M, Kd, acol);
  for (int c = 0; c < nch; ++c) {
    const int s = c & 1;
    mbar_wait(&st.bar[s], (ph >> s) & 1u);
    ph ^= 1u << s;
    const bool mv = c * SCOL + g < M;
    const double* ap = st.buf + (s * SCOL + g) * SPAD;
    double acc[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll 4
    for (int kb = kb0; kb < kb1; ++kb) {
      const int kk = kb * 8 + 2 * t;
      const bool kv = kk < Kd;
      const double2 a = (mv && kv) ? ld2(ap + kk) : make_double2(0.0, 0.0);
      double2 b[NT];
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = kv ? ld2(bp[j] + kk) : make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        dmma_8x8x4(acc[j][0], acc[j][1], a.x, b[j].x);
        dmma_8x8x4(acc[j][0], acc[j][1], a.y, b[j].y);
      }
    }
    double* P = part + warp * 64 * NT;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      P[g * 8 * NT + j * 8 + 2 * t] = acc[j][0];
      P[g * 8 * NT + j * 8 + 2 * t + 1] = acc[j][1];
    }
    cbar();
    for (int e = threadIdx.x; e < 64 * NT; e += FT) {
      const int m = c * SCOL + e / (8 * NT), n = e % (8 * NT);
      if (m < M) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < FW; ++w) sum += part[w * 64 * NT + e];
        out(m, n, sgn(m) * sum);
      }
    }
    cbar();
    if (c + 2 < nch) stage_issue(st, s, c + 2, M, Kd, acol);
  }
}

// epi(r, c, v): v = sum_{k<Kd} acol(k)[r] * B[k + c*ldb]; the Kd columns of the
// big operand are staged 8 at a time (one 8-k block per stage).
template <int NT, class ACol, class Epi>
__device__ void nn16_tma(int rows, int Kd, ACol acol, const double* B, int ldb, Epi epi,
                         const Stager& st, unsigned& ph) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  constexpr int GPW = MAXROWS / 16 / FW;
  const int ngr = (rows + 15) / 16;
  const int nch = (Kd + SCOL - 1) / SCOL;
  double acc[GPW][NT][2][2];
#pragma unroll
  for (int i = 0; i < GPW; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j)
      acc[i][j][0][0] = acc[i][j][0][1] = acc[i][j][1][0] = acc[i][j][1][1] = 0.0;
  if (nch > 0) stage_issue(st, 0, 0, Kd, rows, acol);
  if (nch > 1) stage_issue(st, 1, 1, Kd, rows, acol);
  for (int c = 0; c < nch; ++c) {
    const int s = c & 1;
    const int kk = c * SCOL + 2 * t;
    double2 aw[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const double* bj = B + kk + (long long)(j * 8 + g) * ldb;
      aw[j] = kk + 1 < Kd ? ld2(bj) : make_double2(kk < Kd ? bj[0] : 0.0, 0.0);
    }
    mbar_wait(&st.bar[s], (ph >> s) & 1u);
    ph ^= 1u << s;
    const double* c0p = st.buf + (s * SCOL + 2 * t) * SPAD;
    const double* c1p = c0p + SPAD;
    const bool v0 = kk < Kd, v1 = kk + 1 < Kd;
#pragma unroll
    for (int i = 0; i < GPW; ++i) {
      const int gr = warp + FW * i;
      const int r = gr * 16 + 2 * g;
      double2 b0 = make_double2(0.0, 0.0), b1 = make_double2(0.0, 0.0);
      if (gr < ngr && r < rows) {
        if (v0) b0 = ld2(c0p + r);
        if (v1) b1 = ld2(c1p + r);
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        dmma_8x8x4(acc[i][j][0][0], acc[i][j][0][1], aw[j].x, b0.x);
        dmma_8x8x4(acc[i][j][1][0], acc[i][j][1][1], aw[j].x, b0.y);
        dmma_8x8x4(acc[i][j][0][0], acc[i][j][0][1], aw[j].y, b1.x);
        dmma_8x8x4(acc[i][j][1][0], acc[i][j][1][1], aw[j].y, b1.y);
      }
    }
    cbar();
    if (c + 2 < nch) stage_issue(st, s, c + 2, Kd, rows, acol);
  }
#pragma unroll
  for (int i = 0; i < GPW; ++i) {
    const int gr = warp + FW * i;
    if (gr >= ngr) continue;
    const int r0 = gr * 16 + 4 * t;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int cc = j * 8 + g;
      if (r0 < rows) {
        epi(r0, cc, acc[i][j][0][0]);
        epi(r0 + 1, cc, acc[i][j][1][0]);
      }
      if (r0 + 2 < rows) {
        epi(r0 + 2, cc, acc[i][j][0][1]);
        epi(r0 + 3, cc, acc[i][j][1][1]);
      }
    }
  }
  cbar();
}

// one classical pass of column j of the register-resident panel against the
// columns p < j (each thread owns RPT tile rows).  Every warp writes its
// reduce-scattered partial dots to shared memory (double-buffered by pass
// parity), ONE barrier, then lane p of every warp sums coefficient p over the
// warps in a fixed order and the update takes it by shuffle.  Warp 0 adds the
// coefficients to Rp(:, j) when rpj != null.
// NORM: the same reduction also returns ||y_J||^2 BEFORE the update (slot J),
// so a second pass yields the post-pass norm by Pythagoras,
// ||y - Y c||^2 = ||y||^2 - ||c||^2 (Y orthonormal), without a third barrier.
template <int BS, int J, bool NORM = false>
__device__ __forceinline__ void cgs_pass_reg(double (&y)[RPT][BS], FSmem& S, double* rpj,
                                             int& par, double* sq_out = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int JN = J + (NORM ? 1 : 0);
  constexpr int N = JN <= 2 ? 2 : JN <= 4 ? 4 : JN <= 8 ? 8 : JN <= 16 ? 16 : 32;
  constexpr int SH = (N == 2 ? 4 : N == 4 ? 3 : N == 8 ? 2 : N == 16 ? 1 : 0);  // 5 - log2 N
  double part[N];
#pragma unroll
  for (int p = 0; p < N; ++p) {
    double v = 0.0;
    if (p < J) {
#pragma unroll
      for (int i = 0; i < RPT; ++i) v += y[i][p] * y[i][J];
    } else if (NORM && p == J) {
#pragma unroll
      for (int i = 0; i < RPT; ++i) v += y[i][J] * y[i][J];
    }
    part[p] = v;
  }
  const double red = warp_reduce_scatter<N>(part);
  double* wp = S.wpart + par * (FW * 32);
  par ^= 1;
  if ((lane & ((1 << SH) - 1)) == 0) wp[warp * 32 + (lane >> SH)] = red;
  cbar();
  double c = 0.0;
  if (lane < JN) {
    double h0 = 0.0, h1 = 0.0;
#pragma unroll
    for (int w = 0; w < FW; w += 2) {
      h0 += wp[w * 32 + lane];
      h1 += wp[(w + 1) * 32 + lane];
    }
    c = h0 + h1;
  }
  if (rpj && warp == 0 && lane < J) rpj[lane] += c;
  double cf[J > 0 ? J : 1];
#pragma unroll
  for (int p = 0; p < J; ++p) cf[p] = __shfl_sync(0xffffffffu, c, p);
  if (NORM) {
    double ysq = __shfl_sync(0xffffffffu, c, J), csq = 0.0;
#pragma unroll
    for (int p = 0; p < J; ++p) csq += cf[p] * cf[p];
    *sq_out = ysq - csq;
  }
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
    for (int p = 0; p < J; p += 4) {
      a0 += cf[p] * y[i][p];
      if (p + 1 < J) a1 += cf[p + 1] * y[i][p + 1];
      if (p + 2 < J) a2 += cf[p + 2] * y[i][p + 2];
      if (p + 3 < J) a3 += cf[p + 3] * y[i][p + 3];
    }
    y[i][J] -= (a0 + a1) + (a2 + a3);
  }
}

// ||column||_2 over the tile rows of all consumer threads (one barrier)
template <int BS>
__device__ __forceinline__ double cta_norm(const double (&y)[RPT][BS], int J, FSmem& S, int& par) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v = 0.0;
#pragma unroll
  for (int i = 0; i < RPT; ++i) v += y[i][J] * y[i][J];
  v = warp_sum(v);
  double* wr = S.wpart + par * (FW * 32);  // shares the pass buffers' parity
  par ^= 1;
  if (lane == 0) wr[warp] = v;
  cbar();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < FW; ++w) s += wr[w];
  return sqrt(s);
}

// deficient column J (norm below tau after its passes): record the first tiny
// norm, restart from a fresh direction of the tile's own stream, project it off
// Q and the earlier panel columns (dense_kernels.cpp:348-372); returns the norm
// to normalize by
template <int BS, int J>
__device__ __forceinline__ double replace_column(TileCtx& T, FSmem& S, double (&y)[RPT][BS], double nj,
                                              int& par) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0 && !S.defi[J]) {
    S.defi[J] = 1;
    S.tiny[J] = isfinite(nj) ? nj : 0.0;
  }
  const long long c0 = *T.cur;
  {
    volatile long long* av = T.av;
    while (*av < c0 + T.rows) __nanosleep(64);
    __threadfence_block();
  }
  cbar();
  if (threadIdx.x == 0) *T.cur = c0 + T.rows;
  const double* gb = T.G.buf + (long long)T.s * T.G.cap;
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int r = threadIdx.x + i * FT;
    y[i][J] = r < T.rows ? gb[(c0 + r) % T.G.cap] : 0.0;
  }
  const int q = T.q;
  if (q > 0) {
    const FusedSlot& sl = *T.sl;
    double* yj = S.Y + (long long)J * T.ldy;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int r = threadIdx.x + i * FT;
      if (r < T.rows) yj[r] = y[i][J];
    }
    cbar();
    for (int tq = warp; tq < q; tq += FW) {
      const double* qt = sl.Q + (long long)tq * T.rows;
      double s = 0.0;
      for (int i2 = lane; i2 < T.rows; i2 += 32) s += qt[i2] * yj[i2];
      s = warp_sum(s);
      if (lane == 0) sl.repC[tq] = s;
    }
    cbar();
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int r = threadIdx.x + i * FT;
      if (r < T.rows) {
        double s = 0.0;
        for (int tq = 0; tq < q; ++tq) s += sl.Q[(long long)tq * T.rows + r] * sl.repC[tq];
        y[i][J] -= s;
      }
    }
  }
  if (J > 0) {
    cgs_pass_reg<BS, J>(y, S, nullptr, par);
    cgs_pass_reg<BS, J>(y, S, nullptr, par);
  }
  nj = cta_norm<BS>(y, J, S, par);
  if (nj == 0.0) {
#pragma unroll
    for (int i = 0; i < RPT; ++i) y[i][J] = (threadIdx.x + i * FT == J % T.rows) ? 1.0 : 0.0;
    nj = 1.0;
  }
  return nj;
}

// panel MGS2 of one sweep (dense_kernels.cpp:331-375) with the panel held in
// registers (rows tid + i*FT of the tile in thread tid); Rp is accumulated,
// deficient columns are replaced from the tile's stream and projected against
// Q and the earlier panel columns.
template <int BS, int J>
__device__ __forceinline__ void mgs_column(TileCtx& T, FSmem& S, double (&y)[RPT][BS], double tau,
                                           int& par) {
  if (J >= T.wlim) return;  // uniform
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* rpj = S.Rp + J * BS;
  double nj;
  if (J > 0 && T.passes > 1) {
    cgs_pass_reg<BS, J>(y, S, rpj, par);
    double sq;
    cgs_pass_reg<BS, J, true>(y, S, rpj, par, &sq);
    nj = sqrt(fmax(sq, 0.0));
  } else {
    if (J > 0) cgs_pass_reg<BS, J>(y, S, rpj, par);
    nj = cta_norm<BS>(y, J, S, par);
  }
  if (!(nj >= tau)) {
    nj = replace_column<BS, J>(T, S, y, nj, par);
    if (threadIdx.x == 0) rpj[J] = 0.0;
  } else {
    if (threadIdx.x == 0) rpj[J] = nj;
  }
  const double inv = 1.0 / nj;
#pragma unroll
  for (int i = 0; i < RPT; ++i) y[i][J] *= inv;
}

template <int BS, int J>
struct MgsUnroll {
  __device__ __forceinline__ static void run(TileCtx& T, FSmem& S, double (&y)[RPT][BS],
                                             double tau, int& par) {
    mgs_column<BS, J>(T, S, y, tau, par);
    MgsUnroll<BS, J + 1>::run(T, S, y, tau, par);
  }
};
template <int BS>
struct MgsUnroll<BS, BS> {
  __device__ __forceinline__ static void run(TileCtx&, FSmem&, double (&)[RPT][BS], double, int&) {}
};

__host__ __device__ constexpr int pow2ceil(int v) { return v <= 2 ? 2 : v <= 4 ? 4 : v <= 8 ? 8 : v <= 16 ? 16 : 32; }

// ---- one-reduction-per-column CGS2 (delayed reorthogonalization) ----------
// Step S (1..BS) finalizes column J = S - 1 and runs the first pass of column S
// with ONE CTA reduction of
//   a = U_{<J}^T v_J, d = v_J^T v_J       (second pass of column J)
//   b = U_{<J}^T y_S, c = v_J^T y_S       (first pass of column S)
// where v_J is column J after its first pass; then
//   v_J <- v_J - U a,  n_J^2 = d - |a|^2 (Pythagoras), u_J = v_J / n_J,
//   u_J^T y_S = (c - a^T b) / n_J,  y_S <- y_S - U_{<J} b - u_J (u_J^T y_S).
// Same two-pass Gram-Schmidt as the reference's panel_mgs (each column is
// projected twice against every earlier column before its norm is taken), in
// half the synchronizations of column-wise CGS2.  A deficient column J
// (n_J < tau) is replaced exactly as in panel_mgs, and column S then takes a
// full first pass against the final columns.
template <int BS, int SS>
__device__ __forceinline__ void dcgs_step(TileCtx& T, FSmem& S, double (&y)[RPT][BS], double tau,
                                          int& par) {
  constexpr int JA = SS - 1;
  if (JA >= T.wlim) return;  // uniform
  const bool hasb = SS < BS && SS < T.wlim;
  constexpr int CS = SS < BS ? SS : BS - 1;  // compile-time column index of y_S (unused if !hasb)
  constexpr int NV = SS < BS ? 2 * JA + 2 : JA + 1;
  constexpr int N = pow2ceil(NV);
  constexpr int SH = (N == 2 ? 4 : N == 4 ? 3 : N == 8 ? 2 : N == 16 ? 1 : 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double part[N];
#pragma unroll
  for (int p = 0; p < N; ++p) {
    double v = 0.0;
    if (p < JA) {
#pragma unroll
      for (int i = 0; i < RPT; ++i) v += y[i][p] * y[i][JA];
    } else if (p == JA) {
#pragma unroll
      for (int i = 0; i < RPT; ++i) v += y[i][JA] * y[i][JA];
    } else if (SS < BS && p < 2 * JA + 1) {
      if (hasb) {
#pragma unroll
        for (int i = 0; i < RPT; ++i) v += y[i][p - JA - 1] * y[i][CS];
      }
    } else if (SS < BS && p == 2 * JA + 1) {
      if (hasb) {
#pragma unroll
        for (int i = 0; i < RPT; ++i) v += y[i][JA] * y[i][CS];
      }
    }
    part[p] = v;
  }
  const double red = warp_reduce_scatter<N>(part);
  double* wp = S.wpart + par * (FW * 32);
  par ^= 1;
  if ((lane & ((1 << SH) - 1)) == 0) wp[warp * 32 + (lane >> SH)] = red;
  cbar();
  double val = 0.0;
  if (lane < NV) {
    double h0 = 0.0, h1 = 0.0;
#pragma unroll
    for (int w = 0; w < FW; w += 2) {
      h0 += wp[w * 32 + lane];
      h1 += wp[(w + 1) * 32 + lane];
    }
    val = h0 + h1;
  }
  // R bookkeeping by warp 0: R(:,J) += a ; R(:,S) += b
  if (warp == 0) {
    if (lane < JA) S.Rp[lane + JA * BS] += val;
    if (hasb && lane > JA && lane < 2 * JA + 1) S.Rp[(lane - JA - 1) + CS * BS] += val;
  }
  double a[JA > 0 ? JA : 1];
#pragma unroll
  for (int p = 0; p < JA; ++p) a[p] = __shfl_sync(0xffffffffu, val, p);
  const double d = __shfl_sync(0xffffffffu, val, JA);
  double asq = 0.0;
#pragma unroll
  for (int p = 0; p < JA; ++p) asq += a[p] * a[p];
  // second pass of column J
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int p = 0; p < JA; p += 2) {
      s0 += a[p] * y[i][p];
      if (p + 1 < JA) s1 += a[p + 1] * y[i][p + 1];
    }
    y[i][JA] -= s0 + s1;
  }
  double nj = sqrt(fmax(d - asq, 0.0));
  if (!(nj >= tau)) {
    nj = replace_column<BS, JA>(T, S, y, nj, par);
    if (threadIdx.x == 0) S.Rp[JA + JA * BS] = 0.0;
    const double inv = 1.0 / nj;
#pragma unroll
    for (int i = 0; i < RPT; ++i) y[i][JA] *= inv;
    if (SS < BS && hasb) cgs_pass_reg<BS, CS>(y, S, S.Rp + CS * BS, par);
    return;
  }
  if (threadIdx.x == 0) S.Rp[JA + JA * BS] = nj;
  const double inv = 1.0 / nj;
#pragma unroll
  for (int i = 0; i < RPT; ++i) y[i][JA] *= inv;
  if (SS < BS && hasb) {
    double bb[JA > 0 ? JA : 1];
    double ab = 0.0;
#pragma unroll
    for (int p = 0; p < JA; ++p) {
      bb[p] = __shfl_sync(0xffffffffu, val, JA + 1 + p);
      ab += a[p] * bb[p];
    }
    const double c = __shfl_sync(0xffffffffu, val, 2 * JA + 1);
    const double beta = (c - ab) * inv;
    if (threadIdx.x == 0) S.Rp[JA + CS * BS] += beta;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      double s0 = beta * y[i][JA], s1 = 0.0;
#pragma unroll
      for (int p = 0; p < JA; p += 2) {
        s0 += bb[p] * y[i][p];
        if (p + 1 < JA) s1 += bb[p + 1] * y[i][p + 1];
      }
      y[i][CS] -= s0 + s1;
    }
  }
}

template <int BS, int SS>
struct DcgsUnroll {
  __device__ __forceinline__ static void run(TileCtx& T, FSmem& S, double (&y)[RPT][BS],
                                             double tau, int& par) {
    dcgs_step<BS, SS>(T, S, y, tau, par);
    DcgsUnroll<BS, SS + 1>::run(T, S, y, tau, par);
  }
};
template <int BS>
struct DcgsUnroll<BS, BS + 1> {
  __device__ __forceinline__ static void run(TileCtx&, FSmem&, double (&)[RPT][BS], double, int&) {}
};

template <int BS>
__device__ void panel_r_update(FSmem& S, int sweep);

template <int NT>
__device__ void panel_sweep(TileCtx& T, FSmem& S, int sweep, double tau) {
  constexpr int BS = NT * 8;
  for (int e = threadIdx.x; e < BS * BS; e += FT) S.Rp[e] = 0.0;
  if (sweep == 0)
    for (int j = threadIdx.x; j < BS; j += FT) {
      S.defi[j] = 0;
      S.tiny[j] = 0.0;
    }
  double y[RPT][BS];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int r = threadIdx.x + i * FT;
#pragma unroll
    for (int c = 0; c < BS; ++c) y[i][c] = r < T.rows ? S.Y[r + c * T.ldy] : 0.0;
  }
  cbar();
  int par = 0;
  // one reduction per column up to 16 columns (2j + 2 <= 32 reduced values per
  // step); the 32-column recompression panel keeps the column-wise CGS2
  if constexpr (BS <= 16) DcgsUnroll<BS, 1>::run(T, S, y, tau, par);
  else MgsUnroll<BS, 0>::run(T, S, y, tau, par);
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int r = threadIdx.x + i * FT;
    if (r < T.rows) {
#pragma unroll
      for (int c = 0; c < BS; ++c) S.Y[r + c * T.ldy] = y[i][c];
    }
  }
  cbar();
  panel_r_update<BS>(S, sweep);
}

// R <- Rp R   (R = I before the first sweep)
template <int BS>
__device__ void panel_r_update(FSmem& S, int sweep) {
  const int w = BS;
  if (sweep == 0) {
    for (int e = threadIdx.x; e < w * w; e += FT) S.R[e] = S.Rp[e];
  } else {
    for (int e = threadIdx.x; e < w * w; e += FT) {
      const int p = e % w, jj = e / w;
      double sum = 0.0;
      for (int tt = p; tt <= jj; ++tt) sum += S.Rp[p + tt * w] * S.R[tt + jj * w];
      S.Rt[e] = p <= jj ? sum : 0.0;
    }
    cbar();
    for (int e = threadIdx.x; e < w * w; e += FT) S.R[e] = S.Rt[e];
  }
  cbar();
}

// ---- second orthogonalization sweep as one Gram product ---------------------
// After sweep 1 the panel is orthonormal and orthogonal to Q to O(eps), so
// sweep 2's {C = Q^T Y, Y -= Q C, panel MGS2} is, to rounding, Y <- (Y - QC) R2^{-1}
// with R2 = chol((Y - QC)^T (Y - QC)) = chol(G - C^T C), G = Y^T Y = I + F,
// ||F|| = O(eps) and C^T C = O(eps^2).  To first order (the dropped terms are
// O(||F||^2) = O(eps^2)):
//   R2     = I + striu(F) + diag(F)/2        (what MGS2 accumulates: R2_ij = y_i^T y_j)
//   R2^-1  = I - striu(F) - diag(F)/2
// so the sweep is
//   [C; G] = [Q | Y]^T Y                 one DMMA product (q + bs) x bs
//   Y <- [Y | Q] [R2^-1; -C R2^-1]       one DMMA product, in place
// with no serial factorization.  No column can deflate in this sweep when
// tau < 1/4 (unit columns); the caller runs the column-wise sweep otherwise,
// and also when |F| > 1e-6 anywhere (a panel that is not orthonormal).
// Returns false (uniform) when the fast path does not apply.  R2 -> S.Rp.
template <int NT>
__device__ bool sweep2_gram(const FusedSlot& sl, TileCtx& T, FSmem& S, double* coef,
                            int* s_ok) {
  constexpr int BS = NT * 8;
  const int q = T.q, rows = T.rows, ldy = T.ldy, ldc = (q + 1) & ~1;
  const int ldk = (q + BS + 1) & ~1;
  double* G = S.Rt;  // bs x bs
  if (threadIdx.x == 0) *s_ok = 1;
  tn16<NT>(
      q + BS, rows,
      [&](int m) {
        return m < q ? (const double*)(sl.Q + (long long)m * rows)
                     : (const double*)(S.Y + (long long)(m - q) * ldy);
      },
      [&](int n) { return (const double*)(S.Y + (long long)n * ldy); }, [](int) { return 1.0; },
      [&](int m, int n, double v) {
        if (m < q) sl.Cq[m + (long long)n * ldc] = v;
        else G[(m - q) + n * BS] = v;
      },
      S.part);  // ends with a barrier
  for (int e = threadIdx.x; e < BS * BS; e += FT) {
    const int i = e % BS, j = e / BS;
    const double f = G[e] - (i == j ? 1.0 : 0.0);
    if (!(fabs(f) <= 1e-6)) *s_ok = 0;  // benign race: every writer stores 0
    const double r = i < j ? f : i == j ? 1.0 + 0.5 * f : 0.0;
    S.Rp[e] = r;
    coef[i + (long long)j * ldk] = i == j ? 1.0 - 0.5 * f : i < j ? -f : 0.0;
  }
  cbar();
  if (!*s_ok) return false;
  // coef rows bs..bs+q-1: -C R2^{-1}
  for (int e = threadIdx.x; e < q * BS; e += FT) {
    const int i = e % q, j = e / q;
    double v = 0.0;
    for (int l = 0; l <= j; ++l) v += sl.Cq[i + (long long)l * ldc] * coef[l + (long long)j * ldk];
    coef[BS + i + (long long)j * ldk] = -v;
  }
  cbar();
  nn16<NT>(
      rows, q + BS,
      [&](int k) {
        return k < BS ? (const double*)(S.Y + (long long)k * ldy)
                      : (const double*)(sl.Q + (long long)(k - BS) * rows);
      },
      coef, ldk, [&](int m, int n, double v) { S.Y[m + n * ldy] = v; });
  return true;
}

// ---- in-CTA one-sided Jacobi SVD of the small core (svd_truncate, ----------
// dense_kernels.cpp:422-454): A (n x n, ld n) <- U Sigma, V <- right vectors
// (both unsorted); sig[] the column norms; perm[] orders them descending (ties
// by index, like the batched kernel); returns #{sigma > cut}.
__device__ __noinline__ int cta_jacobi_svd(double* A, double* V, double* sig, int* perm, int n, double cut,
                              double* wred, int* flag) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < n * n; e += FT) V[e] = (e % n == e / n) ? 1.0 : 0.0;
  double f = 0.0;
  for (int e = threadIdx.x; e < n * n; e += FT) f += A[e] * A[e];
  f = cta_sum(f, wred);
  const double tiny2 = f * 1e-34;
  const double tol = fmax(1e-15, 2.0 * sqrt((double)n) * 2.220446049250313e-16);
  const int nn = n + (n & 1);
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    cbar();
    for (int step = 0; step < nn - 1; ++step) {
      for (int pi = warp; pi < nn / 2; pi += FW) {
        const int p = (step + pi) % (nn - 1);
        const int q = pi == 0 ? nn - 1 : (step - pi + nn - 1) % (nn - 1);
        if (p >= n || q >= n) continue;
        double* ap = A + p * n;
        double* aq = A + q * n;
        double al = 0, be = 0, ga = 0;
        for (int r = lane; r < n; r += 32) {
          al += ap[r] * ap[r];
          be += aq[r] * aq[r];
          ga += ap[r] * aq[r];
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (al > tiny2 && be > tiny2 && ga * ga > tol * tol * (al * be)) {
          const double dl = be - al;
          const double tt =
              (dl >= 0 ? 2.0 * ga : -2.0 * ga) / (fabs(dl) + sqrt(dl * dl + 4.0 * ga * ga));
          const double c = rsqrt(1.0 + tt * tt), sn = c * tt;
          for (int r = lane; r < n; r += 32) {
            const double x = ap[r], y = aq[r];
            ap[r] = c * x - sn * y;
            aq[r] = sn * x + c * y;
          }
          double* vp = V + p * n;
          double* vq = V + q * n;
          for (int r = lane; r < n; r += 32) {
            const double x = vp[r], y = vq[r];
            vp[r] = c * x - sn * y;
            vq[r] = sn * x + c * y;
          }
          if (lane == 0) *flag = 1;
        }
      }
      cbar();
    }
    if (!*flag) break;
    cbar();
  }
  for (int p = warp; p < n; p += FW) {
    double v = 0.0;
    for (int r = lane; r < n; r += 32) v += A[p * n + r] * A[p * n + r];
    v = warp_sum(v);
    if (lane == 0) sig[p] = sqrt(v);
  }
  cbar();
  int cnt = 0;
  for (int p = threadIdx.x; p < n; p += FT) {
    const double sp = sig[p];
    int rk = 0;
    for (int q = 0; q < n; ++q) rk += (sig[q] > sp || (sig[q] == sp && q < p)) ? 1 : 0;
    perm[rk] = p;
  }
  for (int p = 0; p < n; ++p) cnt += sig[p] > cut ? 1 : 0;
  cbar();
  return cnt;
}

// ---- producer warp: the tile's exact tlr::Rng gaussian stream -------------
// Runs concurrently with the consumer warps, keeping the ring buffer ahead of
// the consumption cursor (Marsaglia polar pairs of mt19937_64 draws,
// util.hpp:24-53, the same sequence cta_generate appends).  Publishes the
// produced count through shared memory after a block-scope fence.
constexpr int PQ = 128;  // polar pairs per producer batch
struct ProdSmem {
  uint64_t mt[MT_N];
  double pu[PQ], pv[PQ], pq[PQ];
};
__device__ void stream_producer(const FusedArgs& A, int s, volatile long long* s_rel,
                                volatile long long* s_av, volatile int* s_stop, ProdSmem& P) {
  const int lane = threadIdx.x & 31;
  RngState* g = &A.G.st[s];
  double* buf = A.G.buf + (long long)s * A.G.cap;
  const long long cap = A.G.cap;
  for (int i = lane; i < MT_N; i += 32) P.mt[i] = g->mt[i];
  int idx = g->idx;
  long long have = *s_av;
  __syncwarp();
  while (!*s_stop) {
    const long long rel = *s_rel;  // everything before it is consumed and released
    long long room = cap - (have - rel);
    if (room < 2 * PQ) {
      __nanosleep(200);
      continue;
    }
    // accept PQ polar pairs (cheap integer/FP work, ballot-compacted into smem)
    int got = 0;
    while (got < PQ) {
      if (idx >= MT_N) {
        warp_mt_twist(P.mt);
        idx = 0;
      }
      int n_att = (MT_N - idx) / 2;
      if (n_att > 32) n_att = 32;
      bool acc = false;
      double u = 0.0, v = 0.0, q = 0.0;
      if (lane < n_att) {
        u = 2.0 * mt_uniform(mt_temper(P.mt[idx + 2 * lane])) - 1.0;
        v = 2.0 * mt_uniform(mt_temper(P.mt[idx + 2 * lane + 1])) - 1.0;
        q = u * u + v * v;
        acc = (q < 1.0) && (q != 0.0);
      }
      const unsigned mask = __ballot_sync(0xffffffffu, acc);
      const int rank = __popc(mask & ((1u << lane) - 1u));
      const int nacc = __popc(mask), left = PQ - got;
      if (acc && rank < left) {
        P.pu[got + rank] = u;
        P.pv[got + rank] = v;
        P.pq[got + rank] = q;
      }
      if (nacc >= left) {
        unsigned m2 = mask;
        for (int t = 0; t < left - 1; ++t) m2 &= m2 - 1;
        idx += 2 * __ffs(m2);
        got = PQ;
      } else {
        idx += 2 * n_att;
        got += nacc;
      }
    }
    __syncwarp();
    // transform: PQ / 32 independent pairs per lane (log / sqrt latency overlapped)
#pragma unroll
    for (int i = 0; i < PQ / 32; ++i) {
      const int e = lane + 32 * i;
      const double q = P.pq[e];
      const double f = sqrt(-2.0 * log(q) / q);
      const long long p0 = (have + 2LL * e) % cap;  // pairs never straddle the wrap
      buf[p0] = P.pu[e] * f;
      buf[p0 + 1] = P.pv[e] * f;
    }
    have += 2LL * PQ;
    __threadfence();  // ring values are read by the leader and (clusters) its helpers
    __syncwarp();
    if (lane == 0) *s_av = have;
  }
  __syncwarp();
  for (int i = lane; i < MT_N; i += 32) g->mt[i] = P.mt[i];
  if (lane == 0) {
    g->idx = idx;
    g->have_cached = 0;
    A.G.avail[s] = have;
  }
}

// ---- exit projection + SVD recompression of one converged tile ------------
// (ara.cpp:380-398 and recompress_pair, ara.cpp:201-211), in the tile's CTA
// while slower tiles are still sampling:
//   B = E^T Q (cols x q) -> Z R = orthog(empty, B) (same panel MGS2, same stream)
//   -> SVD of R cut at (1 - 1/eta) eps -> Uo = Q V_s, Vo = Z U_s sigma.
template <int NTQ>
__device__ __noinline__ int recompress_tile(const FusedArgs& A, const FusedSlot& sl, TileCtx& T, FSmem& S,
                               int q, int* s_flag) {
  constexpr int BSQ = NTQ * 8;
  const int rows = sl.rows, cols = A.cols, ldy = T.ldy;
  const int kA = sl.kA, KW = kA + A.K, ldw = (KW + 1) & ~1;
  // projection into the smem panel (columns >= q hold don't-care values)
  if (sl.Ad) {
    tn16<NTQ>(
        cols, rows, [&](int m) { return sl.Ad + (long long)m * sl.ldad; },
        [&](int n) { return (const double*)(sl.Q + (long long)n * rows); }, [](int) { return 1.0; },
        [&](int m, int n, double v) { S.Y[m + n * ldy] = v; }, S.part);
  } else {
    tn16<NTQ>(
        KW, rows,
        [&](int m) { return m < kA ? sl.UA + (long long)m * rows : sl.H + (long long)(m - kA) * rows; },
        [&](int n) { return (const double*)(sl.Q + (long long)n * rows); },
        [&](int m) { return m < kA ? 1.0 : -1.0; },
        [&](int m, int n, double v) { sl.W[m + (long long)n * ldw] = v; }, S.part);
    nn16<NTQ>(
        cols, KW,
        [&](int k) { return k < kA ? sl.VA + (long long)k * cols : A.Ucat + (long long)(k - kA) * cols; },
        sl.W, ldw, [&](int m, int n, double v) { S.Y[m + n * ldy] = v; });
  }
  // orthog(empty, B): tau from the q real columns, two panel MGS2 sweeps
  TileCtx T2 = T;
  T2.rows = cols;
  T2.q = 0;
  T2.wlim = q;
  __shared__ double s_tau2;
  {
    double f = 0.0;
    for (int r = threadIdx.x; r < cols; r += FT)
      for (int c = 0; c < q; ++c) f += S.Y[r + c * ldy] * S.Y[r + c * ldy];
    f = cta_sum(f, S.wred);
    if (threadIdx.x == 0) {
      const double tau = 100.0 * DBL_EPSILON * sqrt(f);
      s_tau2 = tau == 0.0 ? DBL_MIN : tau;
    }
    cbar();
  }
  panel_sweep<NTQ>(T2, S, 0, s_tau2);
  panel_sweep<NTQ>(T2, S, 1, s_tau2);
  // R (q x q, ld q) with the deficient-column convention of orthog
  double* Ra = S.part;          // q x q
  double* Va = S.part + q * q;  // q x q
  for (int e = threadIdx.x; e < q * q; e += FT) {
    const int i = e % q, j = e / q;
    double v = S.R[i + j * BSQ];
    if (S.defi[j]) v = (i == j) ? S.tiny[j] : 0.0;
    Ra[e] = v;
  }
  cbar();
  double* sig = S.sig;
  int* perm = S.perm;
  const int r = cta_jacobi_svd(Ra, Va, sig, perm, q, A.cut, S.wred, s_flag);
  // Uo = Q V_s ; Vo = Z (U_s sigma)   (first r singular triplets, descending)
  for (int e = threadIdx.x; e < rows * r; e += FT) {
    const int row = e % rows, c = e / rows;
    const double* v = Va + perm[c] * q;
    double acc = 0.0;
    for (int k = 0; k < q; ++k) acc += sl.Q[row + (long long)k * rows] * v[k];
    sl.Uo[row + (long long)c * rows] = acc;
  }
  for (int e = threadIdx.x; e < cols * r; e += FT) {
    const int row = e % cols, c = e / cols;
    const double* u = Ra + perm[c] * q;
    double acc = 0.0;
    for (int k = 0; k < q; ++k) acc += S.Y[row + k * ldy] * u[k];
    sl.Vo[row + (long long)c * cols] = acc;
  }
  cbar();
  return r;
}

// ---- cluster split of the sampling products (CL CTAs per tile) ---------------
// The leader CTA (cluster rank 0) runs the tile's whole ARA; the CL - 1 helper
// CTAs join each round's two sampling products, which are the largest part of a
// round:  W = [V^A | -U_k,:]^T Omega is split by rows of W (each CTA a slice of
// the kA + K reduction vectors, into the global scratch W), and Y = [U^A | H] W
// by tile rows (helpers store their rows straight into the leader's shared
// panel through DSMEM).  Per round:  leader publishes Omega (go) -> every CTA
// computes its W slice -> all-to-all "W done" -> every CTA computes its Y rows
// -> helpers signal "Y done" to the leader.  Signalling is by mbarriers with
// cluster-scope release/acquire, so the leader's free-running producer warp
// needs no cluster-wide barrier.
struct ClusterSync {
  uint64_t go, wdone, ydone;
  unsigned long long om;  // Omega of the round (written by the leader)
  int run;                // 1: another round, 0: the tile is done
};

template <int NT>
__device__ __forceinline__ void sample_slice(const FusedArgs& A, const FusedSlot& sl, FSmem& S,
                                             const double* Om, int crank, int CL, int rows,
                                             int ldy, ClusterSync& cs, unsigned& wd_ph) {
  const int cols = A.cols, kA = sl.kA, KW = kA + A.K, ldw = (KW + 1) & ~1;
  // W rows of this CTA, in 8-row DMMA tiles
  const int mt = (KW + 7) / 8;
  const int m0 = min(KW, 8 * (crank * mt / CL)), m1 = min(KW, 8 * ((crank + 1) * mt / CL));
  if (m1 > m0)
    tn16<NT>(
        m1 - m0, cols,
        [&](int m) {
          m += m0;
          return m < kA ? sl.VA + (long long)m * cols : A.Ucat + (long long)(m - kA) * cols;
        },
        [&](int n) { return Om + (long long)n * cols; },
        [&](int m) { return m + m0 < kA ? 1.0 : -1.0; },
        [&](int m, int n, double v) { sl.W[m + m0 + (long long)n * ldw] = v; }, S.part);
  __threadfence();  // W is read by the other CTAs of the cluster
  cbar();
  if (threadIdx.x == 0)
    for (int c = 0; c < CL; ++c) mbar_arrive_remote(map_shared(&cs.wdone, c));
  mbar_wait_cluster(&cs.wdone, wd_ph);
  wd_ph ^= 1;
  // Y rows of this CTA, in 16-row groups
  const int ng = (rows + 15) / 16;
  const int r0 = 16 * (crank * ng / CL), r1 = min(rows, 16 * ((crank + 1) * ng / CL));
  if (r1 <= r0) return;
  auto acolY = [&](int k) {
    return (k < kA ? sl.UA + (long long)k * rows : sl.H + (long long)(k - kA) * rows) + r0;
  };
  if (crank == 0) {
    nn16<NT>(r1 - r0, KW, acolY, sl.W, ldw,
             [&](int m, int n, double v) { S.Y[m + r0 + n * ldy] = v; });
  } else {
    const unsigned ybase = map_shared(S.Y, 0);
    nn16<NT>(r1 - r0, KW, acolY, sl.W, ldw, [&](int m, int n, double v) {
      st_cluster_f64(ybase + 8u * (unsigned)(m + r0 + n * ldy), v);
    });
  }
}

template <int NT, int CL>
__global__ void __launch_bounds__(FTP, 1) ara_fused_kernel(FusedArgs A) {
  extern __shared__ __align__(16) double fsm[];
  const int s = blockIdx.x / CL;
  const int crank = CL > 1 ? (int)cluster_ctarank() : 0;
  const FusedSlot& sl = A.slots[s];
  const int rows = sl.rows, cols = A.cols, bs = NT * 8;
  constexpr int BQ = NT * 8 > FUSED_QMAX ? NT * 8 : FUSED_QMAX;
  const int ldy = A.ldy;
  FSmem S;
  {
    double* p = fsm;
    S.Y = p;
    p += A.ysz;
    S.R = p; p += BQ * BQ;
    S.Rp = p; p += BQ * BQ;
    S.Rt = p; p += BQ * BQ;
    S.part = p; p += (PART_UNITS * 64 * NT > 2 * FUSED_QMAX * FUSED_QMAX
                          ? PART_UNITS * 64 * NT : 2 * FUSED_QMAX * FUSED_QMAX);
    S.cbuf = p; p += BQ;
    S.wpart = p; p += 2 * FW * 32;
    S.wred = p; p += FW;
    S.tiny = p; p += BQ;
    S.cn = p; p += BQ;
    S.nm = p; p += BQ;
    S.recent = p; p += A.window;
    S.keep = reinterpret_cast<int*>(p); p += BQ;
    S.sig = p; p += FUSED_QMAX;
    S.perm = reinterpret_cast<int*>(p); p += FUSED_QMAX;
    S.defi = reinterpret_cast<uint8_t*>(p);
  }
  __shared__ long long s_cur, s_av, s_rel;
  __shared__ int s_q, s_done, s_nkeep, s_rounds, s_conv, s_rcount, s_rpos, s_stop, s_ok;
  __shared__ double s_tau;
  __shared__ ProdSmem prod;
  __shared__ ClusterSync csync;
  if (CL > 1) {
    if (threadIdx.x == 0) {
      mbar_init(&csync.go, 1);
      mbar_init(&csync.wdone, CL);
      mbar_init(&csync.ydone, CL - 1);
    }
    // every CTA's barriers exist before anyone signals them (all threads)
    cluster_sync_all();
  }
  if (CL > 1 && crank > 0) {
    // ---- helper CTA: the tile's sampling products, round by round ----------
    if (threadIdx.x >= FT) return;
    unsigned go_ph = 0, wd_ph = 0;
    const unsigned ydone0 = map_shared(&csync.ydone, 0);
    const int ldy = A.ldy;
    FSmem S;
    S.Y = fsm;
    S.part = fsm + A.ysz + 3 * (NT * 8 > FUSED_QMAX ? NT * 8 : FUSED_QMAX) *
                                   (NT * 8 > FUSED_QMAX ? NT * 8 : FUSED_QMAX);
    while (true) {
      mbar_wait_cluster(&csync.go, go_ph);
      go_ph ^= 1;
      if (!csync.run) break;
      sample_slice<NT>(A, sl, S, (const double*)csync.om, crank, CL, sl.rows, ldy, csync, wd_ph);
      fence_cluster();
      cbar();
      if (threadIdx.x == 0) mbar_arrive_remote(ydone0);
    }
    return;
  }
  if (threadIdx.x == 0) {
    s_cur = A.G.cursor[s];
    s_av = A.G.avail[s];
    s_rel = s_cur;
    s_stop = 0;
    s_q = 0;
    s_done = sl.cap <= 0;
    s_rounds = 0;
    s_conv = 0;
    s_rcount = 0;
    s_rpos = 0;
  }
  __syncthreads();
  if (threadIdx.x >= FT) {
    stream_producer(A, s, &s_rel, &s_av, &s_stop, prod);
    return;
  }
  TileCtx T{&sl, A.G, s, rows, cols, bs, ldy, 0, &s_cur, &s_av, bs, A.mgs_passes, A.dcgs};
  const double* gb = A.G.buf + (long long)s * A.G.cap;
  const int kA = sl.kA, K = A.K, KW = kA + K;
  const int ldw = (KW + 1) & ~1;
  // TMA staging for the sampling products: after the bs-column Y panel, inside
  // the (FUSED_QMAX-column) panel region that recompression uses later
  __shared__ __align__(8) uint64_t s_sbar[2];
  Stager stg{nullptr, s_sbar};
  unsigned sph = 0;
  const bool use_tma = CL == 1 && A.stage && NT <= 2 && cols <= MAXROWS && rows <= MAXROWS;
  unsigned wd_ph = 0, yd_ph = 0;
  // leader: release the helpers (one more round, or done)
  auto publish = [&](const double* om, int run) {
    if (CL > 1 && threadIdx.x == 0)
      for (int c = 1; c < CL; ++c) {
        st_cluster_u64(map_shared(&csync.om, c), (unsigned long long)om);
        st_cluster_u32(map_shared(&csync.run, c), (unsigned)run);
        mbar_arrive_remote(map_shared(&csync.go, c));
      }
  };
  if (use_tma) {
    stg.buf = S.Y + (((long long)ldy * bs + 15) & ~15LL);
    if (threadIdx.x == 0) {
      mbar_init(&s_sbar[0], 1);
      mbar_init(&s_sbar[1], 1);
    }
    cbar();
  }

  long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long t_prev = clock64(), t_begin = t_prev;
  auto tick = [&](int slot) {
    if (A.prof && threadIdx.x == 0) {
      const long long t = clock64();
      pc[slot] += t - t_prev;
      t_prev = t;
    }
  };
  double fl = 0.0;  // algorithmic flops of this CTA (thread 0)
  while (!s_done && s_rounds < A.max_rounds) {
    if (threadIdx.x == 0) {
      const double r = rows, c = cols, kw = sl.Ad ? 0.0 : KW, b2 = bs;
      fl += sl.Ad ? 2.0 * r * c * b2 : 2.0 * kw * (c + r) * b2;  // sampling
      fl += 2.0 * r * b2 + 4.0 * 2.0 * r * b2 * b2;               // tau + panel MGS2 x 2 sweeps
      fl += 2.0 * 2.0 * 2.0 * r * s_q * b2;                       // BGS deflation, 2 sweeps
    }
    // ---- draw: make sure Omega and every possible replacement are available
    const double* Om;
    {
      const long long need = (long long)cols * bs;  // replacements wait on demand
      {
        // the previous round is complete: release its values to the producer
        if (threadIdx.x == 0) *(volatile long long*)&s_rel = s_cur;
        volatile long long* av = &s_av;
        const long long c0 = s_cur;
        while (*av - c0 < need) __nanosleep(64);
        __threadfence_block();
      }
      const long long cur = s_cur, n = (long long)cols * bs;
      const long long start = cur % A.G.cap;
      if (start + n <= A.G.cap) {
        Om = gb + start;  // contiguous in the ring: read in place
      } else {
        ring_copy(gb, A.G.cap, cur, n, sl.Om, FT);
        Om = sl.Om;
      }
      cbar();
      if (threadIdx.x == 0) s_cur = cur + n;
    }
    tick(0);
    // ---- sample -------------------------------------------------------------
    if (sl.Ad) {
      // dense operator: Y = A_tile Omega
      nn16<NT>(
          rows, cols, [&](int k) { return sl.Ad + (long long)k * sl.ldad; }, Om, cols,
          [&](int m, int n, double v) { S.Y[m + n * ldy] = v; });
    } else {
      auto acolW = [&](int m) {
        return m < kA ? sl.VA + (long long)m * cols : A.Ucat + (long long)(m - kA) * cols;
      };
      auto acolY = [&](int k) {
        return k < kA ? sl.UA + (long long)k * rows : sl.H + (long long)(k - kA) * rows;
      };
      auto sgnW = [&](int m) { return m < kA ? 1.0 : -1.0; };
      auto outW = [&](int m, int n, double v) { sl.W[m + (long long)n * ldw] = v; };
      auto epiY = [&](int m, int n, double v) { S.Y[m + n * ldy] = v; };
      if (CL > 1) {
        __threadfence();  // a wrapped Omega was assembled in global memory by this CTA
        cbar();
        publish(Om, 1);
        sample_slice<NT>(A, sl, S, Om, 0, CL, rows, ldy, csync, wd_ph);
        mbar_wait_cluster(&csync.ydone, yd_ph);  // the helpers' rows are in S.Y
        yd_ph ^= 1;
        cbar();
      } else if (use_tma) {
        // W = [V^A | -U_k,:]^T Omega   (KW x bs, ld ldw), then Y = [U^A | H] W
        tn16_tma<NT>(KW, cols, acolW, [&](int n) { return Om + (long long)n * cols; }, sgnW, outW,
                     S.part, stg, sph);
        nn16_tma<NT>(rows, KW, acolY, sl.W, ldw, epiY, stg, sph);
      } else {
        tn16<NT>(KW, cols, acolW, [&](int n) { return Om + (long long)n * cols; }, sgnW, outW,
                 S.part);
        nn16<NT>(rows, KW, acolY, sl.W, ldw, epiY);
      }
    }
    tick(1);
    // ---- orthog (dense_kernels.cpp:379-420) ------------------------------------
    {
      double f = 0.0;
      for (int r = threadIdx.x; r < rows; r += FT)
        for (int c = 0; c < bs; ++c) {
          const double y = S.Y[r + c * ldy];
          f += y * y;
        }
      f = cta_sum(f, S.wred);
      if (threadIdx.x == 0) {
        double tau = 100.0 * DBL_EPSILON * sqrt(f);
        s_tau = tau == 0.0 ? DBL_MIN : tau;
      }
      cbar();
    }
    T.q = s_q;
    tick(2);
    for (int sweep = 0; sweep < 2; ++sweep) {
      if (sweep == 1 && A.fast_sweep2 && s_tau < 0.25 &&
          sweep2_gram<NT>(sl, T, S, sl.Cq + (long long)((sl.cap + 1) & ~1) * bs, &s_ok)) {
        panel_r_update<NT * 8>(S, 1);
        tick(4);
        break;
      }
      if (T.q > 0) {
        const int q = T.q, ldc = (q + 1) & ~1;
        // C = Q^T Y
        tn16<NT>(
            q, rows, [&](int m) { return sl.Q + (long long)m * rows; },
            [&](int n) { return (const double*)(S.Y + n * ldy); }, [](int) { return 1.0; },
            [&](int m, int n, double v) { sl.Cq[m + (long long)n * ldc] = v; }, S.part);
        // Y -= Q C
        nn16<NT>(
            rows, q, [&](int k) { return sl.Q + (long long)k * rows; }, sl.Cq, ldc,
            [&](int m, int n, double v) { S.Y[m + n * ldy] -= v; });
      }
      tick(3);
      panel_sweep<NT>(T, S, sweep, s_tau);
      tick(4);
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
    cbar();
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
    cbar();
    {
      const int nk = s_nkeep, q0 = s_q - s_nkeep;
      for (int e = threadIdx.x; e < nk * rows; e += FT) {
        const int c = e / rows, r = e % rows;
        sl.Q[(long long)(q0 + c) * rows + r] = S.Y[r + S.keep[c] * ldy];
      }
    }
    cbar();
    tick(5);
  }
  publish(nullptr, 0);  // the helpers leave
  // ---- exit projection + recompression of this tile (q <= FUSED_QMAX) --------
  __shared__ int s_flag;
  if (A.recompress) {
    const int q = s_q;
    int rf = -1;
    if (q == 0) rf = 0;
    else if (q <= 16) rf = recompress_tile<2>(A, sl, T, S, q, &s_flag);
    else if (q <= FUSED_QMAX) rf = recompress_tile<4>(A, sl, T, S, q, &s_flag);
    if (threadIdx.x == 0) {
      A.rank_out[s] = rf;
      if (rf >= 0 && q > 0) {
        const double r = rows, c = cols, kw = sl.Ad ? 0.0 : KW, qq = q;
        fl += sl.Ad ? 2.0 * r * c * qq : 2.0 * kw * (r + c) * qq;  // exit projection
        fl += 4.0 * 2.0 * c * qq * qq + 2.0 * (r + c) * qq * rf;   // orthog of B + final products
      }
    }
  }
  if (threadIdx.x == 0 && A.flops_out) A.flops_out[s] = fl;
  if (threadIdx.x == 0) *(volatile int*)&s_stop = 1;
  if (A.prof && threadIdx.x == 0) {
    pc[6] = clock64() - t_begin;
    pc[7] = s_rounds;
    for (int i = 0; i < 8; ++i) A.prof[8LL * s + i] = pc[i];
  }
  if (threadIdx.x == 0) {
    A.qcols[s] = s_q;
    A.rounds[s] = s_rounds;
    A.conv[s] = s_conv;
    A.G.cursor[s] = s_cur;  // avail and the generator state: written by the producer
  }
}

size_t fused_smem_bytes(int maxrows, int bs, int window, int* ldy, long long* ysz) {
  int l = ((maxrows + 15) / 16) * 16 + 4;
  long long y = (long long)l * std::max(bs, FUSED_QMAX);
  if (bs <= 16) y = std::max(y, (((long long)l * bs + 15) & ~15LL) + 2LL * SCOL * SPAD);
  y = (y + 1) & ~1LL;
  *ldy = l;
  *ysz = y;
  const long long partn = std::max<long long>((long long)PART_UNITS * 64 * (bs / 8),
                                              2LL * FUSED_QMAX * FUSED_QMAX);
  const int bq = std::max(bs, FUSED_QMAX);
  long long d = y + 3LL * bq * bq + partn + bq + 2 * FW * 32 + FW + 2 * FUSED_QMAX +
                3LL * bq + window + bq /*keep ints*/ + bq;
  return (size_t)d * 8 + 64;
}

}  // namespace

bool ara_fused_supported(int maxrows, int bs, int window) {
  if (maxrows > MAXROWS) return false;  // callers also need even rows / cols
  // bs = 24 / 32 take the graph path (measured faster there; see ara.cu), so
  // only the 8- and 16-column instances are compiled
  if (bs != 8 && bs != 16) return false;
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

template <int NT, int CL>
void launch_fused(const FusedArgs& args, int T, size_t bytes, cudaStream_t st) {
  static size_t lim = enable_max_dyn_smem(ara_fused_kernel<NT, CL>);
  if (bytes > lim) throw CudaError("ara_fused: shared memory budget exceeded");
  if (CL == 1) {
    ara_fused_kernel<NT, CL><<<T, FTP, bytes, st>>>(args);
    return;
  }
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((unsigned)(T * CL));
  lc.blockDim = dim3(FTP);
  lc.dynamicSmemBytes = bytes;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  TLRG_CUDA(cudaLaunchKernelEx(&lc, ara_fused_kernel<NT, CL>, args));
}

void ara_fused(FusedArgs args, int T, int maxrows, cudaStream_t st, int cl) {
  if (T <= 0) return;
  const int bs = args.bs;
  // the panel stride must cover the exit projection B (cols x q) as well as
  // the tile rows: a column whose tiles are all shorter than the diagonal
  // block (n % b != 0, or a multi-GPU share holding only the short last tile)
  // would otherwise alias B's columns
  maxrows = std::max(maxrows, args.cols);
  if (maxrows > MAXROWS) throw CudaError("ara_fused: tile larger than the fused panel");
  long long ysz;
  size_t bytes = fused_smem_bytes(maxrows, bs, args.window, &args.ldy, &ysz);
  args.ysz = ysz;
  args.stg_half = 0;
  {
    // TMA-staged sampling operands: correct, but measured slower than the direct
    // 128-bit fragment loads at cfg2 (per-chunk barriers dominate) -> opt-in
    const char* e = std::getenv("TLRG_FUSED_TMA");
    args.stage = (bs <= 16 && e && e[0] == '1') ? 1 : 0;
  }
  if (cl > 1) args.stage = 0;
  if (bs == 8) {
    launch_fused<1, 1>(args, T, bytes, st);
  } else if (bs == 16) {
    if (cl >= 4) launch_fused<2, 4>(args, T, bytes, st);
    else if (cl == 2) launch_fused<2, 2>(args, T, bytes, st);
    else launch_fused<2, 1>(args, T, bytes, st);
  } else {
    throw CudaError("ara_fused: unsupported block size");
  }
  TLRG_CUDA(cudaGetLastError());
}

}  // namespace tlrg
