// Column step of the left-looking TLR factorization on the device:
//   column_setup : row-k concatenation U_k,: and the Gram blocks
//                  G_ij = V_ij^T [D_j] V_kj (one GEMM per j over the stored
//                  panel suffix), i.e. the j-sum of Eq. 1/Eq. 3 re-associated
//                  so that every ARA round streams only U^A and H_i.
//   column_H     : H_i = sum_j U_ij G_ij  (block-diagonal products)
//   column_ara   : dynamic-batched ARA (ara.cpp:302-419) with exact reference
//                  Gaussian streams, BGS2/MGS2 orthogonalisation, absorb and
//                  convergence on device, batched exit projection and SVD
//                  recompression.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <set>

#include <unordered_map>

#include "core.h"

namespace tlrg {


void column_setup(Ctx& C, const Matrix& M, int k, const DBlocks& D, ColumnSetup& cs) {
  const int b = M.b, nb = M.nb;
  cs = ColumnSetup();
  cs.k = k;
  cs.rk = M.rows(k);
  for (int j = 0; j < k; ++j) {
    int r = M.rank[M.t(k, j)];
    if (r > 0) {
      cs.J.push_back(j);
      cs.seg.push_back(cs.K);
      cs.K += r;
    }
  }
  if (cs.K == 0) return;
  const int K = cs.K, rk = cs.rk;
  cs.Ucat = C.buf<double>("Ucat", (size_t)rk * K);
  cs.Wcat = C.buf<double>("Wcat", (size_t)b * K);
  std::vector<CopyItem> cp;
  for (size_t jj = 0; jj < cs.J.size(); ++jj) {
    int j = cs.J[jj], r = M.rank[M.t(k, j)];
    cp.push_back({M.U[M.t(k, j)], cs.Ucat + (size_t)cs.seg[jj] * rk, rk, rk, rk, r});
    cp.push_back({M.V[M.t(k, j)], cs.Wcat + (size_t)cs.seg[jj] * b, b, b, b, r});
  }
  batched_copy(C.push(cp), (int)cp.size(), C.st);
  ++C.launches;
  if (D.on()) {
    // [D_j] V_kj for every j (Eq. 3), one launch
    std::vector<BdItem> bi;
    for (size_t jj = 0; jj < cs.J.size(); ++jj) {
      int j = cs.J[jj], r = M.rank[M.t(k, j)];
      bi.push_back({D.d + (size_t)j * b, D.e + (size_t)j * b, D.s2 + (size_t)j * b,
                    cs.Wcat + (size_t)cs.seg[jj] * b, r});
    }
    bd_apply_batched(C.push(bi), (int)bi.size(), b, b, C.st);
    ++C.launches;
  }
  // Gram blocks over the suffix i >= k of each panel j
  std::vector<const double*> suf(cs.J.size(), nullptr);
  std::vector<CopyItem> gather;
  size_t gathered = 0;
  cs.S.assign(cs.J.size(), 0);
  cs.goff.assign(cs.J.size(), 0);
  long long gtot = 0;
  for (size_t jj = 0; jj < cs.J.size(); ++jj) {
    int j = cs.J[jj];
    int S = 0;
    bool contiguous = true;
    const double* first = nullptr;
    for (int i = k; i < nb; ++i) {
      int r = M.rank[M.t(i, j)];
      if (r == 0) continue;
      const double* p = M.V[M.t(i, j)];
      if (!first) first = p;
      else if (p != first + (size_t)b * S) contiguous = false;
      S += r;
    }
    cs.S[jj] = S;
    cs.goff[jj] = gtot;
    gtot += (long long)S * M.rank[M.t(k, j)];
    if (contiguous) {
      suf[jj] = first;
    } else {
      gathered += (size_t)b * S;
    }
  }
  double* gbuf = gathered ? C.buf<double>("Vsuf", gathered) : nullptr;
  size_t goff2 = 0;
  for (size_t jj = 0; jj < cs.J.size(); ++jj) {
    if (suf[jj] || cs.S[jj] == 0) continue;
    int j = cs.J[jj];
    suf[jj] = gbuf + goff2;
    size_t col = 0;
    for (int i = k; i < nb; ++i) {
      int r = M.rank[M.t(i, j)];
      if (r == 0) continue;
      gather.push_back({M.V[M.t(i, j)], gbuf + goff2 + col * b, b, b, b, r});
      col += r;
    }
    goff2 += (size_t)b * cs.S[jj];
  }
  if (!gather.empty()) {
    batched_copy(C.push(gather), (int)gather.size(), C.st);
    ++C.launches;
  }
  cs.G = C.buf<double>("G", (size_t)std::max<long long>(gtot, 1));
  std::vector<GemmProblem> pr;
  for (size_t jj = 0; jj < cs.J.size(); ++jj) {
    if (cs.S[jj] == 0) continue;
    GemmProblem g{};
    g.A = suf[jj];
    g.lda = b;
    g.transA = 1;
    g.B = cs.Wcat + (size_t)cs.seg[jj] * b;
    g.ldb = b;
    g.C = cs.G + cs.goff[jj];
    g.ldc = cs.S[jj];
    g.M = cs.S[jj];
    g.N = M.rank[M.t(k, cs.J[jj])];
    g.K = b;
    g.alpha = 1.0;
    g.beta = 0.0;
    pr.push_back(g);
  }
  C.gemm(pr);
}

void column_H(Ctx& C, const Matrix& M, const ColumnSetup& cs, const std::vector<int>& targets,
              double* H, long long stride) {
  if (cs.K == 0 || targets.empty()) return;
  const int k = cs.k;
  // prefix of ranks inside each panel suffix: row offset of G_ij in G_j
  std::vector<BlockItem> items;
  items.reserve(targets.size() * cs.J.size());
  std::vector<std::vector<int>> pre(cs.J.size());
  for (size_t jj = 0; jj < cs.J.size(); ++jj) {
    int j = cs.J[jj];
    pre[jj].assign(M.nb - k + 1, 0);
    for (int i = k; i < M.nb; ++i) pre[jj][i - k + 1] = pre[jj][i - k] + M.rank[M.t(i, j)];
  }
  for (size_t t = 0; t < targets.size(); ++t) {
    int i = targets[t], ri = M.rows(i);
    for (size_t jj = 0; jj < cs.J.size(); ++jj) {
      int j = cs.J[jj];
      int kij = M.rank[M.t(i, j)];
      int kkj = M.rank[M.t(k, j)];
      BlockItem it{};
      it.U = kij ? M.U[M.t(i, j)] : nullptr;
      it.G = cs.G + cs.goff[jj] + pre[jj][i - k];
      it.ldg = std::max(cs.S[jj], 1);
      it.H = H + t * stride + (long long)cs.seg[jj] * ri;
      it.ldh = ri;
      it.rows = ri;
      it.kij = kij;
      it.kkj = kkj;
      items.push_back(it);
    }
  }
  block_products(C.push(items), (int)items.size(), M.b, C.st);
  ++C.launches;
}

// column_H with the T x J block list expanded on the device (tile-table mirror)
static void column_H_dev(Ctx& C, const Matrix& M, const ColumnSetup& cs,
                         const std::vector<int>& targets, double* H, long long stride) {
  if (cs.K == 0 || targets.empty() || cs.J.empty()) return;
  const int T = (int)targets.size(), nJ = (int)cs.J.size();
  std::vector<long long> cols((size_t)T + 5 * nJ);
  for (int t = 0; t < T; ++t) cols[t] = targets[t];
  for (int jj = 0; jj < nJ; ++jj) {
    cols[T + jj] = cs.J[jj];
    cols[T + nJ + jj] = cs.S[jj];
    cols[T + 2 * nJ + jj] = cs.seg[jj];
    cols[T + 3 * nJ + jj] = M.rank[M.t(cs.k, cs.J[jj])];
    cols[T + 4 * nJ + jj] = cs.goff[jj];
  }
  HProductArgs a{};
  a.cols = C.push(cols);
  a.rank = cs.d_rank;
  a.U = cs.d_U;
  a.G = cs.G;
  a.H = H;
  a.stride = stride;
  a.n = M.n;
  a.T = T;
  a.nJ = nJ;
  a.k = cs.k;
  a.b = M.b;
  h_products(a, C.st);
  ++C.launches;
}

std::vector<int> column_queue(const Matrix& M, int k) {
  std::vector<int> order;
  for (int i = k + 1; i < M.nb; ++i) order.push_back(i);
  // large stored ranks first, ties by i (ara.cpp:308-317)
  std::stable_sort(order.begin(), order.end(), [&](int a, int c) {
    int ra = M.rank[M.t(a, k)], rc = M.rank[M.t(c, k)];
    if (ra != rc) return ra > rc;
    return a < c;
  });
  // structurally zero expressions never enter (ara.cpp:328-345)
  std::vector<int> queue;
  for (int i : order) {
    bool zero = M.rank[M.t(i, k)] == 0;
    for (int j = 0; j < k && zero; ++j)
      if (M.rank[M.t(i, j)] > 0 && M.rank[M.t(k, j)] > 0) zero = false;
    if (!zero) queue.push_back(i);
  }
  return queue;
}

void column_prepare(Ctx& C, const Matrix& M, int k, const AraCfg& cfg, StreamPrep& P) {
  P.T = 0;
  P.k = k;
  P.queue = column_queue(M, k);
  const std::vector<int>& queue = P.queue;
  if (queue.empty()) return;
  std::vector<uint64_t> seeds;
  std::vector<int> rws;
  int maxrows = 0;
  for (int i : queue) {
    seeds.push_back(ara_column_seed(cfg.seed, i, k));
    rws.push_back(M.rows(i));
    maxrows = std::max(maxrows, M.rows(i));
  }
  const char* pf = std::getenv("TLRG_PREFILL");  // 0: fused kernel generates from scratch
  const bool fused = ara_fused_eligible(M.rows(k), rws, cfg.bs, cfg.window > 0 ? cfg.window : cfg.bs);
  if (fused && pf && pf[0] == '0') return;
  // fused path: the first round of every slot's stream, generated while the
  // column setup and H products run, in a ring the producer warp continues;
  // graph path: 8 rounds ahead in a 12-round ring
  if (fused) streams_prepare(C, seeds, M.rows(k), cfg.bs, maxrows, 1, P, 6);
  else streams_prepare(C, seeds, M.rows(k), cfg.bs, maxrows, 8, P);
}

std::vector<TileResult> column_ara(Ctx& C, const Matrix& M, int k, const ColumnSetup& cs,
                                   const AraCfg& cfg, Store& store, ColumnStats& cst,
                                   StreamPrep* pre, int part_rank, int part_world,
                                   const std::function<void()>& on_launch) {
  const int nb = M.nb, b = M.b, rk = M.rows(k), bs = cfg.bs, K = cs.K;
  std::vector<TileResult> res;
  for (int i = k + 1; i < nb; ++i) {
    TileResult r;
    r.i = i;
    res.push_back(r);
  }
  if (res.empty()) return res;
  const char* cpe = std::getenv("TLRG_COLPROF");
  const bool prof = cpe && cpe[0] == '2';
  auto tq0 = std::chrono::steady_clock::now();
  auto since = [&] {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tq0)
        .count();
  };
  std::vector<int> queue = pre && pre->k == k ? pre->queue : column_queue(M, k);
  const double m_queue = since();
  if (part_world > 1) {
    // intra-column split: slot s of the rank-sorted queue
    // belongs to rank s % world, which balances the fat near-diagonal tiles
    std::vector<int> mine;
    for (size_t s = 0; s < queue.size(); ++s)
      if ((int)(s % part_world) == part_rank) mine.push_back(queue[s]);
    queue.swap(mine);
  }
  const int T = (int)queue.size();
  if (T == 0) return res;

  AraSlots S;
  S.cols = rk;
  std::vector<int> kA(T);
  int kAmax = 0;
  for (int s = 0; s < T; ++s) {
    int i = queue[s];
    S.rows.push_back(M.rows(i));
    S.cap.push_back(std::min(M.rows(i), rk));  // ara.cpp:342-343
    S.seeds.push_back(ara_column_seed(cfg.seed, i, k));
    kA[s] = M.rank[M.t(i, k)];
    kAmax = std::max(kAmax, kA[s]);
  }
  // reference-formulation flops per sampled vector; statistics
  // only, read by ara_batch after the kernel: filled while the ARA runs
  auto fill_sref = [&]() {
    S.Sref.resize(T);
    for (int s = 0; s < T; ++s) {
      const int i = queue[s];
      double v = 4.0 * rk * kA[s];
      for (int j = 0; j < k; ++j) {
        int a = M.rank[M.t(k, j)], c = M.rank[M.t(i, j)];
        if (a > 0 && c > 0) v += 4.0 * b * (a + c);
      }
      S.Sref[s] = v;
    }
  };
  const long long Hstride = (long long)b * K;
  double* H = K ? C.buf<double>("H", (size_t)T * Hstride) : nullptr;
  if (cs.d_rank) column_H_dev(C, M, cs, queue, H, Hstride);
  else column_H(C, M, cs, queue, H, Hstride);
  const double m_h = since();
  double* Z = C.buf<double>("Z", (size_t)T * std::max(kAmax, 1) * bs);
  double* T1 = K ? C.buf<double>("T1", (size_t)K * bs * T) : nullptr;

  AraOperator op;
  // H_s (U_k,:^T Omega_s) has a long reduction (K = sum_j rank(k, j), up to
  // ~4000 at cfg3) over few output tiles (rows x bs = 4 CTA tiles at m = 512):
  // split it into S chunks of ~512 written to a workspace (beside the U^A
  // product, which they do not depend on), then Y -= [W_0 .. W_S-1] [I; ..; I]
  // as one more GEMM (products with exact 1/0, chunks summed in order:
  // deterministic)
  static const int ks_min = [] {  // TLRG_KSPLIT_MIN / _CHUNK: tuning switches
    const char* e = std::getenv("TLRG_KSPLIT_MIN");
    return e ? std::atoi(e) : 1024;
  }();
  static const int ks_chunk = [] {
    const char* e = std::getenv("TLRG_KSPLIT_CHUNK");
    return e ? std::max(64, std::atoi(e)) : 512;
  }();
  const int ksplit = K >= ks_min ? std::max(1, std::min(8, K / ks_chunk)) : 1;
  const int kchunk = ksplit > 1 ? ((K + ksplit - 1) / ksplit + 15) / 16 * 16 : K;
  double* Wsplit = nullptr;
  double* Istack = nullptr;
  if (ksplit > 1) {
    int rmax = 0;
    for (int s = 0; s < T; ++s) rmax = std::max(rmax, S.rows[s]);
    Wsplit = C.buf<double>("Ysplit", (size_t)T * ksplit * rmax * bs);
    std::vector<double> hI((size_t)ksplit * bs * bs, 0.0);
    for (int c = 0; c < ksplit; ++c)
      for (int j = 0; j < bs; ++j) hI[(size_t)c * bs + j + (size_t)j * ksplit * bs] = 1.0;
    Istack = C.push(hI);  // lives in the column's descriptor arena, like the GEMM plans
  }
  // Y_s = U^A (V^A^T Omega_s) - H_s (U_k,:^T Omega_s)   (Eq. 1 with the j-sum in H)
  op.sample_plan = [&](const double* Om, double* Y, long long Ystride, const int* done,
                       std::vector<std::vector<GemmProblem>>& stages) {
    stages.assign(3, {});
    for (int s = 0; s < T; ++s) {
      const double* Oms = Om + (size_t)s * rk * bs;
      if (K > 0) {
        GemmProblem g{};
        g.A = cs.Ucat; g.lda = rk; g.transA = 1;
        g.B = Oms; g.ldb = rk;
        g.C = T1 + (size_t)s * bs * K; g.ldc = K;
        g.M = K; g.N = bs; g.K = rk; g.alpha = 1.0; g.skip = done + s;
        stages[0].push_back(g);
      }
      if (kA[s] > 0) {
        GemmProblem g{};
        g.A = M.V[M.t(queue[s], k)]; g.lda = rk; g.transA = 1;
        g.B = Oms; g.ldb = rk;
        g.C = Z + (size_t)s * kAmax * bs; g.ldc = kA[s];
        g.M = kA[s]; g.N = bs; g.K = rk; g.alpha = 1.0; g.skip = done + s;
        stages[0].push_back(g);
      }
      GemmProblem y{};
      y.A = kA[s] ? M.U[M.t(queue[s], k)] : Y; y.lda = S.rows[s];
      y.B = kA[s] ? Z + (size_t)s * kAmax * bs : Y; y.ldb = std::max(kA[s], 1);
      y.C = Y + s * Ystride; y.ldc = S.rows[s];
      y.M = S.rows[s]; y.N = bs; y.K = kA[s]; y.alpha = 1.0; y.beta = 0.0; y.skip = done + s;
      stages[1].push_back(y);
      if (K > 0 && ksplit > 1) {
        const int rs = S.rows[s];
        double* Ws = Wsplit + (size_t)s * ksplit * rs * bs;
        for (int c = 0; c < ksplit; ++c) {
          const int k0 = c * kchunk, kc = std::min(K, k0 + kchunk) - k0;
          GemmProblem h{};
          h.A = H + s * Hstride + (long long)k0 * rs; h.lda = rs;
          h.B = T1 + (size_t)s * bs * K + k0; h.ldb = K;
          h.C = Ws + (size_t)c * rs * bs; h.ldc = rs;
          h.M = rs; h.N = bs; h.K = std::max(kc, 0); h.alpha = 1.0; h.beta = 0.0;
          h.skip = done + s;
          stages[1].push_back(h);
        }
        GemmProblem r{};
        r.A = Ws; r.lda = rs;
        r.B = Istack; r.ldb = (long long)ksplit * bs;
        r.C = Y + s * Ystride; r.ldc = rs;
        r.M = rs; r.N = bs; r.K = ksplit * bs; r.alpha = -1.0; r.beta = 1.0; r.skip = done + s;
        stages[2].push_back(r);
      } else if (K > 0) {
        GemmProblem h{};
        h.A = H + s * Hstride; h.lda = S.rows[s];
        h.B = T1 + (size_t)s * bs * K; h.ldb = K;
        h.C = Y + s * Ystride; h.ldc = S.rows[s];
        h.M = S.rows[s]; h.N = bs; h.K = K; h.alpha = -1.0; h.beta = 1.0; h.skip = done + s;
        stages[2].push_back(h);
      }
    }
  };
  // B_s = V^A (U^A^T Q) - U_k,: (H_s^T Q)
  op.project = [&](const std::vector<int>& q, const double* Q, long long Qstride, double* Bb,
                   const std::vector<long long>& boff) {
    std::vector<long long> poff(T);
    long long ptot = 0;
    for (int s = 0; s < T; ++s) {
      poff[s] = ptot;
      ptot += (long long)(kA[s] + K) * q[s];
    }
    double* P = C.buf<double>("P", (size_t)std::max(ptot, 1LL));
    std::vector<GemmProblem> pr;
    for (int s = 0; s < T; ++s) {
      if (q[s] == 0) continue;
      int i = queue[s], ld = kA[s] + K;
      if (kA[s]) {
        GemmProblem g{};
        g.A = M.U[M.t(i, k)]; g.lda = S.rows[s]; g.transA = 1;
        g.B = Q + s * Qstride; g.ldb = S.rows[s];
        g.C = P + poff[s]; g.ldc = ld;
        g.M = kA[s]; g.N = q[s]; g.K = S.rows[s]; g.alpha = 1.0;
        pr.push_back(g);
      }
      if (K) {
        GemmProblem g{};
        g.A = H + s * Hstride; g.lda = S.rows[s]; g.transA = 1;
        g.B = Q + s * Qstride; g.ldb = S.rows[s];
        g.C = P + poff[s] + kA[s]; g.ldc = ld;
        g.M = K; g.N = q[s]; g.K = S.rows[s]; g.alpha = 1.0;
        pr.push_back(g);
      }
    }
    C.gemm(pr);
    pr.clear();
    for (int s = 0; s < T; ++s) {
      if (q[s] == 0) continue;
      int i = queue[s], ld = kA[s] + K;
      GemmProblem g{};
      g.A = kA[s] ? M.V[M.t(i, k)] : Bb; g.lda = rk;
      g.B = P + poff[s]; g.ldb = ld;
      g.C = Bb + boff[s]; g.ldc = rk;
      g.M = rk; g.N = q[s]; g.K = kA[s]; g.alpha = 1.0; g.beta = 0.0;
      pr.push_back(g);
    }
    C.gemm(pr);
    if (K) {
      pr.clear();
      for (int s = 0; s < T; ++s) {
        if (q[s] == 0) continue;
        GemmProblem g{};
        g.A = cs.Ucat; g.lda = rk;
        g.B = P + poff[s] + kA[s]; g.ldb = kA[s] + K;
        g.C = Bb + boff[s]; g.ldc = rk;
        g.M = rk; g.N = q[s]; g.K = K; g.alpha = -1.0; g.beta = 1.0;
        pr.push_back(g);
      }
      C.gemm(pr);
    }
  };
  // the same operator in the fused kernel's form
  op.fused.on = true;
  op.fused.Ucat = cs.Ucat;
  op.fused.K = K;
  for (int s = 0; s < T; ++s) {
    const long long t = M.t(queue[s], k);
    op.fused.UA.push_back(kA[s] ? M.U[t] : nullptr);
    op.fused.VA.push_back(kA[s] ? M.V[t] : nullptr);
    op.fused.kA.push_back(kA[s]);
    op.fused.H.push_back(K ? H + s * Hstride : nullptr);
  }
  // results land in one panel ordered by ascending i (keeps V panels contiguous)
  std::vector<int> slot_of(nb, -1);
  for (int s = 0; s < T; ++s) slot_of[queue[s]] = s;
  std::vector<int> out_order;
  for (int i = k + 1; i < nb; ++i)
    if (slot_of[i] >= 0) out_order.push_back(slot_of[i]);
  AraOut out;
  const double m_op = since();
  auto hook = [&] {
    if (prof)
      std::fprintf(stderr, "colara %d T=%d J=%zu | queue %.3f H %.3f op %.3f launch %.3f ms\n",
                   k, T, cs.J.size(), m_queue, m_h, m_op, since());
    if (on_launch) on_launch();
    fill_sref();
  };
  ara_batch(C, S, op, cfg, store, out_order, cst, out, pre, hook);
  for (int i = k + 1; i < nb; ++i) {
    TileResult& r = res[i - k - 1];
    int s = slot_of[i];
    if (s < 0) continue;
    r.rank = out.rank[s];
    r.rounds = out.rounds[s];
    r.converged = out.conv[s] != 0;
    r.U = out.U[s];
    r.V = out.V[s];
  }
  return res;
}

// ----------------------------------------------------------------- Store ---
namespace {
std::mutex& ctx_mu() {
  static std::mutex m;
  return m;
}
std::set<const void*>& ctx_set() {
  static std::set<const void*> s;
  return s;
}
}  // namespace
bool ctx_alive(const void* ctx) {
  std::lock_guard<std::mutex> lk(ctx_mu());
  return ctx && ctx_set().count(ctx);
}
void ctx_register(const void* ctx, bool alive) {
  std::lock_guard<std::mutex> lk(ctx_mu());
  if (alive) ctx_set().insert(ctx);
  else ctx_set().erase(ctx);
}
void stream_free(const void* ctx, cudaStream_t st, void* p) {
  if (!p) return;
  if (st && ctx_alive(ctx)) cudaFreeAsync(p, st);
  else cudaFree(p);
}
namespace {
constexpr size_t kChunk = (size_t)1 << 23;  // 64 MiB of doubles
std::mutex& chunk_mu() {
  static std::mutex m;
  return m;
}
std::unordered_map<const void*, std::vector<void*>>& chunk_cache() {
  static std::unordered_map<const void*, std::vector<void*>> c;
  return c;
}
}  // namespace
void chunk_cache_release(const void* ctx) {
  std::vector<void*> v;
  {
    std::lock_guard<std::mutex> lk(chunk_mu());
    auto it = chunk_cache().find(ctx);
    if (it == chunk_cache().end()) return;
    v.swap(it->second);
    chunk_cache().erase(it);
  }
  for (void* p : v) cudaFree(p);
}
void chunk_cache_reserve(const void* ctx, size_t doubles, cudaStream_t st) {
  const size_t need = (doubles + kChunk - 1) / kChunk;
  size_t have;
  {
    std::lock_guard<std::mutex> lk(chunk_mu());
    have = chunk_cache()[ctx].size();
  }
  for (; have < need; ++have) {
    void* p = nullptr;
    TLRG_CUDA(cudaMallocAsync(&p, kChunk * sizeof(double), st));
    std::lock_guard<std::mutex> lk(chunk_mu());
    chunk_cache()[ctx].push_back(p);
  }
}
double* Store::alloc(size_t n) {
  n = (n + 31) & ~(size_t)31;  // 256-byte granules
  if (!cur || used + n > cap) {
    const size_t c = std::max(n, kChunk);  // >= 64 MiB chunks
    void* p = nullptr;
    if (c == kChunk && ctx_alive(owner)) {
      std::lock_guard<std::mutex> lk(chunk_mu());
      auto& v = chunk_cache()[owner];
      if (!v.empty()) {
        p = v.back();
        v.pop_back();
      }
    }
    if (!p) TLRG_CUDA(cudaMallocAsync(&p, c * sizeof(double), st));
    chunks.push_back(p);
    chunk_len.push_back(c);
    cur = static_cast<double*>(p);
    cap = c;
    used = 0;
  }
  double* r = cur + used;
  used += n;
  total += n;
  return r;
}
Store::~Store() {
  const bool alive = st && ctx_alive(owner);
  // chunks go back to the owner's cache once the work touching them is done
  if (alive && !chunks.empty()) cudaStreamSynchronize(st);
  for (size_t i = 0; i < chunks.size(); ++i) {
    if (alive && chunk_len[i] == kChunk) {
      std::lock_guard<std::mutex> lk(chunk_mu());
      chunk_cache()[owner].push_back(chunks[i]);
    } else {
      stream_free(owner, st, chunks[i]);
    }
  }
}

}  // namespace tlrg
