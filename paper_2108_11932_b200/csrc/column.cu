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
#include <cstring>
#include <numeric>

#include "core.h"

namespace tlrg {

namespace {
struct Timer {
  cudaEvent_t a, b;
  cudaStream_t st;
  explicit Timer(cudaStream_t s) : st(s) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
  }
  void start() { cudaEventRecord(a, st); }
  void stop() { cudaEventRecord(b, st); }
  double ms() {
    float f = 0;
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&f, a, b);
    return f;
  }
  ~Timer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};
}  // namespace

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
    for (size_t jj = 0; jj < cs.J.size(); ++jj) {
      int j = cs.J[jj], r = M.rank[M.t(k, j)];
      bd_apply(D.d + (size_t)j * b, D.e + (size_t)j * b, D.s2 + (size_t)j * b, b,
               cs.Wcat + (size_t)cs.seg[jj] * b, b, r, C.st);
      ++C.launches;
    }
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

std::vector<TileResult> column_ara(Ctx& C, const Matrix& M, int k, const ColumnSetup& cs,
                                   const AraCfg& cfg, Store& store, ColumnStats& cst) {
  const int nb = M.nb, b = M.b, rk = M.rows(k), bs = cfg.bs, K = cs.K;
  const int window = cfg.window > 0 ? cfg.window : bs;
  std::vector<TileResult> res;
  for (int i = k + 1; i < nb; ++i) {
    TileResult r;
    r.i = i;
    res.push_back(r);
  }
  if (res.empty()) return res;
  // rank-sorted order (ara.cpp:308-317)
  std::vector<int> order;
  for (int i = k + 1; i < nb; ++i) order.push_back(i);
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
  const int T = (int)queue.size();
  if (T == 0) return res;

  // ---- per-slot state -----------------------------------------------------
  std::vector<int> rows(T), cap(T), kA(T), q(T, 0);
  int kAmax = 0, maxrows = 0;
  for (int s = 0; s < T; ++s) {
    int i = queue[s];
    rows[s] = M.rows(i);
    cap[s] = std::min(rows[s], rk);
    kA[s] = M.rank[M.t(i, k)];
    kAmax = std::max(kAmax, kA[s]);
    maxrows = std::max(maxrows, rows[s]);
  }
  const long long Ystride = (long long)b * bs, Qstride = (long long)b * rk;
  const long long Hstride = (long long)b * K;
  double* H = K ? C.buf<double>("H", (size_t)T * Hstride) : nullptr;
  column_H(C, M, cs, queue, H, Hstride);
  double* Om = C.buf<double>("Om", (size_t)rk * bs * T);
  double* Y = C.buf<double>("Y", (size_t)T * Ystride);
  double* Q = C.buf<double>("Q", (size_t)T * Qstride);
  double* Z = C.buf<double>("Z", (size_t)T * std::max(kAmax, 1) * bs);
  double* T1 = K ? C.buf<double>("T1", (size_t)K * bs * T) : nullptr;
  double* Cdef = C.buf<double>("Cdef", (size_t)T * rk * bs);
  double* R = C.buf<double>("R", (size_t)T * bs * bs);
  double* Rp = C.buf<double>("Rp", (size_t)T * 2 * bs * bs);
  double* tiny = C.buf<double>("tiny", (size_t)T * bs);
  uint8_t* defi = C.buf<uint8_t>("defi", (size_t)T * bs);
  double* cn = C.buf<double>("cn", (size_t)T * bs);
  double* nm = C.buf<double>("nm", (size_t)T * bs);
  double* recent = C.buf<double>("recent", (size_t)T * window);
  int* ints = C.buf<int>("ints", (size_t)T * 6);
  int *qcols = ints, *rounds = ints + T, *conv = ints + 2 * T, *done = ints + 3 * T,
      *rcount = ints + 4 * T, *rpos = ints + 5 * T;
  RngState* rng = C.buf<RngState>("rng", (size_t)T);
  TLRG_CUDA(cudaMemsetAsync(ints, 0, sizeof(int) * T * 6, C.st));
  {
    std::vector<uint64_t> seeds(T);
    for (int s = 0; s < T; ++s) seeds[s] = ara_column_seed(cfg.seed, queue[s], k);
    rng_seed(rng, C.push(seeds), T, C.st);
    ++C.launches;
  }
  // reference-formulation flops per sampled vector
  std::vector<double> Sik(T, 0.0);
  for (int s = 0; s < T; ++s) {
    int i = queue[s];
    double v = 4.0 * rk * kA[s];
    for (int j = 0; j < k; ++j) {
      int a = M.rank[M.t(k, j)], c = M.rank[M.t(i, j)];
      if (a > 0 && c > 0) v += 4.0 * b * (a + c);
    }
    Sik[s] = v;
  }

  Timer tm(C.st);
  std::vector<int> act(T);
  std::iota(act.begin(), act.end(), 0);
  int* h_flags = C.pinned_ints((size_t)2 * T);
  while (!act.empty()) {
    const int Ta = (int)act.size();
    tm.start();
    int* d_act = C.push(act);
    rng_draw(rng, d_act, Ta, Om, (long long)rk * bs, (long long)rk * bs, C.st);
    ++C.launches;
    std::vector<GemmProblem> pr;
    if (K > 0) {
      GemmProblem g{};
      g.A = cs.Ucat; g.lda = rk; g.transA = 1;
      g.B = Om; g.ldb = rk;
      g.C = T1; g.ldc = K;
      g.M = K; g.N = Ta * bs; g.K = rk; g.alpha = 1.0;
      pr.push_back(g);
    }
    for (int a = 0; a < Ta; ++a) {
      int s = act[a];
      if (kA[s] == 0) continue;
      int i = queue[s];
      GemmProblem g{};
      g.A = M.V[M.t(i, k)]; g.lda = rk; g.transA = 1;
      g.B = Om + (size_t)a * rk * bs; g.ldb = rk;
      g.C = Z + (size_t)s * kAmax * bs; g.ldc = kA[s];
      g.M = kA[s]; g.N = bs; g.K = rk; g.alpha = 1.0;
      pr.push_back(g);
    }
    C.gemm(pr);
    pr.clear();
    for (int a = 0; a < Ta; ++a) {
      int s = act[a], i = queue[s];
      GemmProblem g{};
      g.A = kA[s] ? M.U[M.t(i, k)] : Y; g.lda = rows[s];
      g.B = kA[s] ? Z + (size_t)s * kAmax * bs : Y; g.ldb = std::max(kA[s], 1);
      g.C = Y + s * Ystride; g.ldc = rows[s];
      g.M = rows[s]; g.N = bs; g.K = kA[s]; g.alpha = 1.0; g.beta = 0.0;
      pr.push_back(g);
    }
    C.gemm(pr);
    if (K > 0) {
      pr.clear();
      for (int a = 0; a < Ta; ++a) {
        int s = act[a];
        GemmProblem g{};
        g.A = H + s * Hstride; g.lda = rows[s];
        g.B = T1 + (size_t)a * bs * K; g.ldb = K;
        g.C = Y + s * Ystride; g.ldc = rows[s];
        g.M = rows[s]; g.N = bs; g.K = K; g.alpha = -1.0; g.beta = 1.0;
        pr.push_back(g);
      }
      C.gemm(pr);
    }
    tm.stop();
    cst.t_sampling += 0;  // accumulated below after the sync
    Timer to(C.st);
    to.start();
    std::vector<PanelTask> tasks(Ta);
    for (int a = 0; a < Ta; ++a) {
      int s = act[a];
      PanelTask& P = tasks[a];
      P.Y = Y + s * Ystride;
      P.Q = Q + s * Qstride;
      P.R = R + (size_t)s * bs * bs;
      P.Rp = Rp + (size_t)s * 2 * bs * bs;
      P.tiny = tiny + (size_t)s * bs;
      P.deficient = defi + (size_t)s * bs;
      P.col_norms = cn + (size_t)s * bs;
      P.new_mass = nm + (size_t)s * bs;
      P.rng = rng + s;
      P.tau = 0;
      P.rows = rows[s];
      P.width = bs;
      P.q = q[s];
    }
    PanelTask* d_tasks = C.push(tasks);
    panel_tau(d_tasks, Ta, C.st);
    ++C.launches;
    for (int sweep = 0; sweep < 2; ++sweep) {
      std::vector<GemmProblem> p1, p2;
      for (int a = 0; a < Ta; ++a) {
        int s = act[a];
        if (q[s] == 0) continue;
        GemmProblem g{};
        g.A = Q + s * Qstride; g.lda = rows[s]; g.transA = 1;
        g.B = Y + s * Ystride; g.ldb = rows[s];
        g.C = Cdef + (size_t)s * rk * bs; g.ldc = q[s];
        g.M = q[s]; g.N = bs; g.K = rows[s]; g.alpha = 1.0;
        p1.push_back(g);
        GemmProblem h{};
        h.A = Q + s * Qstride; h.lda = rows[s];
        h.B = Cdef + (size_t)s * rk * bs; h.ldb = q[s];
        h.C = Y + s * Ystride; h.ldc = rows[s];
        h.M = rows[s]; h.N = bs; h.K = q[s]; h.alpha = -1.0; h.beta = 1.0;
        p2.push_back(h);
      }
      if (!p1.empty()) {
        C.gemm(p1);
        C.gemm(p2);
      }
      panel_mgs(d_tasks, Ta, sweep, sweep == 1, bs, maxrows, C.st);
      ++C.launches;
    }
    std::vector<AbsorbTask> ab(Ta);
    for (int a = 0; a < Ta; ++a) {
      int s = act[a];
      AbsorbTask& A = ab[a];
      A.Y = Y + s * Ystride;
      A.Q = Q + s * Qstride;
      A.col_norms = cn + (size_t)s * bs;
      A.new_mass = nm + (size_t)s * bs;
      A.recent = recent + (size_t)s * window;
      A.qcols = qcols + s;
      A.recent_count = rcount + s;
      A.recent_pos = rpos + s;
      A.rounds = rounds + s;
      A.converged = conv + s;
      A.done = done + s;
      A.rows = rows[s];
      A.bs = bs;
      A.cap = cap[s];
      A.window = window;
      A.eps = cfg.eps;
      A.eta = cfg.safety;
    }
    ara_absorb(C.push(ab), Ta, C.st);
    ++C.launches;
    to.stop();
    TLRG_CUDA(cudaMemcpyAsync(h_flags, done, sizeof(int) * T, cudaMemcpyDeviceToHost, C.st));
    TLRG_CUDA(cudaMemcpyAsync(h_flags + T, qcols, sizeof(int) * T, cudaMemcpyDeviceToHost, C.st));
    C.sync();
    cst.t_sampling += tm.ms() * 1e-3;
    cst.t_orthog += to.ms() * 1e-3;
    cst.tile_rounds += Ta;
    for (int a = 0; a < Ta; ++a) cst.flops_ref += bs * Sik[act[a]];
    std::vector<int> stay;
    for (int s : act) {
      q[s] = h_flags[T + s];
      if (!h_flags[s]) stay.push_back(s);
    }
    act.swap(stay);
  }
  std::vector<int> h_rounds(T), h_conv(T);
  TLRG_CUDA(cudaMemcpy(h_rounds.data(), rounds, sizeof(int) * T, cudaMemcpyDeviceToHost));
  TLRG_CUDA(cudaMemcpy(h_conv.data(), conv, sizeof(int) * T, cudaMemcpyDeviceToHost));

  // ---- exit projection B = E^T Q (ara.cpp:380-387), all tiles batched -------
  Timer tp(C.st);
  tp.start();
  std::vector<long long> poff(T), boff(T);
  long long ptot = 0, btot = 0;
  int qmax = 0;
  for (int s = 0; s < T; ++s) {
    poff[s] = ptot;
    boff[s] = btot;
    ptot += (long long)(kA[s] + K) * q[s];
    btot += (long long)rk * q[s];
    qmax = std::max(qmax, q[s]);
    cst.flops_ref += q[s] * Sik[s];
  }
  double* P = C.buf<double>("P", (size_t)std::max(ptot, 1LL));
  double* Bb = C.buf<double>("B", (size_t)std::max(btot, 1LL));
  {
    std::vector<GemmProblem> pr;
    for (int s = 0; s < T; ++s) {
      if (q[s] == 0) continue;
      int i = queue[s], ld = kA[s] + K;
      if (kA[s]) {
        GemmProblem g{};
        g.A = M.U[M.t(i, k)]; g.lda = rows[s]; g.transA = 1;
        g.B = Q + s * Qstride; g.ldb = rows[s];
        g.C = P + poff[s]; g.ldc = ld;
        g.M = kA[s]; g.N = q[s]; g.K = rows[s]; g.alpha = 1.0;
        pr.push_back(g);
      }
      if (K) {
        GemmProblem g{};
        g.A = H + s * Hstride; g.lda = rows[s]; g.transA = 1;
        g.B = Q + s * Qstride; g.ldb = rows[s];
        g.C = P + poff[s] + kA[s]; g.ldc = ld;
        g.M = K; g.N = q[s]; g.K = rows[s]; g.alpha = 1.0;
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
        int ld = kA[s] + K;
        GemmProblem g{};
        g.A = cs.Ucat; g.lda = rk;
        g.B = P + poff[s] + kA[s]; g.ldb = ld;
        g.C = Bb + boff[s]; g.ldc = rk;
        g.M = rk; g.N = q[s]; g.K = K; g.alpha = -1.0; g.beta = 1.0;
        pr.push_back(g);
      }
      C.gemm(pr);
    }
  }
  tp.stop();

  // ---- recompression (ara.cpp:201-211) --------------------------------------
  Timer tr(C.st);
  tr.start();
  std::vector<int> fr(T, 0);  // final ranks
  const double cut = (1.0 - 1.0 / cfg.safety) * cfg.eps;
  const bool recomp = cfg.recompress && cut > 0.0;
  std::vector<long long> roff(T);
  long long rtot = 0;
  for (int s = 0; s < T; ++s) {
    roff[s] = rtot;
    rtot += (long long)q[s] * q[s];
  }
  double *Rr = nullptr, *Vs = nullptr;
  if (recomp && qmax > 0) {
    Rr = C.buf<double>("Rr", (size_t)rtot + 1);
    double* Rpr = C.buf<double>("Rpr", (size_t)2 * rtot + 1);
    Vs = C.buf<double>("Vs", (size_t)rtot + 1);
    double* work = C.buf<double>("svdwork", (size_t)2 * rtot + 1);
    double* sig = C.buf<double>("sig", (size_t)T * qmax + 1);
    double* vec = C.buf<double>("rvec", (size_t)T * qmax * 3 + 1);
    uint8_t* df = C.buf<uint8_t>("rdef", (size_t)T * qmax + 1);
    int* rko = C.buf<int>("rank_out", (size_t)T);
    std::vector<PanelTask> tasks;
    std::vector<SvdTask> svd;
    std::vector<int> sl;
    for (int s = 0; s < T; ++s) {
      if (q[s] == 0) continue;
      PanelTask P{};
      P.Y = Bb + boff[s];
      P.Q = nullptr;
      P.R = Rr + roff[s];
      P.Rp = Rpr + 2 * roff[s];
      P.tiny = vec + (size_t)s * qmax * 3;
      P.col_norms = P.tiny + qmax;
      P.new_mass = P.tiny + 2 * qmax;
      P.deficient = df + (size_t)s * qmax;
      P.rng = rng + s;
      P.rows = rk;
      P.width = q[s];
      P.q = 0;
      tasks.push_back(P);
      SvdTask V{};
      V.A = Rr + roff[s];
      V.V = Vs + roff[s];
      V.sig = sig + (size_t)s * qmax;
      V.work = work + 2 * roff[s];
      V.rank_out = rko + s;
      V.n = q[s];
      V.cut = cut;
      svd.push_back(V);
      sl.push_back(s);
    }
    PanelTask* d_tasks = C.push(tasks);
    panel_tau(d_tasks, (int)tasks.size(), C.st);
    panel_mgs(d_tasks, (int)tasks.size(), 0, 0, qmax, rk, C.st);
    panel_mgs(d_tasks, (int)tasks.size(), 1, 1, qmax, rk, C.st);
    jacobi_svd(C.push(svd), (int)svd.size(), qmax, C.st);
    C.launches += 4;
    std::vector<int> hr(T);
    TLRG_CUDA(cudaMemcpyAsync(hr.data(), rko, sizeof(int) * T, cudaMemcpyDeviceToHost, C.st));
    C.sync();
    for (int s : sl) fr[s] = hr[s];
  } else {
    for (int s = 0; s < T; ++s) fr[s] = q[s];
  }
  // ---- write the column panel (ascending i) ---------------------------------
  std::vector<int> slot_of(nb, -1);
  for (int s = 0; s < T; ++s) slot_of[queue[s]] = s;
  long long utot = 0, vtot = 0;
  for (int i = k + 1; i < nb; ++i) {
    int s = slot_of[i];
    if (s < 0) continue;
    utot += (long long)rows[s] * fr[s];
    vtot += (long long)rk * fr[s];
  }
  double* Up = utot ? store.alloc((size_t)utot) : nullptr;
  double* Vp = vtot ? store.alloc((size_t)vtot) : nullptr;
  std::vector<GemmProblem> pu;
  std::vector<CopyItem> cpy;
  long long uo = 0, vo = 0;
  for (int i = k + 1; i < nb; ++i) {
    TileResult& r = res[i - k - 1];
    int s = slot_of[i];
    if (s < 0) {
      r.rank = 0;
      r.converged = true;
      r.rounds = 0;
      continue;
    }
    r.rank = fr[s];
    r.rounds = h_rounds[s];
    r.converged = h_conv[s] != 0;
    if (fr[s] == 0) continue;
    r.U = Up + uo;
    r.V = Vp + vo;
    uo += (long long)rows[s] * fr[s];
    vo += (long long)rk * fr[s];
    if (recomp) {
      GemmProblem g{};
      g.A = Q + s * Qstride; g.lda = rows[s];
      g.B = Vs + roff[s]; g.ldb = q[s];
      g.C = r.U; g.ldc = rows[s];
      g.M = rows[s]; g.N = fr[s]; g.K = q[s]; g.alpha = 1.0;
      pu.push_back(g);
      GemmProblem h{};
      h.A = Bb + boff[s]; h.lda = rk;
      h.B = Rr + roff[s]; h.ldb = q[s];
      h.C = r.V; h.ldc = rk;
      h.M = rk; h.N = fr[s]; h.K = q[s]; h.alpha = 1.0;
      pu.push_back(h);
    } else {
      cpy.push_back({Q + s * Qstride, r.U, rows[s], rows[s], rows[s], fr[s]});
      cpy.push_back({Bb + boff[s], r.V, rk, rk, rk, fr[s]});
    }
  }
  if (!pu.empty()) C.gemm(pu);
  if (!cpy.empty()) {
    batched_copy(C.push(cpy), (int)cpy.size(), C.st);
    ++C.launches;
  }
  tr.stop();
  C.sync();
  cst.t_projection += tp.ms() * 1e-3;
  cst.t_recompress += tr.ms() * 1e-3;
  return res;
}

// ----------------------------------------------------------------- Store ---
double* Store::alloc(size_t n) {
  n = (n + 31) & ~(size_t)31;  // 256-byte granules
  if (!cur || used + n > cap) {
    size_t c = std::max(n, (size_t)1 << 23);  // >= 64 MiB chunks
    void* p = nullptr;
    TLRG_CUDA(cudaMalloc(&p, c * sizeof(double)));
    chunks.push_back(p);
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
  for (void* p : chunks) cudaFree(p);
}

}  // namespace tlrg
