// Batched adaptive randomized approximation (ARA) on the device.
//
// One call runs the reference's per-tile TileState machine (ara.cpp:155-195)
// for a whole batch of tiles at once, with every tile resident (the GPU
// replacement for the rank-sorted subset scheduler, ara.cpp:302-404: the
// per-tile streams make results independent of the schedule, test_ara.cpp
// "subset capacity changes scheduling only").  Per round:
//   draw   : per-tile tlr::Rng gaussian blocks (exact mt19937_64 streams)
//   sample : Y = E Omega  (operator callback -> grouped DMMA GEMMs)
//   orthog : BGS2 against Q (grouped GEMMs) + per-tile MGS2 panel kernel
//   absorb : keep filter, basis append, window convergence (device flags)
// Converged tiles leave; one D2H of the flags per round drives compaction.
// At the end all tiles are projected (B = E^T Q) and recompressed (orthog of B
// + one-sided Jacobi SVD of R, cut at (1 - 1/eta) eps) in batches, and the
// final factors are written into a contiguous panel.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>

#include "core.h"

namespace tlrg {
extern std::chrono::steady_clock::time_point g_fused_launch, g_ara_waited,
    g_ara_recomp;  // factor.cu (COLPROF probes)


namespace {
// CUDA events recycled per thread and device (creating and destroying six
// events per column cost tens of microseconds of host time in the loop)
std::vector<cudaEvent_t>& event_pool() {
  thread_local std::map<int, std::vector<cudaEvent_t>> pools;
  int dev = 0;
  cudaGetDevice(&dev);
  return pools[dev];
}
cudaEvent_t event_take() {
  auto& p = event_pool();
  if (p.empty()) {
    cudaEvent_t e;
    TLRG_CUDA(cudaEventCreate(&e));
    return e;
  }
  cudaEvent_t e = p.back();
  p.pop_back();
  return e;
}
struct Timer {
  cudaEvent_t a, b;
  explicit Timer() : a(event_take()), b(event_take()) {}
  void start(cudaStream_t s) { cudaEventRecord(a, s); }
  void stop(cudaStream_t s) { cudaEventRecord(b, s); }
  double sec() {
    float f = 0;
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&f, a, b);
    return f * 1e-3;
  }
  // hand the recorded pair to the caller (read later, see column_stats_resolve)
  std::pair<cudaEvent_t, cudaEvent_t> release() {
    auto r = std::make_pair(a, b);
    a = b = nullptr;
    return r;
  }
  ~Timer() {
    auto& p = event_pool();
    if (a) p.push_back(a);
    if (b) p.push_back(b);
  }
};
__global__ void ara_loop_cond_kernel(cudaGraphConditionalHandle h, int* active, int max_rounds) {
  int it = ++active[1];
  cudaGraphSetConditional(h, (active[0] > 0 && it < max_rounds) ? 1 : 0);
}
__global__ void ara_loop_count_kernel(int* active) { ++active[1]; }
void ara_loop_cond_host(int* active, cudaStream_t st) {
  ara_loop_count_kernel<<<1, 1, 0, st>>>(active);
  TLRG_CUDA(cudaGetLastError());
}
void ara_loop_cond(cudaGraphConditionalHandle h, int* active, int max_rounds, cudaStream_t st) {
  ara_loop_cond_kernel<<<1, 1, 0, st>>>(h, active, max_rounds);
  TLRG_CUDA(cudaGetLastError());
}
}  // namespace

void column_stats_resolve(ColumnStats& cst) {
  auto fold = [](std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& v, double& acc) {
    auto& pool = event_pool();
    for (auto& e : v) {
      float f = 0;
      cudaEventSynchronize(e.second);
      cudaEventElapsedTime(&f, e.first, e.second);
      acc += f * 1e-3;
      pool.push_back(e.first);
      pool.push_back(e.second);
    }
    v.clear();
  };
  fold(cst.pending_proj, cst.t_projection);
  fold(cst.pending_recomp, cst.t_recompress);
}

bool ara_fused_eligible(int cols, const std::vector<int>& rows, int bs, int window) {
  const char* nf = std::getenv("TLRG_NO_FUSED");
  if (nf && nf[0] == '1') return false;
  // bs = 32 (configs 3-5): the per-tile products are heavy enough that the
  // batched multi-CTA GEMMs of the graph path win (measured at config 3)
  if (bs > 16) return false;
  if (cols % 2) return false;
  int maxrows = 0;
  for (int r : rows) {
    if (r % 2) return false;
    maxrows = std::max(maxrows, r);
  }
  // the shared-memory panel holds both the tile rows (sampling) and the
  // cols x q exit projection B (recompression): size it for the larger
  return ara_fused_supported(std::max(maxrows, cols), bs, window);
}

void streams_prepare(Ctx& C, const std::vector<uint64_t>& seeds, int cols, int bs, int maxrows,
                     int rounds_ahead, StreamPrep& P, int ring_rounds) {
  const int T = (int)seeds.size();
  P.T = T;
  P.seeds = seeds;
  GaussStreams& G = P.G;
  G.st = C.buf<RngState>("p_rng", (size_t)T);
  G.cap = ((long long)ring_rounds * cols * bs + 4LL * bs * maxrows + 1) & ~1LL;
  G.buf = C.buf<double>("p_gbuf", (size_t)T * G.cap);
  long long* gl = C.buf<long long>("p_gcur", (size_t)2 * T);
  G.avail = gl;
  G.cursor = gl + T;
  P.pre = std::min<long long>(G.cap, (long long)rounds_ahead * cols * bs +
                                         (ring_rounds >= 12 ? 2LL * bs * maxrows : 0));
  P.pre = (P.pre + 1) & ~1LL;
  uint64_t* d_seeds = C.buf<uint64_t>("p_seeds", (size_t)T);
  int* d_slots = C.buf<int>("p_slots", (size_t)T);
  long long* d_want = C.buf<long long>("p_want", (size_t)T);
  std::vector<int> slots(T);
  std::vector<long long> want(T, P.pre);
  for (int s = 0; s < T; ++s) slots[s] = s;
  TLRG_CUDA(cudaMemsetAsync(gl, 0, sizeof(long long) * 2 * T, C.st2));
  TLRG_CUDA(cudaMemcpyAsync(d_seeds, seeds.data(), 8 * T, cudaMemcpyHostToDevice, C.st2));
  TLRG_CUDA(cudaMemcpyAsync(d_slots, slots.data(), 4 * T, cudaMemcpyHostToDevice, C.st2));
  TLRG_CUDA(cudaMemcpyAsync(d_want, want.data(), 8 * T, cudaMemcpyHostToDevice, C.st2));
  rng_seed(G.st, d_seeds, T, C.st2);
  gauss_generate(G, d_slots, d_want, T, C.st2);
  C.launches += 2;
  if (!P.ev) TLRG_CUDA(cudaEventCreateWithFlags(&P.ev, cudaEventDisableTiming));
  TLRG_CUDA(cudaEventRecord(P.ev, C.st2));
}

void ara_batch(Ctx& C, const AraSlots& S, const AraOperator& op, const AraCfg& cfg, Store& store,
               const std::vector<int>& out_order, ColumnStats& cst, AraOut& out,
               StreamPrep* pre, const std::function<void()>& on_launch) {
  const int T = (int)S.rows.size();
  const int bs = cfg.bs, cols = S.cols;
  const int window = cfg.window > 0 ? cfg.window : bs;
  out.rank.assign(T, 0);
  out.rounds.assign(T, 0);
  out.conv.assign(T, 1);
  out.U.assign(T, nullptr);
  out.V.assign(T, nullptr);
  if (T == 0) return;
  int maxrows = 0, capmax = 0;
  for (int s = 0; s < T; ++s) {
    maxrows = std::max(maxrows, S.rows[s]);
    capmax = std::max(capmax, S.cap[s]);
  }
  const long long Ystride = (long long)maxrows * bs, Qstride = (long long)maxrows * capmax;
  double* Om = C.buf<double>("Om", (size_t)cols * bs * T);
  double* Y = C.buf<double>("Y", (size_t)T * Ystride);
  double* Q = C.buf<double>("Q", (size_t)T * Qstride);
  double* Cdef = C.buf<double>("Cdef", (size_t)T * capmax * bs);
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
  TLRG_CUDA(cudaMemsetAsync(ints, 0, sizeof(int) * T * 6, C.st));
  const bool use_fused = op.fused.on && ara_fused_eligible(cols, S.rows, bs, window);
  // per-tile gaussian streams (exact tlr::Rng sequences), consumed by cursor
  GaussStreams G;
  std::vector<long long> h_av(T, 0), h_cur(T, 0);
  // streams generated ahead on the side stream (column_prepare): the graph path
  // consumes them by cursor; the fused kernel's producer warp continues them, so
  // its first round does not wait for the in-kernel generator
  if (pre && pre->T == T && pre->seeds == S.seeds &&
      pre->G.cap >= 2LL * cols * bs + 4LL * bs * maxrows) {
    G = pre->G;
    TLRG_CUDA(cudaStreamWaitEvent(C.st, pre->ev, 0));
    for (int s = 0; s < T; ++s) h_av[s] = pre->pre;
  } else {
    G.st = C.buf<RngState>("rng", (size_t)T);
    G.cap = (6LL * cols * bs + 4LL * bs * maxrows + 1) & ~1LL;
    G.buf = C.buf<double>("gbuf", (size_t)T * G.cap);
    long long* gl = C.buf<long long>("gcur", (size_t)2 * T);
    G.avail = gl;
    G.cursor = gl + T;
    TLRG_CUDA(cudaMemsetAsync(gl, 0, sizeof(long long) * 2 * T, C.st));
    rng_seed(G.st, C.push(S.seeds), T, C.st);
    ++C.launches;
  }
  const long long gchunk = 2LL * cols * bs;
  // make sure every listed slot has `need` values ready beyond its cursor
  auto ensure = [&](const std::vector<int>& slots, const std::vector<long long>& need) {
    std::vector<int> gen;
    std::vector<long long> want;
    for (size_t t = 0; t < slots.size(); ++t) {
      int s = slots[t];
      if (h_av[s] - h_cur[s] >= need[t]) continue;
      long long w = std::min(h_cur[s] + G.cap, h_cur[s] + need[t] + gchunk) & ~1LL;
      gen.push_back(s);
      want.push_back(w);
      h_av[s] = w;
    }
    if (!gen.empty()) {
      gauss_generate(G, C.push(gen), C.push(want), (int)gen.size(), C.st);
      ++C.launches;
    }
  };

  std::vector<int> q(T, 0);
  int* active = C.buf<int>("active", 2);  // [0] tiles still resident, [1] loop counter
  int* d_rows = C.buf<int>("slot_rows", (size_t)T);
  if (!use_fused) {  // round-loop state of the graph path
    std::vector<int> init{T, 0};
    TLRG_CUDA(cudaMemcpyAsync(active, init.data(), sizeof(int) * 2, cudaMemcpyHostToDevice, C.st));
    TLRG_CUDA(cudaMemcpyAsync(d_rows, S.rows.data(), sizeof(int) * T, cudaMemcpyHostToDevice,
                              C.st));
  }
  int capall = 0;
  for (int s = 0; s < T; ++s) capall = std::max(capall, S.cap[s]);
  const int max_rounds = 4 * capall + 8;  // a tile gains >= 1 column per round or converges
  Timer tm;
  bool recomp_in_kernel = false;
  double *Uo = nullptr, *Vo = nullptr;
  int* rank_in = nullptr;
  double* fl_dev = nullptr;
  std::vector<double> h_fl(T, 0.0);
  std::vector<int> h_rank_in(T, -1);
  std::vector<std::pair<cudaGraphExec_t, cudaGraph_t>> graph_cleanup;
  if (use_fused) {
    // ---- every round of every tile in ONE launch (one CTA per tile) ----------
    tm.start(C.st);
    const AraFusedOp& fo = op.fused;
    long long wtot = 0;
    std::vector<long long> woff(T);
    for (int s = 0; s < T; ++s) {
      woff[s] = wtot;
      wtot += (long long)((fo.Ad.empty() || !fo.Ad[s] ? fo.kA[s] + fo.K : 0) + 2) *
              std::max(bs, FUSED_QMAX);
    }
    recomp_in_kernel = cfg.recompress && (1.0 - 1.0 / cfg.safety) * cfg.eps > 0.0;
    Uo = C.buf<double>("fusedUo", (size_t)T * maxrows * FUSED_QMAX);
    Vo = C.buf<double>("fusedVo", (size_t)T * cols * FUSED_QMAX);
    rank_in = C.buf<int>("fusedRank", (size_t)T);
    double* Wb = C.buf<double>("fusedW", (size_t)wtot);
    double* rc = C.buf<double>("fusedRC", (size_t)T * capmax);
    const size_t cqs = (size_t)(2 * capmax + bs + 4) * bs;
    double* Cqf = C.buf<double>("fusedCq", (size_t)T * cqs);
    std::vector<FusedSlot> slots(T);
    for (int s = 0; s < T; ++s) {
      FusedSlot& f = slots[s];
      f = FusedSlot{};
      f.UA = fo.UA.empty() ? nullptr : fo.UA[s];
      f.VA = fo.VA.empty() ? nullptr : fo.VA[s];
      f.H = fo.H.empty() ? nullptr : fo.H[s];
      f.kA = fo.kA.empty() ? 0 : fo.kA[s];
      f.Ad = fo.Ad.empty() ? nullptr : fo.Ad[s];
      f.ldad = fo.ldad.empty() ? 0 : fo.ldad[s];
      f.rows = S.rows[s];
      f.cap = S.cap[s];
      f.Q = Q + s * Qstride;
      f.Om = Om + (size_t)s * cols * bs;
      f.W = Wb + woff[s];
      f.Cq = Cqf + (size_t)s * cqs;
      f.repC = rc + (size_t)s * capmax;
      f.Uo = Uo + (size_t)s * maxrows * FUSED_QMAX;
      f.Vo = Vo + (size_t)s * cols * FUSED_QMAX;
    }
    FusedArgs fa{};
    fa.slots = C.push(slots);
    fa.G = G;
    fa.Ucat = fo.Ucat;
    fa.K = fo.K;
    fa.cols = cols;
    fa.bs = bs;
    fa.window = window;
    fa.max_rounds = max_rounds;
    fa.eps = cfg.eps;
    fa.eta = cfg.safety;
    fa.qcols = qcols;
    fa.rounds = rounds;
    fa.conv = conv;
    fa.recompress = recomp_in_kernel ? 1 : 0;
    fa.cut = (1.0 - 1.0 / cfg.safety) * cfg.eps;
    fa.rank_out = rank_in;
    fl_dev = C.buf<double>("fusedFlops", (size_t)T);
    fa.flops_out = fl_dev;
    fa.mgs_passes = 2;  // MGS2 as the reference (one pass measurably changes ranks/rounds)
    {
      const char* e = std::getenv("TLRG_SWEEP2");  // 0: column-wise second sweep (A/B)
      fa.fast_sweep2 = !(e && e[0] == '0');
      const char* d = std::getenv("TLRG_DCGS");  // 0: column-wise CGS2 panel (A/B)
      fa.dcgs = !(d && d[0] == '0');
    }
    const char* fp = std::getenv("TLRG_FUSED_PROF");
    long long* dprof = nullptr;
    if (fp && fp[0] == '1') {
      dprof = C.buf<long long>("fused_prof", (size_t)T * 8);
      fa.prof = dprof;
    }
    g_fused_launch = std::chrono::steady_clock::now();
    // CTAs per tile: the slowest tile's round chain is the column's critical
    // path, so columns with few tiles give each tile a cluster that shares its
    // sampling products (TLRG_CLUSTER=n forces n; the T limits are tunable)
    int cl = 1;
    {
      bool dense = false;
      for (int s = 0; s < T && !dense; ++s) dense = !fo.Ad.empty() && fo.Ad[s];
      auto envi = [](const char* n, int d) {
        const char* e = std::getenv(n);
        return e ? std::atoi(e) : d;
      };
      if (bs == 16 && !dense) {
        const int t4 = envi("TLRG_CL4_MAXT", 37), t2 = envi("TLRG_CL2_MAXT", 74);
        cl = T <= t4 ? 4 : T <= t2 ? 2 : 1;
        const int force = envi("TLRG_CLUSTER", 0);
        if (force > 0) cl = force >= 4 ? 4 : force >= 2 ? 2 : 1;
      }
    }
    ara_fused(fa, T, maxrows, C.st, cl);
    ++C.launches;
    if (dprof) {
      std::vector<long long> hp((size_t)T * 8);
      TLRG_CUDA(cudaMemcpyAsync(hp.data(), dprof, sizeof(long long) * T * 8,
                                cudaMemcpyDeviceToHost, C.st));
      C.wait();
      int w = 0;
      for (int s2 = 1; s2 < T; ++s2)
        if (hp[8 * s2 + 6] > hp[8 * w + 6]) w = s2;
      long long tot = 0, rds = 0;
      for (int s2 = 0; s2 < T; ++s2) {
        tot += hp[8 * s2 + 6];
        rds += hp[8 * s2 + 7];
      }
      std::fprintf(stderr,
                   "fused T=%d K=%d slowest slot %d rounds %lld: draw %lld sample %lld tau %lld "
                   "deflate %lld mgs %lld absorb %lld total %lld kcyc | mean rounds %.2f mean "
                   "total %lld kcyc\n",
                   T, fo.K, w, hp[8 * w + 7], hp[8 * w] / 1000, hp[8 * w + 1] / 1000,
                   hp[8 * w + 2] / 1000, hp[8 * w + 3] / 1000, hp[8 * w + 4] / 1000,
                   hp[8 * w + 5] / 1000, hp[8 * w + 6] / 1000, (double)rds / T, tot / T / 1000);
    }
  } else {
  // ---- static per-column launch tables (staged before capture) ---------------
  std::vector<std::vector<GemmProblem>> stages;
  op.sample_plan(Om, Y, Ystride, done, stages);
  std::vector<GemmPlan> sample_plans;
  for (auto& st : stages) sample_plans.push_back(gemm_plan(st, C.desc, C.st));
  std::vector<GemmProblem> pc, py;
  for (int s = 0; s < T; ++s) {
    GemmProblem g{};
    g.A = Q + s * Qstride; g.lda = S.rows[s]; g.transA = 1;
    g.B = Y + s * Ystride; g.ldb = S.rows[s];
    g.C = Cdef + (size_t)s * capmax * bs; g.ldc = S.cap[s];
    g.M = S.cap[s]; g.N = bs; g.K = S.rows[s]; g.alpha = 1.0;
    g.Mp = qcols + s; g.skip = done + s;
    pc.push_back(g);
    GemmProblem h{};
    h.A = Q + s * Qstride; h.lda = S.rows[s];
    h.B = Cdef + (size_t)s * capmax * bs; h.ldb = S.cap[s];
    h.C = Y + s * Ystride; h.ldc = S.rows[s];
    h.M = S.rows[s]; h.N = bs; h.K = S.cap[s]; h.alpha = -1.0; h.beta = 1.0;
    h.Kp = qcols + s; h.skip = done + s;
    py.push_back(h);
  }
  GemmPlan plan_c = gemm_plan(pc, C.desc, C.st), plan_y = gemm_plan(py, C.desc, C.st);
  double* rep = C.buf<double>("rep", (size_t)T * maxrows * bs);
  double* repC = C.buf<double>("repC", (size_t)T * capmax * bs);
  std::vector<PanelTask> tasks(T);
  for (int s = 0; s < T; ++s) {
    PanelTask& P = tasks[s];
    P = PanelTask{};
    P.Y = Y + s * Ystride;
    P.Q = Q + s * Qstride;
    P.R = R + (size_t)s * bs * bs;
    P.Rp = Rp + (size_t)s * 2 * bs * bs;
    P.tiny = tiny + (size_t)s * bs;
    P.deficient = defi + (size_t)s * bs;
    P.col_norms = cn + (size_t)s * bs;
    P.new_mass = nm + (size_t)s * bs;
    P.gbuf = G.buf + (long long)s * G.cap;
    P.gcursor = G.cursor + s;
    P.gcap = G.cap;
    P.rep = rep + (size_t)s * maxrows * bs;
    P.repC = repC + (size_t)s * capmax * bs;
    P.rows = S.rows[s];
    P.width = bs;
    P.done = done + s;
    P.qdev = qcols + s;
    P.Qw = Q + s * Qstride;
    P.recent = recent + (size_t)s * window;
    P.qcols = qcols + s;
    P.rcount = rcount + s;
    P.rpos = rpos + s;
    P.rounds = rounds + s;
    P.conv = conv + s;
    P.donew = done + s;
    P.active = active;
    P.cap = S.cap[s];
    P.window = window;
    P.eps = cfg.eps;
    P.eta = cfg.safety;
  }
  PanelTask* d_tasks = C.push(tasks);
  // ---- the round loop: one CUDA graph, conditional WHILE node on device ------
  tm.start(C.st);
  // the gaussian rings are refilled on a side branch of the round (fork after
  // this round's Omega is copied out, join before the loop condition): the
  // sequential mt19937_64 + polar generation overlaps the products and sweeps
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  TLRG_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
  TLRG_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
  const long long topup_low = G.cap - 2LL * cols * bs;
  auto enqueue_round = [&]() {
    gauss_round(G, done, d_rows, T, cols, bs, Om, C.st);
    TLRG_CUDA(cudaEventRecord(ev_fork, C.st));
    TLRG_CUDA(cudaStreamWaitEvent(C.st2, ev_fork, 0));
    gauss_topup(G, done, T, topup_low, C.st2);
    TLRG_CUDA(cudaEventRecord(ev_join, C.st2));
    for (auto& pl : sample_plans) gemm_launch(pl, C.st);
    panel_tau(d_tasks, T, C.st);
    for (int sweep = 0; sweep < 2; ++sweep) {
      gemm_launch(plan_c, C.st);  // C = Q^T Y      (dense_kernels.cpp:399)
      gemm_launch(plan_y, C.st);  // Y -= Q C       (dense_kernels.cpp:400)
      panel_mgs(d_tasks, T, sweep, sweep == 1, bs, maxrows, C.st);
    }
    TLRG_CUDA(cudaStreamWaitEvent(C.st, ev_join, 0));
  };
  const char* ng = std::getenv("TLRG_NO_GRAPH");
  if (ng && ng[0] == '1') {
    // host-driven replay of the same static round (profiling / debugging)
    int* h = C.pinned_ints(2);
    for (int it = 0;; ++it) {
      enqueue_round();
      ara_loop_cond_host(active, C.st);
      TLRG_CUDA(cudaMemcpyAsync(h, active, sizeof(int) * 2, cudaMemcpyDeviceToHost, C.st));
      TLRG_CUDA(cudaStreamSynchronize(C.st));
      if (h[0] <= 0 || it + 1 >= max_rounds) break;
    }
  } else {
    cudaGraph_t graph = nullptr, body = nullptr;
    cudaGraphExec_t exec = nullptr;
    TLRG_CUDA(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle handle;
    TLRG_CUDA(cudaGraphConditionalHandleCreate(&handle, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = handle;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    TLRG_CUDA(cudaGraphAddNode(&cnode, graph, nullptr, 0, &cp));
    body = cp.conditional.phGraph_out[0];
    TLRG_CUDA(cudaStreamBeginCaptureToGraph(C.st, body, nullptr, nullptr, 0,
                                            cudaStreamCaptureModeRelaxed));
    enqueue_round();
    ara_loop_cond(handle, active, max_rounds, C.st);
    TLRG_CUDA(cudaStreamEndCapture(C.st, &body));
    TLRG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    TLRG_CUDA(cudaGraphLaunch(exec, C.st));
    graph_cleanup.push_back({exec, graph});
  }
  cudaEventDestroy(ev_fork);
  cudaEventDestroy(ev_join);
  }
  tm.stop(C.st);
  if (on_launch) on_launch();
  std::vector<int> hq(T), h_rounds(T), h_conv(T), hact(2);
  std::vector<long long> hav(T), hcur(T);
  {
    // all per-tile results in a few copies into pinned staging (pageable
    // destinations would make every copy its own blocking round trip)
    int* hI = C.pinned_ints((size_t)4 * T + 2);  // [q | rounds | conv | rank_in | active]
    double* hD = C.pinned_dbl((size_t)3 * T);   // [avail | cursor | flops]
    TLRG_CUDA(cudaMemcpyAsync(hI, qcols, sizeof(int) * 3 * T, cudaMemcpyDeviceToHost, C.st));
    if (recomp_in_kernel)
      TLRG_CUDA(cudaMemcpyAsync(hI + 3 * T, rank_in, sizeof(int) * T, cudaMemcpyDeviceToHost,
                                C.st));
    if (!use_fused)
      TLRG_CUDA(cudaMemcpyAsync(hI + 4 * T, active, sizeof(int) * 2, cudaMemcpyDeviceToHost,
                                C.st));
    if (G.cursor == G.avail + T) {
      TLRG_CUDA(cudaMemcpyAsync(hD, G.avail, sizeof(long long) * 2 * T, cudaMemcpyDeviceToHost,
                                C.st));
    } else {
      TLRG_CUDA(cudaMemcpyAsync(hD, G.avail, sizeof(long long) * T, cudaMemcpyDeviceToHost, C.st));
      TLRG_CUDA(cudaMemcpyAsync(hD + T, G.cursor, sizeof(long long) * T, cudaMemcpyDeviceToHost,
                                C.st));
    }
    if (fl_dev)
      TLRG_CUDA(cudaMemcpyAsync(hD + 2 * T, fl_dev, sizeof(double) * T, cudaMemcpyDeviceToHost,
                                C.st));
    C.wait();
    std::copy(hI, hI + T, hq.begin());
    std::copy(hI + T, hI + 2 * T, h_rounds.begin());
    std::copy(hI + 2 * T, hI + 3 * T, h_conv.begin());
    if (recomp_in_kernel) std::copy(hI + 3 * T, hI + 4 * T, h_rank_in.begin());
    hact[0] = hI[4 * T];
    hact[1] = hI[4 * T + 1];
    std::memcpy(hav.data(), hD, sizeof(long long) * T);
    std::memcpy(hcur.data(), hD + T, sizeof(long long) * T);
    if (fl_dev) std::copy(hD + 2 * T, hD + 3 * T, h_fl.begin());
  }
  g_ara_waited = std::chrono::steady_clock::now();
  for (auto& gc : graph_cleanup) {
    cudaGraphExecDestroy(gc.first);
    cudaGraphDestroy(gc.second);
  }
  if (use_fused) {
    for (int s = 0; s < T; ++s)
      if (!h_conv[s] && hq[s] < S.cap[s])
        throw CudaError("ara_batch: round limit reached with tiles still resident");
  } else {
    if (hact[0] > 0) throw CudaError("ara_batch: round limit reached with tiles still resident");
    C.launches += (long long)hact[1] * 16;
  }
  cst.t_sampling += tm.sec();  // the fused round loop (draws, sampling, orthog, absorb)
  if (use_fused) {
    cst.t_fused += tm.sec();
    cst.fused_launches += 1;
    for (int s = 0; s < T; ++s) cst.flops_fused += h_fl[s];
  }
  for (int s = 0; s < T; ++s) {
    q[s] = hq[s];
    h_av[s] = hav[s];
    h_cur[s] = hcur[s];
    cst.tile_rounds += h_rounds[s];
    if (!S.Sref.empty()) cst.flops_ref += (double)bs * h_rounds[s] * S.Sref[s];
  }
  {
    const char* fp = std::getenv("TLRG_FUSED_PROF");
    if (fp && fp[0] == '1') {
      int qm = 0;
      long long qs = 0;
      for (int s = 0; s < T; ++s) {
        qm = std::max(qm, q[s]);
        qs += q[s];
      }
      std::fprintf(stderr, "ara T=%d basis width max %d mean %.1f\n", T, qm, (double)qs / T);
    }
  }

  // tiles recompressed in the fused kernel drop out of the batched path
  std::vector<int> q_all = q;
  if (recomp_in_kernel)
    for (int s = 0; s < T; ++s)
      if (h_rank_in[s] >= 0) q[s] = 0;
  // ---- exit projection B = E^T Q (ara.cpp:380-387), all tiles at once ------
  Timer tp, tr;
  tp.start(C.st);
  std::vector<long long> boff(T);
  long long btot = 0;
  int qmax = 0;
  for (int s = 0; s < T; ++s) {
    boff[s] = btot;
    btot += (long long)cols * q[s];
    qmax = std::max(qmax, q[s]);
    if (!S.Sref.empty()) cst.flops_ref += q_all[s] * S.Sref[s];
  }
  double* Bb = C.buf<double>("B", (size_t)std::max(btot, 1LL));
  op.project(q, Q, Qstride, Bb, boff);
  tp.stop(C.st);

  // ---- recompression (ara.cpp:201-211) --------------------------------------
  tr.start(C.st);
  const char* rpe = std::getenv("TLRG_RECPROF");
  const bool recprof = rpe && rpe[0] == '1';
  auto hnow = [] { return std::chrono::steady_clock::now(); };
  auto hms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
  };
  auto h0 = hnow(), h1 = h0, h2 = h0, h3 = h0, h4 = h0;
  std::vector<int> fr(T, 0);
  const double cut = (1.0 - 1.0 / cfg.safety) * cfg.eps;
  const bool recomp = cfg.recompress && cut > 0.0;
  std::vector<long long> roff(T);
  long long rtot = 0;
  for (int s = 0; s < T; ++s) {
    roff[s] = rtot;
    rtot += (long long)q[s] * q[s];
  }
  double *Rr = nullptr, *Vs = nullptr;
  std::vector<char> is_wide(T, 0);
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
    std::vector<SvdTask> svd, svdw;
    std::vector<int> sl;
    // Bases wider than the shared-memory Jacobi skip the QR of B: one-sided
    // Jacobi on B itself (B V = Z R V = Z U_s S, the same rotations as on R in
    // exact arithmetic since B and R share their Gram matrix), one thread-block
    // cluster per tile.  B <- B V = Z U_s S in place, Q <- Q V.
    const int nst = jacobi_staged_max_n();
    const char* wbe = std::getenv("TLRG_WIDE_B");  // 0: QR + Jacobi on R for every tile (A/B)
    const bool wide_b = !(wbe && wbe[0] == '0');
    // (tall panels only: for cols < 512 the QR of B is cheap and the R core
    // goes to the cluster Jacobi below, bitwise the reference-shaped path)
    auto wide = [&](int s) {
      return wide_b && q[s] > nst && q[s] <= 512 && cols >= 512 && cols <= 1024;
    };
    long long wtot = 0;
    for (int s = 0; s < T; ++s) is_wide[s] = q[s] > 0 && recomp && wide(s);
    for (int s = 0; s < T; ++s)
      if (is_wide[s]) wtot += (long long)q[s] * (cols + q[s]);
    double* wwork = wtot ? C.buf<double>("svdwork_wide", (size_t)wtot) : nullptr;
    int qmax_n = 0;
    std::vector<long long> roff2(T, 0);
    long long rtot2 = 0;
    for (int s = 0; s < T; ++s) {
      roff2[s] = rtot2;
      if (!is_wide[s]) {
        rtot2 += q[s];
        qmax_n = std::max(qmax_n, q[s]);
      }
    }
    double* rrep = C.buf<double>("rrep", (size_t)cols * rtot2 + 1);
    {
      std::vector<int> need_s;
      std::vector<long long> need;
      for (int s = 0; s < T; ++s)
        if (q[s] && !is_wide[s]) {
          need_s.push_back(s);
          need.push_back(2LL * q[s] * cols);  // every column replaced in both sweeps
        }
      ensure(need_s, need);
    }
    h1 = hnow();
    long long wo = 0;
    for (int s = 0; s < T; ++s) {
      if (q[s] == 0) continue;
      sl.push_back(s);
      SvdTask V{};
      V.V = Vs + roff[s];
      V.sig = sig + (size_t)s * qmax;
      V.rank_out = rko + s;
      V.n = q[s];
      V.cut = cut;
      if (is_wide[s]) {
        V.A = Bb + boff[s];
        V.m = cols;
        V.work = wwork + wo;
        wo += (long long)q[s] * (cols + q[s]);
        svdw.push_back(V);
        continue;
      }
      PanelTask P{};
      P.Y = Bb + boff[s];
      P.Q = nullptr;
      P.R = Rr + roff[s];
      P.Rp = Rpr + 2 * roff[s];
      P.tiny = vec + (size_t)s * qmax * 3;
      P.col_norms = P.tiny + qmax;
      P.new_mass = P.tiny + 2 * qmax;
      P.deficient = df + (size_t)s * qmax;
      P.gbuf = G.buf + (long long)s * G.cap;
      P.gcursor = G.cursor + s;
      P.gcap = G.cap;
      P.rep = rrep + (size_t)cols * roff2[s];
      P.repC = nullptr;
      P.rows = cols;
      P.width = q[s];
      P.q = 0;
      tasks.push_back(P);
      V.A = Rr + roff[s];
      V.work = work + 2 * roff[s];
      svd.push_back(V);
    }
    // the wide tiles' clusters occupy few SMs for the batch's longest time: the
    // narrow tiles' QR + Jacobi run beside them on the side stream
    cudaEvent_t rfork = nullptr, rjoin = nullptr;
    const bool split = !svdw.empty() && !tasks.empty();
    if (split) {
      TLRG_CUDA(cudaEventCreateWithFlags(&rfork, cudaEventDisableTiming));
      TLRG_CUDA(cudaEventCreateWithFlags(&rjoin, cudaEventDisableTiming));
      TLRG_CUDA(cudaEventRecord(rfork, C.st));
      TLRG_CUDA(cudaStreamWaitEvent(C.st2, rfork, 0));
    }
    if (!svdw.empty()) {
      // widest first: they are the batch's critical path
      std::stable_sort(svdw.begin(), svdw.end(),
                       [](const SvdTask& x, const SvdTask& y) { return x.n > y.n; });
      jacobi_svd_wide(C.push(svdw), (int)svdw.size(), svdw[0].n, C.st, cols);
      ++C.launches;
    }
    if (!tasks.empty()) {
      // (on the side stream when split; the scope restores C.st on every exit)
      StreamScope side(C, split ? C.st2 : C.st);
      PanelTask* d_tasks = C.push(tasks);
      panel_tau(d_tasks, (int)tasks.size(), C.st);
      panel_mgs(d_tasks, (int)tasks.size(), 0, 0, qmax_n, cols, C.st);
      panel_mgs(d_tasks, (int)tasks.size(), 1, 1, qmax_n, cols, C.st);
      // R cores wider than the shared-memory Jacobi: one cluster each, first
      std::stable_sort(svd.begin(), svd.end(),
                       [](const SvdTask& x, const SvdTask& y) { return x.n > y.n; });
      int nwr = 0;
      while (nwr < (int)svd.size() && svd[nwr].n > nst && svd[nwr].n <= 1024) ++nwr;
      SvdTask* d_svd = C.push(svd);
      if (nwr) {
        jacobi_svd_wide(d_svd, nwr, svd[0].n, C.st);
        ++C.launches;
      }
      if (nwr < (int)svd.size())
        jacobi_svd(d_svd + nwr, (int)svd.size() - nwr, svd[nwr].n, C.st);
    }
    if (split) {
      TLRG_CUDA(cudaEventRecord(rjoin, C.st2));
      TLRG_CUDA(cudaStreamWaitEvent(C.st, rjoin, 0));
      cudaEventDestroy(rfork);
      cudaEventDestroy(rjoin);
    }
    C.launches += 4;
    h2 = hnow();
    std::vector<int> hr(T);
    TLRG_CUDA(cudaMemcpyAsync(hr.data(), rko, sizeof(int) * T, cudaMemcpyDeviceToHost, C.st));
    C.wait();
    h3 = hnow();
    for (int s : sl) fr[s] = hr[s];
  } else {
    for (int s = 0; s < T; ++s) fr[s] = q[s];
  }
  if (recomp_in_kernel)
    for (int s = 0; s < T; ++s)
      if (h_rank_in[s] >= 0) fr[s] = h_rank_in[s];
  g_ara_recomp = std::chrono::steady_clock::now();
  // ---- final factors into one contiguous panel (in out_order) -------------
  long long utot = 0, vtot = 0;
  for (int s : out_order) {
    utot += (long long)S.rows[s] * fr[s];
    vtot += (long long)cols * fr[s];
  }
  // [U panel | V panel] in one allocation (one contiguous multi-GPU send buffer)
  double* Up = (utot + vtot) ? store.alloc((size_t)(utot + vtot)) : nullptr;
  double* Vp = vtot ? Up + utot : nullptr;
  h4 = hnow();
  std::vector<GemmProblem> pu;
  std::vector<CopyItem> cpy;
  long long uo = 0, vo = 0;
  for (int s : out_order) {
    out.rank[s] = fr[s];
    out.rounds[s] = h_rounds[s];
    out.conv[s] = h_conv[s] != 0;
    if (fr[s] == 0) continue;
    out.U[s] = Up + uo;
    out.V[s] = Vp + vo;
    uo += (long long)S.rows[s] * fr[s];
    vo += (long long)cols * fr[s];
    if (recomp_in_kernel && h_rank_in[s] >= 0) {
      cpy.push_back({Uo + (size_t)s * maxrows * FUSED_QMAX, out.U[s], S.rows[s], S.rows[s],
                     S.rows[s], fr[s]});
      cpy.push_back({Vo + (size_t)s * cols * FUSED_QMAX, out.V[s], cols, cols, cols, fr[s]});
    } else if (recomp) {
      // Q <- Q V_s ;  B <- Z (U_s sigma)
      GemmProblem g{};
      g.A = Q + s * Qstride; g.lda = S.rows[s];
      g.B = Vs + roff[s]; g.ldb = q[s];
      g.C = out.U[s]; g.ldc = S.rows[s];
      g.M = S.rows[s]; g.N = fr[s]; g.K = q[s]; g.alpha = 1.0;
      pu.push_back(g);
      if (is_wide[s]) {  // B V = Z U_s S is already in place, sorted
        cpy.push_back({Bb + boff[s], out.V[s], cols, cols, cols, fr[s]});
        continue;
      }
      GemmProblem h{};
      h.A = Bb + boff[s]; h.lda = cols;
      h.B = Rr + roff[s]; h.ldb = q[s];
      h.C = out.V[s]; h.ldc = cols;
      h.M = cols; h.N = fr[s]; h.K = q[s]; h.alpha = 1.0;
      pu.push_back(h);
    } else {
      cpy.push_back({Q + s * Qstride, out.U[s], S.rows[s], S.rows[s], S.rows[s], fr[s]});
      cpy.push_back({Bb + boff[s], out.V[s], cols, cols, cols, fr[s]});
    }
  }
  if (!pu.empty()) C.gemm(pu);
  if (!cpy.empty()) {
    batched_copy(C.push(cpy), (int)cpy.size(), C.st);
    ++C.launches;
  }
  tr.stop(C.st);
  // with every tile finished in the fused kernel the projection/recompression
  // phases are empty: leave the panel copy in flight (the column's join waits
  // on this stream) instead of a host round trip just to read the timers
  if (use_fused && qmax == 0) {
    cst.pending_proj.push_back(tp.release());
    cst.pending_recomp.push_back(tr.release());
    return;
  }
  C.wait();
  if (recprof && qmax > 0) {
    int nf = 0;
    for (int s = 0; s < T; ++s) nf += q[s] > 0;
    std::fprintf(stderr,
                 "recomp fallback tiles %d qmax %d | host: setup+ensure %.3f launch %.3f wait %.3f "
                 "alloc %.3f rest %.3f | dev %.3f ms\n",
                 nf, qmax, hms(h0, h1), hms(h1, h2), hms(h2, h3), hms(h3, h4), hms(h4, hnow()),
                 tr.sec() * 1e3);
  }
  cst.t_projection += tp.sec();
  cst.t_recompress += tr.sec();
}

}  // namespace tlrg
