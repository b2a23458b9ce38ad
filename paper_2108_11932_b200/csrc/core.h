// Internal host-side structures of the B200 TLR library.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "kernels.h"

namespace tlrg {

// Error taxonomy of the reference (errors.hpp:10-30) mapped to status codes.
struct Error : std::runtime_error {
  int code, index;
  Error(int c, const std::string& m, int idx = -1) : std::runtime_error(m), code(c), index(idx) {}
};
[[noreturn]] inline void config_error(const std::string& m) { throw Error(2, m); }
[[noreturn]] inline void data_error(const std::string& m) { throw Error(3, m); }
[[noreturn]] inline void numeric_error(const std::string& m, int idx) { throw Error(4, m, idx); }


// Grow-only device scratch buffer.  Only resized at synchronisation points.
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  template <class T>
  T* get(size_t count) {
    size_t bytes = count * sizeof(T) + 256;
    if (bytes > cap) {
      if (p) TLRG_CUDA(cudaFree(p));
      size_t c = bytes + bytes / 4;
      TLRG_CUDA(cudaMalloc(&p, c));
      cap = c;
    }
    return static_cast<T*>(p);
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

// Device memory for low-rank payloads (append-only chunks, never moved).
// Live contexts: stream-ordered frees go to the owner's stream only while it
// exists (Python may collect a matrix after its context); otherwise cudaFree.
bool ctx_alive(const void* ctx);
void ctx_register(const void* ctx, bool alive);
// Per-context cache of standard-size Store chunks: a freed matrix's chunks are
// reused by the next one without a CUDA call (pool growth under
// cudaMallocAsync measured 0.5 - 60 ms per 64 MiB chunk inside the loop).
void chunk_cache_release(const void* ctx);
// top the cache up to cover `doubles` (one pool call per missing chunk, made
// while the device is idle at the start of a factorization)
void chunk_cache_reserve(const void* ctx, size_t doubles, cudaStream_t st);
void stream_free(const void* ctx, cudaStream_t st, void* p);

struct Store {
  cudaStream_t st = nullptr;  // stream-ordered pool allocations (set by the owner)
  const void* owner = nullptr;
  std::vector<void*> chunks;
  std::vector<size_t> chunk_len;  // doubles per chunk
  double* cur = nullptr;
  size_t cap = 0, used = 0;
  size_t total = 0;
  double* alloc(size_t n);
  ~Store();
};

struct Ctx;
// Transport of the multi-GPU column exchange (comm.cu): NCCL or in-process ranks.
struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() = default;
  // host ints: every rank sends n, receives n * world (rank-major)
  virtual void allgather_ints(Ctx& C, const int* send, int n, int* recv) = 0;
  // device buffers: rank r's `counts[r]` doubles land in dst[r] on every other rank
  virtual void broadcast_all(Ctx& C, const double* mine, const std::vector<double*>& dst,
                             const std::vector<long long>& counts) = 0;
};

struct Ctx {
  int device = 0;
  std::shared_ptr<Comm> comm;  // set for multi-GPU factorizations (world > 1)
  cudaStream_t st = nullptr;
  cudaStream_t st2 = nullptr;  // side stream (gaussian stream pre-generation)
  cudaStream_t sd = nullptr;   // diagonal-path stream (SYRK, compensation, POTRF, L_kk^-1)
  cudaStream_t st_main = nullptr;  // the context's own stream (st may be swapped by StreamScope)
  DescArena desc;
  std::map<std::string, DevBuf> bufs;
  // pinned host staging for small D2H reads
  int* h_ints = nullptr;
  size_t h_ints_cap = 0;
  double* h_dbl = nullptr;
  size_t h_dbl_cap = 0;
  double flops = 0.0;
  long long launches = 0;
  // optional per-launch CUDA-event timing of the grouped GEMM (TLRG_KTIMING=1)
  bool ktiming = false;
  double kt_seconds = 0.0, kt_flops = 0.0;
  long long kt_launches = 0;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<std::pair<cudaEvent_t, cudaEvent_t>, double>> ev_pending;

  template <class T>
  T* buf(const std::string& name, size_t count) {
    return bufs[name].get<T>(count);
  }
  int* pinned_ints(size_t n);
  double* pinned_dbl(size_t n);
  cudaEvent_t take_event() {
    if (ev_pool.empty()) {
      cudaEvent_t e;
      TLRG_CUDA(cudaEventCreate(&e));
      return e;
    }
    cudaEvent_t e = ev_pool.back();
    ev_pool.pop_back();
    return e;
  }
  void drain_events() {
    for (auto& p : ev_pending) {
      float ms = 0;
      cudaEventElapsedTime(&ms, p.first.first, p.first.second);
      kt_seconds += ms * 1e-3;
      kt_flops += p.second;
      ++kt_launches;
      ev_pool.push_back(p.first.first);
      ev_pool.push_back(p.first.second);
    }
    ev_pending.clear();
  }
  // full synchronisation point: every stream of the context is idle, so the
  // descriptor arena can be recycled
  void sync() {
    TLRG_CUDA(cudaStreamSynchronize(st));
    if (sd) TLRG_CUDA(cudaStreamSynchronize(sd));
    if (st_main && st_main != st) TLRG_CUDA(cudaStreamSynchronize(st_main));
    desc.reset();
    desc.release_retired();
    if (!ev_pending.empty()) drain_events();
  }
  // wait for the current stream only (no arena recycling): other streams keep
  // running, e.g. the diagonal path while the ARA host loop reads its flags
  void wait() { TLRG_CUDA(cudaStreamSynchronize(st)); }
  template <class T>
  T* push(const std::vector<T>& v) {
    if (v.empty()) return nullptr;
    return static_cast<T*>(desc.push(v.data(), v.size() * sizeof(T), st));
  }
  void gemm(std::vector<GemmProblem>& probs) {
    double f = 0.0;
    for (auto& p : probs)
      if (p.M > 0 && p.N > 0) f += 2.0 * p.M * p.N * p.K;
    flops += f;
    if (ktiming && f > 0) {
      cudaEvent_t a = take_event(), b = take_event();
      TLRG_CUDA(cudaEventRecord(a, st));
      grouped_gemm(probs, desc, st);
      TLRG_CUDA(cudaEventRecord(b, st));
      ev_pending.push_back({{a, b}, f});
    } else {
      grouped_gemm(probs, desc, st);
    }
    ++launches;
  }
  ~Ctx();
};

// Enqueue everything issued inside the scope on another stream of the context
// (the helpers all launch on C.st).
struct StreamScope {
  Ctx& C;
  cudaStream_t saved;
  StreamScope(Ctx& c, cudaStream_t s) : C(c), saved(c.st) { C.st = s; }
  ~StreamScope() { C.st = saved; }
};

// Flat TLR store in HBM (replaces TlrMatrix/LowRankTile/DenseTile,
// tlr_matrix.hpp:16-59): dense diagonal tiles at diag + k*b*b (ld rows(k)),
// low-rank factors addressed through per-tile device pointers and ranks.
struct Matrix {
  Ctx* ctx = nullptr;
  int64_t n = 0;
  int b = 0, nb = 0;
  double eps = 0.0;
  double* diag = nullptr;              // owned
  std::vector<int> rank;               // nb(nb-1)/2
  std::vector<double*> U, V;           // device pointers (null when rank 0)
  std::vector<std::shared_ptr<Store>> stores;  // own the payloads

  int rows(int i) const {
    int64_t r = n - (int64_t)i * b;
    return r < b ? (int)r : b;
  }
  long long t(int i, int j) const { return tri_index(i, j); }
  void free_all();
  ~Matrix() { free_all(); }
};

struct AraCfg {
  int bs = 32;
  double eps = 1e-6;
  int max_rank = 0;
  int window = 0;
  double safety = 10.0;
  bool recompress = true;
  uint64_t seed = 0;
};

// Device-resident LDL^T blocks D_j (flat nb*b arrays), or all null for Chol.
struct DBlocks {
  double* d = nullptr;
  double* e = nullptr;
  uint8_t* s2 = nullptr;
  int* perm = nullptr;
  bool on() const { return d != nullptr; }
};

struct TileResult {
  int i = 0, rank = 0, rounds = 0;
  bool converged = true;
  double* U = nullptr;  // rows(i) x rank (device)
  double* V = nullptr;  // rows(k) x rank (device, before TRSM)
};

struct ColumnStats {
  double t_sampling = 0, t_orthog = 0, t_projection = 0, t_recompress = 0, t_dense = 0;
  long long tile_rounds = 0;
  double flops_ref = 0;  // reference-formulation sampling+projection flops
  double t_fused = 0, flops_fused = 0;  // fused ARA kernel: event time and in-kernel flops
  long long fused_launches = 0;
  // event pairs still in flight when column_ara returned (read at the column
  // join by column_stats_resolve): projection and recompression phases
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending_proj, pending_recomp;
};
// fold the deferred phase timers into t_projection / t_recompress (after a sync)
void column_stats_resolve(ColumnStats& cst);

// Column machinery shared by the factorization and the building-block API.
struct ColumnSetup {
  int k = 0, rk = 0, K = 0;
  std::vector<int> J;          // j < k with rank(k, j) > 0
  std::vector<int> seg;        // column offset of block j in Ucat (indexed like J)
  double* Ucat = nullptr;      // rk x K
  double* Wcat = nullptr;      // b x K  (D_j V_kj)
  double* G = nullptr;         // Gram blocks, per j: S_j x k_kj
  std::vector<long long> goff; // per J entry
  std::vector<int> S;          // per J entry
  std::vector<int> sub_first;  // first i of the gathered suffix (k)
  // device mirror of the tile tables (set by the factorization): the ARA's
  // H_i products then derive their block fields on the device
  const int* d_rank = nullptr;
  const double* const* d_U = nullptr;
};

void column_setup(Ctx& C, const Matrix& M, int k, const DBlocks& D, ColumnSetup& cs);
// H_i = U_i,: G_i for the listed target rows (rows(i) x K each, ld rows(i)).
void column_H(Ctx& C, const Matrix& M, const ColumnSetup& cs, const std::vector<int>& targets,
              double* H, long long stride);

// Generic batched ARA (ara.cu).  Slot s is one tile: rows(s) x cols operator.
struct AraSlots {
  std::vector<int> rows, cap;
  std::vector<uint64_t> seeds;
  std::vector<double> Sref;  // reference flops per sampled vector (optional)
  int cols = 0;
};
// Operator in the fused kernel's form (ara_fused.cu); optional.
struct AraFusedOp {
  bool on = false;
  std::vector<const double*> UA, VA, H, Ad;
  std::vector<int> kA;
  std::vector<long long> ldad;
  const double* Ucat = nullptr;
  int K = 0;
};
struct AraOperator {
  AraFusedOp fused;
  // GEMM stages computing Y_s = E_s Omega_s for every slot s (Omega_s at
  // Om + s*cols*bs, Y_s at Y + s*Ystride); each problem must carry
  // skip = done + s so converged tiles cost nothing in later rounds
  std::function<void(const double* Om, double* Y, long long Ystride, const int* done,
                     std::vector<std::vector<GemmProblem>>& stages)> sample_plan;
  // enqueue B_s = E_s^T Q_s (cols x q_s, ld cols) at Bb + boff[s] for q_s > 0
  std::function<void(const std::vector<int>& q, const double* Q, long long Qstride, double* Bb,
                     const std::vector<long long>& boff)> project;
};
struct AraOut {
  std::vector<int> rank, rounds, conv;
  std::vector<double*> U, V;
};
// Per-slot gaussian streams seeded and pre-generated on the side stream, so the
// generation overlaps whatever the main stream does until the ARA starts.
struct StreamPrep {
  GaussStreams G;
  cudaEvent_t ev = nullptr;
  int T = 0;
  long long pre = 0;  // values generated per slot
  std::vector<uint64_t> seeds;
  int k = -1;              // column the queue below belongs to
  std::vector<int> queue;  // column_queue(M, k), reused by column_ara
  ~StreamPrep() {
    if (ev) cudaEventDestroy(ev);
  }
};
// the fused one-launch ARA applies (even tile sizes, shared-memory budget)
bool ara_fused_eligible(int cols, const std::vector<int>& rows, int bs, int window);
// rounds_ahead rounds of every slot's stream generated on the side stream;
// ring capacity ring_rounds rounds plus replacement room
void streams_prepare(Ctx& C, const std::vector<uint64_t>& seeds, int cols, int bs, int maxrows,
                     int rounds_ahead, StreamPrep& P, int ring_rounds = 12);
void ara_batch(Ctx& C, const AraSlots& S, const AraOperator& op, const AraCfg& cfg, Store& store,
               const std::vector<int>& out_order, ColumnStats& cst, AraOut& out,
               StreamPrep* pre = nullptr, const std::function<void()>& on_launch = {});

// Dynamic-batched ARA over column k (chol_ara_update, ara.cpp:302-419): all
// non-trivial tiles resident, converged tiles leave, exit projection and SVD
// recompression batched at the end.  Results (ascending i) land in a panel
// allocated from `store` (U: sum rows(i)*r, V: rk x sum r contiguous).
std::vector<TileResult> column_ara(Ctx& C, const Matrix& M, int k, const ColumnSetup& cs,
                                   const AraCfg& cfg, Store& store, ColumnStats& cst,
                                   StreamPrep* pre = nullptr, int part_rank = 0,
                                   int part_world = 1,
                                   const std::function<void()>& on_launch = {});
// on_launch: called once the column's ARA work is enqueued (before the host
// waits on it) -- the factorization enqueues its diagonal path there
// multi-GPU: replicate the column's new U/V panel (comm.cu)
void exchange_column(Ctx& C, Comm& cm, const Matrix& M, int k, const std::vector<int>& queue,
                     std::vector<TileResult>& res, double* mine, Store& store);
std::shared_ptr<Comm> make_nccl_comm(int rank, int world, const uint8_t* id);
std::vector<std::shared_ptr<Comm>> make_local_comms(int world);
// slot order of column k's ARA (rank-sorted, structural zeros removed) and the
// early stream pre-generation for it (call at the start of the column)
std::vector<int> column_queue(const Matrix& M, int k);
void column_prepare(Ctx& C, const Matrix& M, int k, const AraCfg& cfg, StreamPrep& P);

struct FactorOpts {
  bool schur = true;
  double shift = 0.0;
  int pivot_norm = 0;          // pivoted mode: 0 Frobenius, 1 power 2-norm estimate
  int pivot_power_iters = 50;
};

struct Stats {
  double t_sampling = 0, t_projection = 0, t_reduction = 0, t_dense = 0, t_orthog = 0,
         t_misc = 0, t_pivot_select = 0, wall = 0, compensation_frob = 0;
  int modified_diagonals = 0;
  uint64_t tile_rounds_resident = 0;
  double t_recompress = 0, t_compensation = 0, flops_exec = 0, flops_ref = 0;
  double t_device = 0;        // CUDA-event time of the whole factorization
  double t_fused = 0, flops_fused = 0;  // fused ARA kernel (the dominant kernel)
  long long fused_launches = 0;
  double kt_gemm_seconds = 0, kt_gemm_flops = 0;  // per-launch GEMM timing (KTIMING)
  long long kt_gemm_launches = 0;
  long long launches = 0;
  std::vector<int> ara_rounds;
  std::vector<double> pivot_trace;
};

struct Factor {
  std::unique_ptr<Matrix> L;
  int mode = 0;  // 0 Chol, 1 LDLT, 2 pivoted Chol
  DBlocks D;     // owned device arrays in LDL mode
  std::vector<int> perm;  // pivoted mode: factor position -> tile (factor.hpp:29)
  int* d_perm = nullptr;  // device copy (solve / residual operators)
  double eps = 0.0;
  Stats stats;
  ~Factor();
};
// tile permutation of a length-n vector (solve.cpp:124-140): forward
// out[block k] = in[block perm[k]], inverse out[block perm[k]] = in[block k]
void tile_perm_device(Ctx& C, const Factor& F, const double* in, double* out, bool inverse);
// pivot_swap(k, p, finalized = k) (tlr_matrix.cpp:66-82) on the tile tables
void pivot_swap_tables(Matrix& M, int k, int p);

std::unique_ptr<Factor> factorize(Ctx& C, std::unique_ptr<Matrix> A, int mode, const AraCfg& cfg,
                                  int parallel_buffers, const FactorOpts& opts);

// build_tlr (tlr_matrix.cpp:98-152) on the device; coords in matrix order.
std::unique_ptr<Matrix> build_tlr_device(Ctx& C, int dim, int64_t n, const double* coords_host,
                                         int kind, double ell, double nugget, int b, double eps,
                                         int compressor, const AraCfg& cfg);

// dense building blocks on device memory
bool potrf_device(Ctx& C, double* A, int n);  // returns success
// modified_cholesky (dense_kernels.cpp:283-309): A in, L out (in place); returns modified flag
bool modified_cholesky_device(Ctx& C, double* A, int n);
void schur_compensation_device(Ctx& C, const double* Dk, int n, double eps, uint64_t seed,
                               double* corr, double* frob, int& rank_hint);

// solve/apply/matvec on device vectors
void matvec_device(Ctx& C, const Matrix& A, const double* x, double* y);
void factor_apply_device(Ctx& C, const Factor& F, const double* x, double* y);
void factor_solve_device(Ctx& C, const Factor& F, double* x);  // in place
double dot_device(Ctx& C, const double* a, const double* b, long long n);
// w = (P A P^T - L L^T) v in the factor frame (difference_apply, solve.cpp:283-297);
// t is n doubles of scratch
void difference_apply_device(Ctx& C, const Matrix& A, const Factor& F, const double* v, double* w,
                             double* t);
// ||A||_F exact tile-wise; Hutchinson estimate of ||P A P^T - L L^T||_F
double frob_norm_device(Ctx& C, const Matrix& A);
double estimate_frob_diff_device(Ctx& C, const Matrix& A, const Factor& F, int probes,
                                 uint64_t seed);
// y <- a*x + b*y on C.st
void axpby_device(Ctx& C, double a, const double* x, double b, double* y, long long n);

}  // namespace tlrg
