// Host-side launch wrappers for the sm_100a kernels (one translation unit per
// kernel family).  All wrappers are asynchronous on `st`.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <memory>
#include <vector>

#include "gemm.cuh"
#include "rng.cuh"

namespace tlrg {

// ---------------------------------------------------------------- GEMM ----
// Grouped DMMA GEMM.  `probs` is filled on the host; the launcher assigns
// tile offsets and stages the table through `desc` (device scratch reused
// after each stream synchronisation by the caller).
struct DescArena;
void grouped_gemm(std::vector<GemmProblem>& probs, DescArena& desc, cudaStream_t st);
// Two-step form: stage the table once (before a graph capture), launch many times.
struct GemmPlan {
  const GemmProblem* d = nullptr;
  const int* owner = nullptr;  // per-CTA problem index
  int n = 0, tiles = 0, bn = 32;
  int big = 0;  // 0: 64 x bn tiles; 1: 128 x 64 (8 warps); 2: 128 x 32 (4 warps)
  // a list mixing large and small problems runs as two launches: the large
  // ones on the large-tile kernel (this plan), the rest on the small one
  std::shared_ptr<GemmPlan> rest;
};
GemmPlan gemm_plan(std::vector<GemmProblem>& probs, DescArena& desc, cudaStream_t st);
void gemm_launch(const GemmPlan& p, cudaStream_t st);

// Device scratch for kernel argument tables: pinned host staging + device
// mirror, bump-allocated and reset by the owner after a stream sync.
struct DescArena {
  struct Retired {
    char* h;
    char* d;
  };
  char* h = nullptr;
  char* d = nullptr;
  size_t cap = 0, used = 0;
  std::vector<Retired> retired;  // outgrown blocks, freed at the owner's next full sync
  void reserve(size_t bytes);
  void* push(const void* src, size_t bytes, cudaStream_t st);  // returns device ptr
  void reset() { used = 0; }
  void release_retired();
  ~DescArena();
};

// ----------------------------------------------------------------- RNG ----
void rng_seed(RngState* states, const uint64_t* d_seeds, int n, cudaStream_t st);
// draw `count` gaussians for each listed state into out + t*out_stride
void rng_draw(RngState* states, const int* d_state_idx, int ntiles, double* out,
              long long count, long long out_stride, cudaStream_t st);

// Per-tile Gaussian streams (pre-generated ring buffers, consumed by cursor).
// The stream of slot s is the exact tlr::Rng(seed_s).gaussian() sequence;
// generation always appends whole polar pairs, so no pair cache is needed.
// Capacities must be even.
struct GaussStreams {
  RngState* st = nullptr;     // generator state, positioned after avail[s] values
  double* buf = nullptr;      // slot s at buf + s*cap
  long long cap = 0;
  long long* avail = nullptr;   // device, values generated
  long long* cursor = nullptr;  // device, values consumed
};
// append values to the listed slots until avail >= want (want is rounded up to even)
void gauss_generate(const GaussStreams& G, const int* d_slots, const long long* d_want, int n,
                    cudaStream_t st);
// out + a*out_stride <- next `count` values of slot d_slots[a]; advances cursors
void gauss_gather(const GaussStreams& G, const int* d_slots, int n, double* out, long long count,
                  long long out_stride, cudaStream_t st);
// one ARA round's draws for ALL slots (skipping done ones): top the stream up
// (compacting when needed) so that this round's Omega and every possible
// deficient-column replacement are available, then copy Omega_s to Om + s*cols*bs.
void gauss_round(const GaussStreams& G, const int* done, const int* rows, int nslots, int cols,
                 int bs, double* Om, cudaStream_t st);
// refill the rings of the not-done slots to capacity when fewer than `low`
// values are ahead of the cursor (the round graph runs it on a side branch)
void gauss_topup(const GaussStreams& G, const int* done, int nslots, long long low,
                 cudaStream_t st);

// --------------------------------------------------------------- ORTHOG ---
// One panel of the reference's orthog (dense_kernels.cpp:331-420) per task.
struct PanelTask {
  double* Y;          // rows x width, ld = rows
  const double* Q;    // rows x q basis (for replacement projection), ld = rows
  double* R;          // width x width accumulated factor (col-major, ld = width)
  double* Rp;         // width x width scratch
  double* tiny;       // width
  uint8_t* deficient; // width
  double* col_norms;  // width (written when finalize)
  double* new_mass;   // width
  const double* gbuf; // tile's gaussian stream (deficient-column replacements)
  long long* gcursor; // its cursor (device)
  long long gcap;     // ring capacity of the stream
  double* rep;        // rows x width scratch: projected replacement directions
  double* repC;       // q x width scratch (Q^T rep)
  double tau;         // 100 * DBL_EPSILON * ||Y_raw||_F (or DBL_MIN)
  int rows, width, q;
  // device-driven ARA round (all optional): skip when *done, basis width from
  // *qdev, and in the finalising sweep run the absorb step (ara.cpp:171-195)
  const int* done;
  const int* qdev;
  double* Qw;          // basis to append to (rows x cap)
  double* recent;      // window ring [window]
  int* qcols;          // in/out basis width
  int* rcount;
  int* rpos;
  int* rounds;
  int* conv;
  int* donew;          // done flag written by absorb
  int* active;         // decremented when the tile leaves
  int cap, window;
  double eps, eta;
};
// tau[t] = 100*eps*||Y_t||_F  (frobenius of the raw sample)
void panel_tau(PanelTask* d_tasks, int ntask, cudaStream_t st);
void panel_mgs(PanelTask* d_tasks, int ntask, int sweep, int finalize, int max_width,
               int max_rows, cudaStream_t st);

// ARA absorb step (ara.cpp:171-195) for a batch of tiles.
struct AbsorbTask {
  const double* Y;        // rows x bs orthonormal panel
  double* Q;              // rows x cap basis, ld = rows
  const double* col_norms;
  const double* new_mass;
  double* recent;         // ring buffer [window]
  int* qcols;             // in/out
  int* recent_count;      // in/out (number of valid entries, <= window)
  int* recent_pos;        // in/out ring position
  int* rounds;            // in/out
  int* converged;         // out
  int* done;              // out
  int rows, bs, cap, window;
  double eps, eta;
};
void ara_absorb(AbsorbTask* d_tasks, int ntask, cudaStream_t st);

// One-sided Jacobi SVD + truncation of small square factors (recompression,
// ara.cpp:201-211 / dense_kernels.cpp:422-454).  A (n x n) is overwritten with
// the scaled left vectors (columns sorted by singular value, descending),
// V receives right vectors; rank_out[t] = #{sigma > cut}.
struct SvdTask {
  double* A;   // n x n, ld = n
  double* V;   // n x n, ld = n
  double* sig; // n (sorted descending on exit)
  double* work; // 2 n^2 scratch, used when the problem does not fit in smem
  int* rank_out;
  int n;        // columns (V is n x n)
  double cut;
  int m;        // rows of A (0 = n)
  double tol;   // rotation threshold (0 = rounding level m * eps_mach)
};
void jacobi_svd(SvdTask* d_tasks, int ntask, int max_n, cudaStream_t st, int max_m = 0);
// Problems too large for the shared-memory path (n > jacobi_staged_max_n(),
// m, n <= 1024): one thread-block cluster per task, the same pair schedule and
// result as jacobi_svd.  max_m = largest row count (0 = max_n).
void jacobi_svd_wide(SvdTask* d_tasks, int ntask, int max_n, cudaStream_t st, int max_m = 0);
int jacobi_staged_max_n();
// symmetric (PSD) core: A <- V diag(lam), V, |lam| sorted descending (n <= 160)
void sym_jacobi(SvdTask* d_tasks, int ntask, int max_n, cudaStream_t st);

// Block-diagonal product H[:, seg_j] = U_ij * G_ij for a set of (tile, j) items.
struct BlockItem {
  const double* U;  // rows x kij, ld = rows
  const double* G;  // kij x kkj, ld = ldg
  double* H;        // rows x kkj, ld = ldh (already offset to seg_j)
  long long ldg, ldh;
  int rows, kij, kkj;
};
void block_products(BlockItem* d_items, int nitems, int max_rows, cudaStream_t st);
// The same products with the per-block fields derived on the device from the
// tile tables (rank / U pointer per lower tile, tri_index order) instead of a
// host-expanded T x J item list.  cols: [targets T | J nJ | S nJ | seg nJ |
// kkj nJ | goff nJ].  Block (t, jj) = blockIdx.x = t * nJ + jj.
struct HProductArgs {
  const long long* cols;
  const int* rank;
  const double* const* U;
  const double* G;
  double* H;
  long long stride, n;
  int T, nJ, k, b;
};
void h_products(const HProductArgs& a, cudaStream_t st);
// tile-table mirror update: rank[t[e]] = r[e], U[t[e]] = u[e]
void tri_update(const long long* t, const int* r, const double* const* u, int n, int* rank,
                const double** U, cudaStream_t st);

// Copy/gather helpers
struct CopyItem {
  const double* src;
  double* dst;
  long long lds, ldd;
  int rows, cols;
};
void batched_copy(CopyItem* d_items, int n, cudaStream_t st);

// ------------------------------------------------------------ FUSED ARA ---
// One CTA per tile runs the whole adaptive loop (ara_fused.cu).
struct FusedSlot {
  // low-rank chain operator: Y = U^A (V^A^T Om) - H (Ucat^T Om)
  const double* UA;   // rows x kA (ld rows)
  const double* VA;   // cols x kA (ld cols)
  const double* H;    // rows x K  (ld rows)
  int kA;
  // dense operator (build_tlr's DenseSampler): Y = Ad Om when Ad != null
  const double* Ad;
  long long ldad;
  int rows, cap;
  double* Q;     // rows x cap basis (ld rows), output
  double* Om;    // cols x bs scratch
  double* W;     // (kA + K) x bs scratch
  double* Cq;    // fused: (2 cap + bs + 4) x bs scratch (C = Q^T Y, then sweep-2 coefficients)
  double* repC;  // cap scratch
  double* Uo;    // rows x QMAX recompressed U (Q V_s), written when recompressed in-kernel
  double* Vo;    // cols x QMAX recompressed V before TRSM (Z U_s sigma)
};
struct FusedArgs {
  const FusedSlot* slots;
  GaussStreams G;
  const double* Ucat;  // cols x K (ld cols), shared by all slots
  int K, cols, bs, window, max_rounds;
  double eps, eta;
  int* qcols;
  int* rounds;
  int* conv;
  int ldy;          // set by the launcher
  long long ysz;    // set by the launcher
  long long stg_half;  // set by the launcher
  long long* prof;     // optional per-slot phase cycle counters (8 per slot)
  int recompress;      // run the exit projection + SVD recompression in-kernel
  double cut;          // (1 - 1/eta) eps
  int* rank_out;       // final rank, or -1 when the tile needs the batched fallback
  double* flops_out;   // per slot: algorithmic FP64 flops executed by the CTA
  int mgs_passes;      // column passes per sweep in the panel MGS (reference: 2)
  int stage;           // TMA-stage the sampling operands (set by the launcher)
  int fast_sweep2;     // second orthog sweep as one Gram product (see ara_fused.cu)
  int dcgs;            // panel CGS2 with one reduction per column (see ara_fused.cu)
};
constexpr int FUSED_QMAX = 32;  // widest basis recompressed in-kernel
bool ara_fused_supported(int maxrows, int bs, int window);
// cl: CTAs per tile (thread-block cluster; 1, 2 or 4) sharing each round's
// sampling products (chain operator only, bs = 16)
void ara_fused(FusedArgs args, int T, int maxrows, cudaStream_t st, int cl = 1);

// ---------------------------------------------------------------- DENSE ---
// Cholesky of an m x m tile in place (lower); info[0] = failing column or -1.
void potrf_impl(double* A, int n, int* info, DescArena& desc, cudaStream_t st);
// Bunch-Kaufman (LAPACK dsytf2, lower) with the reference's unpacking
// (dense_kernels.cpp:236-281): A -> unit-lower L, D (d, e, start2x2), perm.
void sytrf_bk(double* A, int n, double* d, double* e, uint8_t* s2, int* perm, int* info,
              cudaStream_t st);
// X <- L^{-1} B (Chol) or X <- D^{-1} Lunit^{-1} P B (LDL), B rows x nrhs (ld rows).
void trsm_panel(const double* L, int n, double* B, long long nrhs, const int* perm,
                const double* d, const double* e, const uint8_t* s2, int* info,
                cudaStream_t st, double* work = nullptr /* n x nrhs, LDL mode */);
// (shifted) Cholesky-QR step: R^T R = G (+ shift), Rinv = R^{-1}, p <= 160
void cholqr_factor(const double* G, int p, int n, int shift, double* Rinv, cudaStream_t st);
// Y (n x p, ld n) <- Y R^{-1} (R^{-1} upper p x p from cholqr_factor's
// Rinv output); columns with a dropped pivot are zeroed.  In place.
void cholqr_apply(double* Y, int n, int p, const double* R, cudaStream_t st);
// X_bb = L_bb^{-1} for diagonal blocks (offset, length <= 32) of an n x n lower L
void trtri_base(const double* L, int n, double* X, const int* d_offs, const int* d_lens,
                int nblocks, cudaStream_t st);
// D <- 0.5 (D + D^T)
void symmetrize(double* D, int n, cudaStream_t st);
// out = A - D (+ diag(corr)) (+ shift I)
void diag_combine(const double* A, const double* D, const double* corr, double shift,
                  double* out, int n, cudaStream_t st);
// pivot trace helpers
void min_diag_sq(const double* L, int n, double* out, cudaStream_t st);
void min_block_pivot(const double* d, const double* e, const uint8_t* s2, int n, double* out,
                     cudaStream_t st);
// W <- D_j W  (block diagonal apply, rows of W)
struct BdItem {
  const double* d;
  const double* e;
  const uint8_t* s2;
  double* W;
  int cols;
};
void bd_apply_batched(const BdItem* d_items, int nitems, int n, long long ld, cudaStream_t st);
void bd_apply(const double* d, const double* e, const uint8_t* s2, int n, double* W,
              long long ld, int cols, cudaStream_t st);
// Schur compensation helpers
void sym_jacobi_eig(double* B, double* V, double* w, int n, cudaStream_t st);
void rowsum_abs_residual(const double* D, const double* X, const double* lam, int n, int r,
                         double* corr, double* frob_sq, cudaStream_t st);
void fill_gaussian_philox(double* out, long long n, uint64_t seed, cudaStream_t st);

// generic elementwise
void fill_zero(double* p, long long n, cudaStream_t st);
void frob_sq(const double* p, long long n, double* out, cudaStream_t st);
// *out = sum of n values (one CTA, fixed order)
void block_sum_device(const double* p, int n, double* out, cudaStream_t st);

}  // namespace tlrg
