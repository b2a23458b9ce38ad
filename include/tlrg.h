/*
 * tlrg.h — C ABI of the B200-native TLR Cholesky / LDL^T factorization.
 *
 * Drop-in boundary for the reference's C++ API (namespace tlr, headers
 * /root/reference/proj/include/tlr/*.hpp).  Plain pointers and sizes only; all
 * matrix payloads are column-major FP64 in the reference's own layout
 * (tlr_matrix.hpp:16-59): dense diagonal tiles concatenated in tile order, lower
 * tiles (i, j), i > j, at flat index i*(i-1)/2 + j, each stored as U (rows(i) x k)
 * followed in a separate stream by V (rows(j) x k).
 *
 * Status codes follow the reference CLI (tlr_main.cpp:385-397):
 *   0 ok, 2 ConfigError, 3 DataError / DimensionError, 4 NumericError (index =
 *   failing column), 1 any other failure (CUDA error, out of memory).
 * Every call is blocking (returns after device completion).  One context owns a
 * device and its streams; distinct matrices/factors are independent.
 */
#ifndef TLRG_H
#define TLRG_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tlrg_ctx_s* tlrg_ctx;
typedef struct tlrg_matrix_s* tlrg_matrix;
typedef struct tlrg_factor_s* tlrg_factor;

/* AraConfig (ara.hpp:15-23) */
typedef struct {
  int32_t block_samples; /* bs, Gaussian vectors per round (default 32) */
  double eps;            /* absolute 2-norm threshold (default 1e-6) */
  int32_t max_rank;      /* 0 = tile size (ara_single only) */
  int32_t window;        /* convergence window, 0 = block_samples */
  double safety;         /* eta (default 10) */
  int32_t recompress;    /* SVD recompression of the small factor pair (default 1) */
  uint64_t seed;
} tlrg_ara_config;

/* AraWorkspace (ara.hpp:25-30).  On the GPU every active tile of a column is
 * resident at once; subset_capacity / parallel_buffers are accepted for API
 * parity and validated like the reference (sample_left rejects pb < #tiles). */
typedef struct {
  int32_t parallel_buffers; /* default 64 */
  int32_t dense_buffers;    /* default 20 */
  int32_t subset_capacity;  /* default 0 */
} tlrg_workspace;

/* FactorOptions (factor.hpp:15-20) */
typedef struct {
  int32_t schur_compensation; /* default 1 (forced 0 for LDL^T, factor.cpp:304) */
  double diag_shift;          /* default 0 */
  int32_t pivot_norm;         /* pivoted mode: 0 Frobenius (default), 1 2-norm power estimate */
  int32_t pivot_power_iters;  /* pivoted mode, power iterations (default 50) */
} tlrg_factor_options;

/* FactorStats (stats.hpp:9-27) plus device-side counters. */
typedef struct {
  double t_sampling, t_projection, t_reduction, t_dense, t_orthog, t_misc, t_pivot_select, wall;
  double compensation_frob;
  int32_t modified_diagonals;
  uint64_t tile_rounds_resident;
  double t_recompress;       /* untimed in the reference (ara.cpp:388-398) */
  double t_compensation;     /* Schur compensation share of t_misc */
  double flops_exec;         /* FP64 flops executed by the GEMM phases */
  double flops_gemm_ref;     /* reference-formulation F_gemm */
  int64_t kernel_launches;   /* device kernels launched by the factorization */
  double t_device;           /* CUDA-event time of the whole factorization (s) */
  double kt_gemm_seconds;    /* summed grouped-GEMM launch time (TLRG_KTIMING=1) */
  double kt_gemm_flops;      /* flops of those launches */
  int64_t kt_gemm_launches;
  double t_ara_kernel;       /* CUDA-event time of the fused ARA kernels (dominant kernel) */
  double flops_ara_kernel;   /* algorithmic FP64 flops they executed */
  int64_t ara_kernel_launches;
} tlrg_stats;

typedef struct {
  int32_t code;
  int32_t index;
  char msg[256];
} tlrg_status;

void tlrg_default_ara_config(tlrg_ara_config* cfg);
void tlrg_default_workspace(tlrg_workspace* ws);
void tlrg_default_factor_options(tlrg_factor_options* o);

int tlrg_create(int device, tlrg_ctx* ctx, tlrg_status* st);
void tlrg_destroy(tlrg_ctx ctx);

/* ------------------------------------------------------------ multi-GPU --
 * Intra-column split: with a communicator attached,
 * tlrg_factorize deals every column's rank-sorted active tiles round-robin
 * over the ranks (ARA + recompression + TRSM of its share on each GPU, diagonal
 * path replicated) and replicates the new U/V panel with one variable-size
 * all-gather per column.  The factor is bitwise identical for any rank count.
 * NCCL transport: one process per GPU; rank 0 calls tlrg_comm_nccl_id and the
 * 128-byte id is shared out of band.  Local transport: `world` contexts in one
 * process, each factorization driven by its own host thread (tests). */
int tlrg_comm_nccl_id(uint8_t* id /* 128 bytes */, tlrg_status* st);
int tlrg_comm_attach_nccl(tlrg_ctx ctx, int32_t rank, int32_t world, const uint8_t* id,
                          tlrg_status* st);
int tlrg_comm_attach_local(tlrg_ctx* ctxs, int32_t world, tlrg_status* st);
void tlrg_comm_detach(tlrg_ctx ctx);

/* ------------------------------------------------------------------ store --
 * TlrMatrix(n, b) + payload upload (replaces tlr::TlrMatrix, tlr_matrix.hpp:26-59
 * and read_tlr's in-memory result).  ranks has nb(nb-1)/2 entries. */
int tlrg_matrix_upload(tlrg_ctx ctx, int64_t n, int32_t b, double eps, const double* diag,
                       const int32_t* ranks, const double* U, const double* V, tlrg_matrix* out,
                       tlrg_status* st);
int tlrg_matrix_info(tlrg_matrix m, int64_t* n, int32_t* b, int32_t* nb, double* eps);
/* ranks (nb(nb-1)/2) */
int tlrg_matrix_ranks(tlrg_matrix m, int32_t* ranks);
/* download in the upload layout; any pointer may be NULL */
int tlrg_matrix_download(tlrg_matrix m, double* diag, double* U, double* V, tlrg_status* st);
int tlrg_matrix_copy(tlrg_matrix m, tlrg_matrix* out, tlrg_status* st);
void tlrg_matrix_free(tlrg_matrix m);
/* memory_report (tlr_matrix.cpp:229-249): out3 = total, dense, low-rank bytes */
int tlrg_memory_report(tlrg_matrix m, uint64_t* out3);
/* TLRM binary I/O (tlr_matrix.cpp:273-340), bit-compatible with the reference */
int tlrg_write_tlr(tlrg_matrix m, const char* path, tlrg_status* st);
int tlrg_read_tlr(tlrg_ctx ctx, const char* path, tlrg_matrix* out, tlrg_status* st);

/* build_tlr (tlr_matrix.cpp:98-152): construction from a covariance kernel on
 * points given in matrix order (coords n x dim, row-major per point).
 * kernel_kind 0 = exp(-r/ell), 1 = exp(-r^2/(2 ell^2)); compressor 0 = ARA, 1 = SVD. */
int tlrg_build(tlrg_ctx ctx, int32_t dim, int64_t n, const double* coords, int32_t kernel_kind,
               double ell, double nugget, int32_t b, double eps, int32_t compressor,
               const tlrg_ara_config* cfg, tlrg_matrix* out, tlrg_status* st);

/* --------------------------------------------------------------- factor ---
 * tlr_cholesky (mode 0) / tlr_ldlt (mode 1) / tlr_cholesky_pivoted (mode 2)
 * (factor.cpp:115-306; Alg. 8 tile pivoting for mode 2, uniform tiles only).
 * The matrix is CONSUMED (moved into the factor, like the reference's by-value
 * TlrMatrix A); the handle must not be used or freed afterwards. */
int tlrg_factorize(tlrg_ctx ctx, tlrg_matrix A, int32_t mode, const tlrg_ara_config* cfg,
                   const tlrg_workspace* ws, const tlrg_factor_options* opts, tlrg_factor* out,
                   tlrg_status* st);
void tlrg_factor_free(tlrg_factor f);
/* borrowed handle on L (valid while the factor lives; do not free) */
tlrg_matrix tlrg_factor_L(tlrg_factor f);
int tlrg_factor_mode(tlrg_factor f);
int tlrg_factor_stats(tlrg_factor f, tlrg_stats* out, int32_t* ara_rounds /* nb */,
                      double* pivot_trace /* nb */);
/* LDL^T parts of column k: d[n], e[n-1], start2x2[n], intra_perm[n].
   Returns 0, 2 (Cholesky factor or k out of range) or 1 (copy failed). */
int tlrg_factor_dblock(tlrg_factor f, int32_t k, double* d, double* e, uint8_t* s2, int32_t* perm);
/* pivoted mode: factor position -> original tile index (nb entries);
   returns 2 for an unpivoted factor */
int tlrg_factor_perm(tlrg_factor f, int32_t* perm);
/* TLRF I/O (factor.cpp:308-395), bit-compatible with write_factor/read_factor */
int tlrg_write_factor(tlrg_factor f, const char* path, tlrg_status* st);
int tlrg_read_factor(tlrg_ctx ctx, const char* path, tlrg_factor* out, tlrg_status* st);

/* ---------------------------------------------------------------- solve ---
 * factor_solve / factor_apply / tlr_matvec on HOST vectors (solve.cpp:144-214,
 * tlr_matrix.cpp:182-227); the copies are part of the call. */
int tlrg_factor_solve(tlrg_factor f, const double* b, double* x, tlrg_status* st);
int tlrg_factor_apply(tlrg_factor f, const double* x, double* y, tlrg_status* st);
int tlrg_tlr_matvec(tlrg_matrix A, const double* x, double* y, tlrg_status* st);
/* estimate_2norm_diff / estimate_2norm (solve.cpp:301-339) */
int tlrg_estimate_2norm_diff(tlrg_matrix A, tlrg_factor f, int32_t iters, uint64_t seed,
                             double* out, tlrg_status* st);
int tlrg_estimate_2norm(tlrg_matrix A, int32_t iters, uint64_t seed, double* out, tlrg_status* st);
/* Accuracy gates of the north star (no reference
 * function, the oracle restates the identical estimator in
 * oracle/ref_capi.cpp ref_estimate_frob_diff):
 *   tlrg_frob_norm          ||A||_F exact tile-wise
 *   tlrg_estimate_frob_diff Hutchinson estimate of ||P A P^T - L L^T||_F with
 *                           `probes` gaussian probes g_t = tlr::Rng(tile_seed(seed,
 *                           0xF20B, t, 0)), E g_t as difference_apply (solve.cpp:283-297) */
int tlrg_frob_norm(tlrg_matrix A, double* out, tlrg_status* st);
int tlrg_estimate_frob_diff(tlrg_matrix A, tlrg_factor f, int32_t probes, uint64_t seed,
                            double* out, tlrg_status* st);

/* ------------------------------------------------- building blocks (tests) -- */
/* sample_left / sample_left_transpose (ara.cpp:275-300).  omegas: per row tile,
 * rows(k) x width (or rows(i) x width transposed), concatenated.  D blocks
 * (LDL mode) as flat nb*b arrays or NULL.  out: concatenated results. */
int tlrg_sample_left(tlrg_matrix m, const double* dd, const double* de, const uint8_t* ds2,
                     int32_t k, int32_t nrows, const int32_t* rows, int32_t parallel_buffers,
                     const double* omegas, int32_t width, int32_t transpose, double* out,
                     tlrg_status* st);
/* chol_ara_update (ara.cpp:302-419) over column k of m.  Results are returned
 * through tlrg_ara_result_* accessors on the returned handle. */
typedef struct tlrg_ara_s* tlrg_ara;
int tlrg_chol_ara_update(tlrg_matrix m, const double* dd, const double* de, const uint8_t* ds2,
                         int32_t k, const tlrg_ara_config* cfg, const tlrg_workspace* ws,
                         tlrg_ara* out, tlrg_status* st);
int tlrg_ara_count(tlrg_ara a);
/* info[4] = i, rank, converged, rounds; Q rows(i) x rank, B rows(k) x rank */
int tlrg_ara_tile(tlrg_ara a, int32_t t, int32_t* info, double* Q, double* B);
void tlrg_ara_free(tlrg_ara a);
/* timing of the last tlrg_chol_ara_update: [t_device s, tile-rounds,
 * reference-formulation flops, fused-kernel s, fused-kernel flops] */
void tlrg_ara_stats(tlrg_ara a, double* out5);
/* first n gaussians of tlr::Rng(seed) generated on the device */
int tlrg_rng_gaussians(tlrg_ctx ctx, uint64_t seed, int64_t n, double* out, tlrg_status* st);
/* orthog (dense_kernels.cpp:379-420) on the device; same outputs as the
 * oracle driver: Y in/out, R (k x k), col_norms, new_mass, next draw of the rng */
int tlrg_orthog(tlrg_ctx ctx, const double* Q, int32_t rows, int32_t q, double* Y, int32_t k,
                uint64_t seed, double* R, double* col_norms, double* new_mass,
                double* next_draw, tlrg_status* st);
/* dense single-tile kernels */
int tlrg_potrf(tlrg_ctx ctx, const double* A, int32_t n, double* L, int32_t* fail,
               tlrg_status* st);
int tlrg_dense_ldl(tlrg_ctx ctx, const double* A, int32_t n, double* L, double* d, double* e,
                   uint8_t* s2, int32_t* perm, int32_t* info, tlrg_status* st);
int tlrg_schur_compensation(tlrg_ctx ctx, const double* Dk, int32_t n, double eps,
                            double* diag_out, double* frob, tlrg_status* st);
/* one-sided Jacobi SVD of an m x n matrix (the recompression core, svd_truncate
 * dense_kernels.cpp:422-454): US = A V (columns sorted by singular value,
 * descending), V (n x n), sig (n), rank = #{sig > cut}.  Cores wider than the
 * shared-memory kernel run on one thread-block cluster (force_single = 1: the
 * one-CTA kernel, for comparisons). */
int tlrg_jacobi_svd(tlrg_ctx ctx, const double* A, int32_t m, int32_t n, double cut,
                    int32_t force_single, double* US, double* V, double* sig, int32_t* rank,
                    tlrg_status* st);
int tlrg_gemm(tlrg_ctx ctx, int32_t M, int32_t N, int32_t K, int32_t transA, int32_t transB,
              double alpha, const double* A, const double* B, double beta, double* C,
              tlrg_status* st);

/* Page-locked host buffers for the upload/download calls (cudaHostAlloc);
 * transfers from/to them run at link speed.  NULL on failure. */
void* tlrg_host_alloc(uint64_t bytes);
void tlrg_host_free(void* p);

/* Library version string and the sm target it was built for. */
const char* tlrg_version(void);
/* cudaProfilerStart/Stop, to scope ncu / nsys captures to a region */
void tlrg_profiler(int on);

#ifdef __cplusplus
}
#endif
#endif /* TLRG_H */
