// extern "C" boundary (include/tlrg.h) over the device implementation.
#include <cuda_profiler_api.h>

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <memory>

#include "../../include/tlrg.h"
#include "core.h"

using namespace tlrg;

struct tlrg_ctx_s {
  Ctx c;
};
struct tlrg_matrix_s {
  std::unique_ptr<Matrix> m;
  bool borrowed = false;
};
struct tlrg_factor_s {
  std::unique_ptr<Factor> f;
  tlrg_matrix_s Lview;
  Ctx* ctx;
};
struct tlrg_ara_s {
  std::vector<int> i, rank, conv, rounds;
  std::vector<std::vector<double>> Q, B;
  double t_device = 0, t_fused = 0, flops_fused = 0, flops_ref = 0;
  long long tile_rounds = 0;
};

namespace {
void set_status(tlrg_status* st, int code, const char* msg, int index = -1) {
  if (!st) return;
  st->code = code;
  st->index = index;
  std::snprintf(st->msg, sizeof st->msg, "%s", msg ? msg : "");
}
template <class F>
int guarded(tlrg_status* st, F&& f) {
  try {
    f();
    set_status(st, 0, "");
    return 0;
  } catch (const Error& e) {
    set_status(st, e.code, e.what(), e.index);
    return e.code;
  } catch (const std::exception& e) {
    set_status(st, 1, e.what());
    return 1;
  }
}
AraCfg to_cfg(const tlrg_ara_config* c) {
  AraCfg a;
  if (!c) return a;
  a.bs = c->block_samples;
  a.eps = c->eps;
  a.max_rank = c->max_rank;
  a.window = c->window;
  a.safety = c->safety;
  a.recompress = c->recompress != 0;
  a.seed = c->seed;
  return a;
}

std::unique_ptr<Matrix> upload(Ctx& C, int64_t n, int b, double eps, const double* diag,
                               const int32_t* ranks, const double* U, const double* V) {
  if (n < 1 || b < 1 || b > n) config_error("TlrMatrix: bad dimensions");
  auto M = std::make_unique<Matrix>();
  M->ctx = &C;
  M->n = n;
  M->b = b;
  M->nb = (int)((n + b - 1) / b);
  M->eps = eps;
  const int nb = M->nb;
  size_t nt = (size_t)nb * (nb - 1) / 2;
  M->rank.assign(nt, 0);
  M->U.assign(nt, nullptr);
  M->V.assign(nt, nullptr);
  TLRG_CUDA(cudaMallocAsync(&M->diag, sizeof(double) * (size_t)nb * b * b, C.st_main));
  if (diag && n % b == 0) {
    TLRG_CUDA(cudaMemcpyAsync(M->diag, diag, sizeof(double) * (size_t)nb * b * b,
                              cudaMemcpyHostToDevice, C.st));
  } else {
    size_t off = 0;
    for (int k = 0; k < nb; ++k) {
      int r = M->rows(k);
      if (diag)
        TLRG_CUDA(cudaMemcpyAsync(M->diag + (size_t)k * b * b, diag + off, sizeof(double) * r * r,
                                  cudaMemcpyHostToDevice, C.st));
      else
        TLRG_CUDA(cudaMemsetAsync(M->diag + (size_t)k * b * b, 0, sizeof(double) * r * r, C.st));
      off += (size_t)r * r;
    }
  }
  size_t totU = 0, totV = 0;
  for (int i = 1; i < nb; ++i)
    for (int j = 0; j < i; ++j) {
      int r = ranks ? ranks[tri_index(i, j)] : 0;
      if (r < 0) data_error("TlrMatrix: negative rank");
      totU += (size_t)M->rows(i) * r;
      totV += (size_t)M->rows(j) * r;
    }
  auto S = std::make_shared<Store>();
  S->st = C.st_main;
  S->owner = &C;
  M->stores.push_back(S);
  double* dU = totU ? S->alloc(totU) : nullptr;
  double* dV = totV ? S->alloc(totV) : nullptr;
  if (totU) TLRG_CUDA(cudaMemcpyAsync(dU, U, sizeof(double) * totU, cudaMemcpyHostToDevice, C.st));
  if (totV) TLRG_CUDA(cudaMemcpyAsync(dV, V, sizeof(double) * totV, cudaMemcpyHostToDevice, C.st));
  C.sync();
  size_t ou = 0, ov = 0;
  for (int i = 1; i < nb; ++i)
    for (int j = 0; j < i; ++j) {
      long long t = tri_index(i, j);
      int r = ranks ? ranks[t] : 0;
      M->rank[t] = r;
      if (r) {
        M->U[t] = dU + ou;
        M->V[t] = dV + ov;
      }
      ou += (size_t)M->rows(i) * r;
      ov += (size_t)M->rows(j) * r;
    }
  return M;
}

// Device-side gather of the tile payloads into the reference's flat layout,
// then ONE device->host copy per stream (pinned host memory runs at link speed).
void download(const Matrix& M, double* diag, double* U, double* V) {
  Ctx& C = *M.ctx;
  const int nb = M.nb, b = M.b;
  if (diag) {
    if (M.n % b == 0) {
      TLRG_CUDA(cudaMemcpyAsync(diag, M.diag, sizeof(double) * (size_t)nb * b * b,
                                cudaMemcpyDeviceToHost, C.st));
    } else {
      size_t off = 0;
      for (int k = 0; k < nb; ++k) {
        int r = M.rows(k);
        TLRG_CUDA(cudaMemcpyAsync(diag + off, M.diag + (size_t)k * b * b, sizeof(double) * r * r,
                                  cudaMemcpyDeviceToHost, C.st));
        off += (size_t)r * r;
      }
    }
  }
  size_t tu = 0, tv = 0;
  for (int i = 1; i < nb; ++i)
    for (int j = 0; j < i; ++j) {
      int r = M.rank[tri_index(i, j)];
      tu += (size_t)M.rows(i) * r;
      tv += (size_t)M.rows(j) * r;
    }
  if (U || V) {
    double* su = (U && tu) ? C.buf<double>("dl_U", tu) : nullptr;
    double* sv = (V && tv) ? C.buf<double>("dl_V", tv) : nullptr;
    std::vector<CopyItem> cp;
    size_t ou = 0, ov = 0;
    for (int i = 1; i < nb; ++i)
      for (int j = 0; j < i; ++j) {
        long long t = tri_index(i, j);
        int r = M.rank[t];
        if (r) {
          if (su) cp.push_back({M.U[t], su + ou, M.rows(i), M.rows(i), M.rows(i), r});
          if (sv) cp.push_back({M.V[t], sv + ov, M.rows(j), M.rows(j), M.rows(j), r});
        }
        ou += (size_t)M.rows(i) * r;
        ov += (size_t)M.rows(j) * r;
      }
    if (!cp.empty()) batched_copy(C.push(cp), (int)cp.size(), C.st);
    if (su) TLRG_CUDA(cudaMemcpyAsync(U, su, sizeof(double) * tu, cudaMemcpyDeviceToHost, C.st));
    if (sv) TLRG_CUDA(cudaMemcpyAsync(V, sv, sizeof(double) * tv, cudaMemcpyDeviceToHost, C.st));
  }
  C.sync();
}

std::unique_ptr<Matrix> clone(Ctx& C, const Matrix& M) {
  auto R = std::make_unique<Matrix>();
  R->ctx = &C;
  R->n = M.n;
  R->b = M.b;
  R->nb = M.nb;
  R->eps = M.eps;
  R->rank = M.rank;
  R->U.assign(M.U.size(), nullptr);
  R->V.assign(M.V.size(), nullptr);
  size_t dbytes = sizeof(double) * (size_t)M.nb * M.b * M.b;
  TLRG_CUDA(cudaMallocAsync(&R->diag, dbytes, C.st_main));
  TLRG_CUDA(cudaMemcpyAsync(R->diag, M.diag, dbytes, cudaMemcpyDeviceToDevice, C.st));
  size_t tot = 0;
  for (int i = 1; i < M.nb; ++i)
    for (int j = 0; j < i; ++j) {
      int r = M.rank[tri_index(i, j)];
      tot += (size_t)(M.rows(i) + M.rows(j)) * r;
    }
  auto S = std::make_shared<Store>();
  S->st = C.st_main;
  S->owner = &C;
  R->stores.push_back(S);
  double* base = tot ? S->alloc(tot) : nullptr;
  size_t o = 0;
  for (int i = 1; i < M.nb; ++i)
    for (int j = 0; j < i; ++j) {
      long long t = tri_index(i, j);
      int r = M.rank[t];
      if (!r) continue;
      size_t nu = (size_t)M.rows(i) * r, nv = (size_t)M.rows(j) * r;
      R->U[t] = base + o;
      TLRG_CUDA(cudaMemcpyAsync(R->U[t], M.U[t], nu * 8, cudaMemcpyDeviceToDevice, C.st));
      o += nu;
      R->V[t] = base + o;
      TLRG_CUDA(cudaMemcpyAsync(R->V[t], M.V[t], nv * 8, cudaMemcpyDeviceToDevice, C.st));
      o += nv;
    }
  C.sync();
  return R;
}

struct DUpload {
  DBlocks D;
  ~DUpload() {
    if (D.d) cudaFree(D.d);
    if (D.e) cudaFree(D.e);
    if (D.s2) cudaFree(D.s2);
  }
};
void upload_d(DUpload& u, const Matrix& M, const double* dd, const double* de, const uint8_t* ds2) {
  if (!dd) return;
  size_t n = (size_t)M.nb * M.b;
  TLRG_CUDA(cudaMalloc(&u.D.d, n * 8));
  TLRG_CUDA(cudaMalloc(&u.D.e, n * 8));
  TLRG_CUDA(cudaMalloc(&u.D.s2, n));
  TLRG_CUDA(cudaMemcpy(u.D.d, dd, n * 8, cudaMemcpyHostToDevice));
  TLRG_CUDA(cudaMemcpy(u.D.e, de, n * 8, cudaMemcpyHostToDevice));
  TLRG_CUDA(cudaMemcpy(u.D.s2, ds2, n, cudaMemcpyHostToDevice));
}
}  // namespace

extern "C" {

const char* tlrg_version(void) { return "tlrg 0.1 (sm_100a, FP64 DMMA)"; }

void* tlrg_host_alloc(uint64_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocDefault) != cudaSuccess) return nullptr;
  return p;
}
void tlrg_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

void tlrg_profiler(int on) {
  if (on) cudaProfilerStart();
  else cudaProfilerStop();
}

void tlrg_default_ara_config(tlrg_ara_config* c) {
  c->block_samples = 32;
  c->eps = 1e-6;
  c->max_rank = 0;
  c->window = 0;
  c->safety = 10.0;
  c->recompress = 1;
  c->seed = 0;
}
void tlrg_default_workspace(tlrg_workspace* w) {
  w->parallel_buffers = 64;
  w->dense_buffers = 20;
  w->subset_capacity = 0;
}
void tlrg_default_factor_options(tlrg_factor_options* o) {
  o->schur_compensation = 1;
  o->diag_shift = 0.0;
  o->pivot_norm = 0;
  o->pivot_power_iters = 50;
}

int tlrg_create(int device, tlrg_ctx* out, tlrg_status* st) {
  return guarded(st, [&] {
    int n = 0;
    TLRG_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) config_error("tlrg_create: no such CUDA device");
    TLRG_CUDA(cudaSetDevice(device));
    auto* c = new tlrg_ctx_s;
    c->c.device = device;
    TLRG_CUDA(cudaStreamCreateWithFlags(&c->c.st, cudaStreamNonBlocking));
    TLRG_CUDA(cudaStreamCreateWithFlags(&c->c.st2, cudaStreamNonBlocking));
    {
      // the diagonal path's few-CTA kernels run beside the column's one-CTA-per-
      // tile ARA: high priority lets them take SMs ahead of the ARA's second wave
      int lo = 0, hi = 0;
      TLRG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      const char* pe = std::getenv("TLRG_SD_PRIO");
      const bool prio = !(pe && pe[0] == '0');
      TLRG_CUDA(cudaStreamCreateWithPriority(&c->c.sd, cudaStreamNonBlocking, prio ? hi : lo));
    }
    c->c.st_main = c->c.st;
    ctx_register(&c->c, true);
    {
      // stream-ordered allocations for matrices / panels: keep freed blocks in
      // the pool (no synchronous cudaFree in the factorization loop)
      cudaMemPool_t pool;
      TLRG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
      uint64_t thr = ~0ULL;
      TLRG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    }
    c->c.desc.reserve(16 << 20);
    // one-time kernel attribute setup (never inside a graph capture)
    panel_mgs(nullptr, 0, 0, 0, 1, 1, c->c.st);
    jacobi_svd(nullptr, 0, 1, c->c.st);
    *out = c;
  });
}
void tlrg_destroy(tlrg_ctx c) { delete c; }

int tlrg_comm_attach_nccl(tlrg_ctx ctx, int32_t rank, int32_t world, const uint8_t* id,
                          tlrg_status* st) {
  return guarded(st, [&] {
    if (world < 1 || rank < 0 || rank >= world) config_error("tlrg_comm_attach_nccl: bad rank/world");
    TLRG_CUDA(cudaSetDevice(ctx->c.device));
    ctx->c.comm = world > 1 ? make_nccl_comm(rank, world, id) : nullptr;
  });
}
int tlrg_comm_attach_local(tlrg_ctx* ctxs, int32_t world, tlrg_status* st) {
  return guarded(st, [&] {
    if (world < 1) config_error("tlrg_comm_attach_local: bad world");
    auto comms = make_local_comms(world);
    for (int r = 0; r < world; ++r) ctxs[r]->c.comm = world > 1 ? comms[r] : nullptr;
  });
}
void tlrg_comm_detach(tlrg_ctx ctx) { ctx->c.comm.reset(); }

int tlrg_matrix_upload(tlrg_ctx ctx, int64_t n, int32_t b, double eps, const double* diag,
                       const int32_t* ranks, const double* U, const double* V, tlrg_matrix* out,
                       tlrg_status* st) {
  return guarded(st, [&] {
    auto* h = new tlrg_matrix_s;
    h->m = upload(ctx->c, n, b, eps, diag, ranks, U, V);
    *out = h;
  });
}
int tlrg_matrix_info(tlrg_matrix m, int64_t* n, int32_t* b, int32_t* nb, double* eps) {
  if (n) *n = m->m->n;
  if (b) *b = m->m->b;
  if (nb) *nb = m->m->nb;
  if (eps) *eps = m->m->eps;
  return 0;
}
int tlrg_matrix_ranks(tlrg_matrix m, int32_t* r) {
  std::memcpy(r, m->m->rank.data(), sizeof(int) * m->m->rank.size());
  return 0;
}
int tlrg_matrix_download(tlrg_matrix m, double* diag, double* U, double* V, tlrg_status* st) {
  return guarded(st, [&] { download(*m->m, diag, U, V); });
}
int tlrg_matrix_copy(tlrg_matrix m, tlrg_matrix* out, tlrg_status* st) {
  return guarded(st, [&] {
    auto* h = new tlrg_matrix_s;
    h->m = clone(*m->m->ctx, *m->m);
    *out = h;
  });
}
void tlrg_matrix_free(tlrg_matrix m) {
  if (m && !m->borrowed) delete m;
}
int tlrg_memory_report(tlrg_matrix h, uint64_t* out3) {
  const Matrix& M = *h->m;
  uint64_t dense = 0, lr = 0;
  for (int k = 0; k < M.nb; ++k) dense += (uint64_t)M.rows(k) * M.rows(k) * 8;
  for (int i = 1; i < M.nb; ++i)
    for (int j = 0; j < i; ++j)
      lr += (uint64_t)(M.rows(i) + M.rows(j)) * M.rank[tri_index(i, j)] * 8;
  out3[0] = dense + lr;
  out3[1] = dense;
  out3[2] = lr;
  return 0;
}

int tlrg_write_tlr(tlrg_matrix h, const char* path, tlrg_status* st) {
  return guarded(st, [&] {
    const Matrix& M = *h->m;
    std::ofstream f(path, std::ios::binary);
    if (!f) data_error(std::string("write_tlr: cannot open ") + path);
    uint32_t version = 1, b = M.b;
    uint64_t n = M.n;
    f.write("TLRM", 4);
    f.write((const char*)&version, 4);
    f.write((const char*)&n, 8);
    f.write((const char*)&b, 4);
    f.write((const char*)&M.eps, 8);
    std::vector<double> buf;
    for (int k = 0; k < M.nb; ++k) {
      uint32_t r = M.rows(k);
      buf.resize((size_t)r * r);
      TLRG_CUDA(cudaMemcpy(buf.data(), M.diag + (size_t)k * M.b * M.b, 8 * buf.size(),
                           cudaMemcpyDeviceToHost));
      f.write((const char*)&r, 4);
      f.write((const char*)&r, 4);
      f.write((const char*)buf.data(), 8 * buf.size());
    }
    uint64_t count = M.rank.size();
    f.write((const char*)&count, 8);
    for (int i = 1; i < M.nb; ++i)
      for (int j = 0; j < i; ++j) {
        long long t = tri_index(i, j);
        uint32_t ii = i, jj = j, r = M.rank[t];
        f.write((const char*)&ii, 4);
        f.write((const char*)&jj, 4);
        f.write((const char*)&r, 4);
        if (r) {
          buf.resize((size_t)M.rows(i) * r);
          TLRG_CUDA(cudaMemcpy(buf.data(), M.U[t], 8 * buf.size(), cudaMemcpyDeviceToHost));
          f.write((const char*)buf.data(), 8 * buf.size());
          buf.resize((size_t)M.rows(j) * r);
          TLRG_CUDA(cudaMemcpy(buf.data(), M.V[t], 8 * buf.size(), cudaMemcpyDeviceToHost));
          f.write((const char*)buf.data(), 8 * buf.size());
        }
      }
    if (!f) data_error("write_tlr: write failed");
  });
}

namespace {
// read_tlr (tlr_matrix.cpp:301-340) from an open stream; leaves it positioned
// after the TLRM payload (read_factor continues with the trailer there)
std::unique_ptr<Matrix> read_tlr_stream(Ctx& C, std::ifstream& f) {
  char magic[4];
  uint32_t version = 0, b = 0;
  uint64_t n = 0;
  double eps = 0;
  f.read(magic, 4);
  f.read((char*)&version, 4);
  f.read((char*)&n, 8);
  f.read((char*)&b, 4);
  f.read((char*)&eps, 8);
  if (!f || std::memcmp(magic, "TLRM", 4) != 0) data_error("read_tlr: bad magic");
  if (version != 1) data_error("read_tlr: unsupported version");
  if (n < 1 || b < 1 || b > n) config_error("TlrMatrix: bad dimensions");
  int nb = (int)((n + b - 1) / b);
  auto rows = [&](int i) { return (int)std::min<int64_t>(b, (int64_t)n - (int64_t)i * b); };
  std::vector<double> diag;
  for (int k = 0; k < nb; ++k) {
    uint32_t r = 0, c = 0;
    f.read((char*)&r, 4);
    f.read((char*)&c, 4);
    if (!f) data_error("read_tlr: truncated tile header");
    if ((int)r != rows(k) || (int)c != rows(k)) data_error("read_tlr: diagonal tile shape mismatch");
    size_t o = diag.size();
    diag.resize(o + (size_t)r * c);
    f.read((char*)(diag.data() + o), 8 * (size_t)r * c);
    if (!f) data_error("read_tlr: truncated tile payload");
  }
  uint64_t count = 0;
  f.read((char*)&count, 8);
  if (!f || count != (uint64_t)nb * (nb - 1) / 2) data_error("read_tlr: bad tile count");
  std::vector<int32_t> ranks(count, 0);
  std::vector<std::vector<double>> Us(count), Vs(count);
  for (uint64_t q = 0; q < count; ++q) {
    uint32_t i = 0, j = 0, r = 0;
    f.read((char*)&i, 4);
    f.read((char*)&j, 4);
    f.read((char*)&r, 4);
    if (!f || i >= (uint32_t)nb || j >= i) data_error("read_tlr: bad tile index");
    long long t = tri_index(i, j);
    ranks[t] = r;
    Us[t].resize((size_t)rows(i) * r);
    Vs[t].resize((size_t)rows(j) * r);
    f.read((char*)Us[t].data(), 8 * Us[t].size());
    f.read((char*)Vs[t].data(), 8 * Vs[t].size());
    if (!f) data_error("read_tlr: truncated tile payload");
  }
  std::vector<double> U, V;
  for (uint64_t t = 0; t < count; ++t) {
    U.insert(U.end(), Us[t].begin(), Us[t].end());
    V.insert(V.end(), Vs[t].begin(), Vs[t].end());
  }
  return upload(C, (int64_t)n, (int)b, eps, diag.data(), ranks.data(), U.data(), V.data());
}
}  // namespace

int tlrg_read_tlr(tlrg_ctx ctx, const char* path, tlrg_matrix* out, tlrg_status* st) {
  return guarded(st, [&] {
    std::ifstream f(path, std::ios::binary);
    if (!f) data_error(std::string("read_tlr: cannot open ") + path);
    auto* h = new tlrg_matrix_s;
    h->m = read_tlr_stream(ctx->c, f);
    *out = h;
  });
}

int tlrg_factorize(tlrg_ctx ctx, tlrg_matrix A, int32_t mode, const tlrg_ara_config* cfg,
                   const tlrg_workspace* ws, const tlrg_factor_options* opts, tlrg_factor* out,
                   tlrg_status* st) {
  return guarded(st, [&] {
    if (!A || !A->m) config_error("tlrg_factorize: null matrix handle");
    // take A first (by-value TlrMatrix in the reference: consumed even when the
    // call throws).  A borrowed view (tlrg_factor_L) still belongs to its
    // factor: it is deep-copied, like the reference copying F.L into the
    // by-value argument.
    std::unique_ptr<Matrix> M;
    if (A->borrowed) {
      M = clone(*A->m->ctx, *A->m);
    } else {
      M = std::move(A->m);
      delete A;
    }
    if (mode < 0 || mode > 2)
      config_error("tlrg_factorize: mode must be 0 (Chol), 1 (LDLT) or 2 (pivoted Chol)");
    FactorOpts fo;
    if (opts) {
      fo.schur = opts->schur_compensation != 0;
      fo.shift = opts->diag_shift;
      fo.pivot_norm = opts->pivot_norm;
      fo.pivot_power_iters = opts->pivot_power_iters;
    }
    auto F = factorize(ctx->c, std::move(M), mode, to_cfg(cfg), ws ? ws->parallel_buffers : 64, fo);
    auto* h = new tlrg_factor_s;
    h->f = std::move(F);
    h->ctx = &ctx->c;
    h->Lview.m.reset(h->f->L.get());
    h->Lview.borrowed = true;
    *out = h;
  });
}
void tlrg_factor_free(tlrg_factor f) {
  if (!f) return;
  (void)f->Lview.m.release();
  delete f;
}
tlrg_matrix tlrg_factor_L(tlrg_factor f) { return &f->Lview; }
int tlrg_factor_mode(tlrg_factor f) { return f->f->mode; }
int tlrg_factor_stats(tlrg_factor f, tlrg_stats* o, int32_t* ara_rounds, double* pivot_trace) {
  const Stats& S = f->f->stats;
  if (o) {
    o->t_sampling = S.t_sampling;
    o->t_projection = S.t_projection;
    o->t_reduction = S.t_reduction;
    o->t_dense = S.t_dense;
    o->t_orthog = S.t_orthog;
    o->t_misc = S.t_misc;
    o->t_pivot_select = S.t_pivot_select;
    o->wall = S.wall;
    o->compensation_frob = S.compensation_frob;
    o->modified_diagonals = S.modified_diagonals;
    o->tile_rounds_resident = S.tile_rounds_resident;
    o->t_recompress = S.t_recompress;
    o->t_compensation = S.t_compensation;
    o->flops_exec = S.flops_exec;
    o->flops_gemm_ref = S.flops_ref;
    o->kernel_launches = S.launches;
    o->t_device = S.t_device;
    o->kt_gemm_seconds = S.kt_gemm_seconds;
    o->kt_gemm_flops = S.kt_gemm_flops;
    o->kt_gemm_launches = S.kt_gemm_launches;
    o->t_ara_kernel = S.t_fused;
    o->flops_ara_kernel = S.flops_fused;
    o->ara_kernel_launches = S.fused_launches;
  }
  int nb = f->f->L->nb;
  if (ara_rounds)
    for (int k = 0; k < nb; ++k) ara_rounds[k] = S.ara_rounds[k];
  if (pivot_trace)
    for (int k = 0; k < nb; ++k) pivot_trace[k] = S.pivot_trace[k];
  return 0;
}
int tlrg_factor_dblock(tlrg_factor f, int32_t k, double* d, double* e, uint8_t* s2, int32_t* perm) {
  const Factor& F = *f->f;
  if (F.mode != 1) return 2;  // ConfigError: no D blocks in a Cholesky factor
  if (k < 0 || k >= F.L->nb) return 2;
  int b = F.L->b, n = F.L->rows(k);
  size_t o = (size_t)k * b;
  cudaError_t e1 = cudaMemcpy(d, F.D.d + o, 8 * n, cudaMemcpyDeviceToHost);
  cudaError_t e2 = n > 1 ? cudaMemcpy(e, F.D.e + o, 8 * (n - 1), cudaMemcpyDeviceToHost) : cudaSuccess;
  cudaError_t e3 = cudaMemcpy(s2, F.D.s2 + o, n, cudaMemcpyDeviceToHost);
  cudaError_t e4 = cudaMemcpy(perm, F.D.perm + o, 4 * n, cudaMemcpyDeviceToHost);
  return (e1 || e2 || e3 || e4) ? 1 : 0;
}
int tlrg_write_factor(tlrg_factor f, const char* path, tlrg_status* st) {
  int rc = tlrg_write_tlr(&f->Lview, path, st);
  if (rc) return rc;
  return guarded(st, [&] {
    const Factor& F = *f->f;
    std::ofstream o(path, std::ios::binary | std::ios::app);
    if (!o) data_error("write_factor: cannot append");
    uint8_t mode = (uint8_t)F.mode;  // 0 Cholesky, 1 LDLT, 2 pivoted (factor.cpp:311-313)
    o.write((const char*)&mode, 1);
    o.write((const char*)&F.eps, 8);
    if (F.mode == 1) {
      for (int k = 0; k < F.L->nb; ++k) {
        uint32_t n = F.L->rows(k);
        std::vector<double> d(n), e(n > 1 ? n - 1 : 0);
        std::vector<uint8_t> s2(n);
        std::vector<int32_t> p(n);
        tlrg_factor_dblock(f, k, d.data(), e.data(), s2.data(), p.data());
        o.write((const char*)&n, 4);
        o.write((const char*)d.data(), 8 * n);
        if (n > 1) o.write((const char*)e.data(), 8 * (n - 1));
        o.write((const char*)s2.data(), n);
        std::vector<uint32_t> pu(p.begin(), p.end());
        o.write((const char*)pu.data(), 4 * n);
      }
    }
    if (F.mode == 2) {
      std::vector<uint32_t> p(F.perm.begin(), F.perm.end());
      o.write((const char*)p.data(), 4 * p.size());
    }
    if (!o) data_error("write_factor: write failed");
  });
}

// read_factor (factor.cpp:340-395): TLRM payload, then mode, eps, D blocks with
// intra-tile permutations (LDL^T) or the tile permutation (pivoted)
int tlrg_read_factor(tlrg_ctx ctx, const char* path, tlrg_factor* out, tlrg_status* st) {
  return guarded(st, [&] {
    std::ifstream f(path, std::ios::binary);
    if (!f) data_error(std::string("read_factor: cannot open ") + path);
    Ctx& C = ctx->c;
    auto F = std::make_unique<Factor>();
    F->L = read_tlr_stream(C, f);
    const int nb = F->L->nb, b = F->L->b;
    uint8_t mode = 0;
    f.read((char*)&mode, 1);
    f.read((char*)&F->eps, 8);
    if (!f) data_error("read_factor: missing trailer");
    F->mode = mode == 0 ? 0 : mode == 1 ? 1 : 2;
    F->stats.ara_rounds.assign(nb, 0);
    F->stats.pivot_trace.assign(nb, 0.0);
    if (F->mode == 1) {
      std::vector<double> d((size_t)nb * b, 0.0), e((size_t)nb * b, 0.0);
      std::vector<uint8_t> s2((size_t)nb * b, 0);
      std::vector<int32_t> pm((size_t)nb * b, 0);
      for (int k = 0; k < nb; ++k) {
        uint32_t n = 0;
        f.read((char*)&n, 4);
        if (!f || (int)n != F->L->rows(k)) data_error("read_factor: bad D block size");
        const size_t o = (size_t)k * b;
        f.read((char*)(d.data() + o), 8 * n);
        if (n > 1) f.read((char*)(e.data() + o), 8 * (n - 1));
        f.read((char*)(s2.data() + o), n);
        std::vector<uint32_t> p(n);
        f.read((char*)p.data(), 4 * n);
        if (!f) data_error("read_factor: truncated D block");
        for (uint32_t i = 0; i < n; ++i) pm[o + i] = (int32_t)p[i];
      }
      TLRG_CUDA(cudaMalloc(&F->D.d, sizeof(double) * nb * b));
      TLRG_CUDA(cudaMalloc(&F->D.e, sizeof(double) * nb * b));
      TLRG_CUDA(cudaMalloc(&F->D.s2, (size_t)nb * b));
      TLRG_CUDA(cudaMalloc(&F->D.perm, sizeof(int) * nb * b));
      TLRG_CUDA(cudaMemcpy(F->D.d, d.data(), 8 * d.size(), cudaMemcpyHostToDevice));
      TLRG_CUDA(cudaMemcpy(F->D.e, e.data(), 8 * e.size(), cudaMemcpyHostToDevice));
      TLRG_CUDA(cudaMemcpy(F->D.s2, s2.data(), s2.size(), cudaMemcpyHostToDevice));
      TLRG_CUDA(cudaMemcpy(F->D.perm, pm.data(), 4 * pm.size(), cudaMemcpyHostToDevice));
    }
    if (F->mode == 2) {
      std::vector<uint32_t> p(nb);
      f.read((char*)p.data(), 4 * nb);
      if (!f) data_error("read_factor: truncated permutation");
      F->perm.assign(p.begin(), p.end());
      TLRG_CUDA(cudaMalloc(&F->d_perm, sizeof(int) * nb));
      TLRG_CUDA(cudaMemcpy(F->d_perm, F->perm.data(), sizeof(int) * nb, cudaMemcpyHostToDevice));
    }
    auto* h = new tlrg_factor_s;
    h->f = std::move(F);
    h->ctx = &C;
    h->Lview.m.reset(h->f->L.get());
    h->Lview.borrowed = true;
    *out = h;
  });
}

int tlrg_factor_perm(tlrg_factor f, int32_t* perm) {
  const Factor& F = *f->f;
  if (F.perm.empty()) return 2;
  for (size_t i = 0; i < F.perm.size(); ++i) perm[i] = F.perm[i];
  return 0;
}

int tlrg_factor_solve(tlrg_factor f, const double* b, double* x, tlrg_status* st) {
  return guarded(st, [&] {
    Ctx& C = *f->ctx;
    int64_t n = f->f->L->n;
    double* d = C.buf<double>("solve_x", (size_t)n);
    TLRG_CUDA(cudaMemcpyAsync(d, b, 8 * n, cudaMemcpyHostToDevice, C.st));
    factor_solve_device(C, *f->f, d);
    TLRG_CUDA(cudaMemcpyAsync(x, d, 8 * n, cudaMemcpyDeviceToHost, C.st));
    C.sync();
  });
}
int tlrg_factor_apply(tlrg_factor f, const double* x, double* y, tlrg_status* st) {
  return guarded(st, [&] {
    Ctx& C = *f->ctx;
    int64_t n = f->f->L->n;
    double* dx = C.buf<double>("apply_x", (size_t)n);
    double* dy = C.buf<double>("apply_y", (size_t)n);
    TLRG_CUDA(cudaMemcpyAsync(dx, x, 8 * n, cudaMemcpyHostToDevice, C.st));
    factor_apply_device(C, *f->f, dx, dy);
    TLRG_CUDA(cudaMemcpyAsync(y, dy, 8 * n, cudaMemcpyDeviceToHost, C.st));
    C.sync();
  });
}
int tlrg_tlr_matvec(tlrg_matrix A, const double* x, double* y, tlrg_status* st) {
  return guarded(st, [&] {
    Ctx& C = *A->m->ctx;
    int64_t n = A->m->n;
    double* dx = C.buf<double>("mv_x", (size_t)n);
    double* dy = C.buf<double>("mv_y", (size_t)n);
    TLRG_CUDA(cudaMemcpyAsync(dx, x, 8 * n, cudaMemcpyHostToDevice, C.st));
    matvec_device(C, *A->m, dx, dy);
    TLRG_CUDA(cudaMemcpyAsync(y, dy, 8 * n, cudaMemcpyDeviceToHost, C.st));
    C.sync();
  });
}

static double power_iter(Ctx& C, int64_t n, uint64_t seed0, int iters,
                         const std::function<void(const double*, double*)>& op) {
  double* v = C.buf<double>("pw_v", (size_t)n);
  double* w = C.buf<double>("pw_w", (size_t)n);
  RngState* rs = C.buf<RngState>("pw_rng", 1);
  std::vector<uint64_t> s1{seed0};
  rng_seed(rs, C.push(s1), 1, C.st);
  rng_draw(rs, nullptr, 1, v, n, n, C.st);
  double nv = std::sqrt(dot_device(C, v, v, n));
  auto scale = [&](double* p, double s) { axpby_device(C, 0.0, p, s, p, n); };
  scale(v, 1.0 / nv);
  double lambda = 0.0;
  for (int t = 0; t < iters; ++t) {
    op(v, w);
    double nw = std::sqrt(dot_device(C, w, w, n));
    lambda = std::fabs(dot_device(C, v, w, n));
    if (nw < 1e-300) return nw;
    scale(w, 1.0 / nw);
    std::swap(v, w);
  }
  return lambda;
}

int tlrg_estimate_2norm_diff(tlrg_matrix A, tlrg_factor f, int32_t iters, uint64_t seed,
                             double* out, tlrg_status* st) {
  return guarded(st, [&] {
    if (iters < 1) config_error("estimate_2norm_diff: iters must be >= 1");
    Ctx& C = *f->ctx;
    int64_t n = A->m->n;
    double* t = C.buf<double>("pw_t", (size_t)n);
    *out = power_iter(C, n, mix64(seed ^ 0x2fULL), iters, [&](const double* v, double* w) {
      difference_apply_device(C, *A->m, *f->f, v, w, t);
    });
  });
}
int tlrg_frob_norm(tlrg_matrix A, double* out, tlrg_status* st) {
  return guarded(st, [&] { *out = frob_norm_device(*A->m->ctx, *A->m); });
}
int tlrg_estimate_frob_diff(tlrg_matrix A, tlrg_factor f, int32_t probes, uint64_t seed,
                            double* out, tlrg_status* st) {
  return guarded(st, [&] {
    if (probes < 1) config_error("estimate_frob_diff: probes must be >= 1");
    if (A->m->n != f->f->L->n) config_error("estimate_frob_diff: size mismatch");
    *out = estimate_frob_diff_device(*f->ctx, *A->m, *f->f, probes, seed);
  });
}
int tlrg_estimate_2norm(tlrg_matrix A, int32_t iters, uint64_t seed, double* out, tlrg_status* st) {
  return guarded(st, [&] {
    Ctx& C = *A->m->ctx;
    *out = power_iter(C, A->m->n, mix64(seed ^ 0xa2ULL), iters,
                      [&](const double* v, double* w) { matvec_device(C, *A->m, v, w); });
  });
}

// ------------------------------------------------------------ building blocks
int tlrg_sample_left(tlrg_matrix mh, const double* dd, const double* de, const uint8_t* ds2,
                     int32_t k, int32_t nrows, const int32_t* rows, int32_t pb,
                     const double* omegas, int32_t width, int32_t transpose, double* out,
                     tlrg_status* st) {
  return guarded(st, [&] {
    if (nrows == 0) return;
    if (pb / nrows < 1) config_error("sample_left: workspace smaller than one buffer per tile");
    const Matrix& M = *mh->m;
    Ctx& C = *M.ctx;
    DUpload du;
    upload_d(du, M, dd, de, ds2);
    ColumnSetup cs;
    column_setup(C, M, k, du.D, cs);
    const int rk = M.rows(k), K = cs.K, b = M.b;
    std::vector<int> tg(rows, rows + nrows);
    double* H = K ? C.buf<double>("sl_H", (size_t)nrows * b * K) : nullptr;
    column_H(C, M, cs, tg, H, (long long)b * K);
    // inputs
    std::vector<long long> ioff(nrows), ooff(nrows);
    long long itot = 0, otot = 0;
    for (int t = 0; t < nrows; ++t) {
      int ri = M.rows(rows[t]);
      int in_rows = transpose ? ri : rk, out_rows = transpose ? rk : ri;
      ioff[t] = itot;
      ooff[t] = otot;
      itot += (long long)in_rows * width;
      otot += (long long)out_rows * width;
    }
    double* X = C.buf<double>("sl_X", (size_t)itot + 1);
    double* Yo = C.buf<double>("sl_Y", (size_t)otot + 1);
    TLRG_CUDA(cudaMemcpyAsync(X, omegas, 8 * itot, cudaMemcpyHostToDevice, C.st));
    int kAmax = 0;
    for (int t = 0; t < nrows; ++t) kAmax = std::max(kAmax, M.rank[M.t(rows[t], k)]);
    double* Z = C.buf<double>("sl_Z", (size_t)nrows * (kAmax + K) * width + 1);
    long long zs = (long long)(kAmax + K) * width;
    std::vector<GemmProblem> p1, p2, p3;
    for (int t = 0; t < nrows; ++t) {
      int i = rows[t], ri = M.rows(i), kA = M.rank[M.t(i, k)];
      long long q = M.t(i, k);
      double* Zt = Z + t * zs;  // (kA + K) x width, ld kA+K
      int ld = std::max(kA + K, 1);
      const double* Xt = X + ioff[t];
      if (!transpose) {
        // Z1 = VA^T X ; Z2 = Ucat^T X ; Y = UA Z1 - H Z2
        if (kA) p1.push_back({M.V[q], Xt, Zt, rk, rk, ld, kA, width, rk, 1, 0, 1.0, 0.0, 0, 0});
        if (K) p1.push_back({cs.Ucat, Xt, Zt + kA, rk, rk, ld, K, width, rk, 1, 0, 1.0, 0.0, 0, 0});
        p2.push_back({kA ? M.U[q] : Yo, kA ? Zt : Yo, Yo + ooff[t], ri, ld, ri, ri, width, kA, 0, 0,
                      1.0, 0.0, 0, 0});
        if (K)
          p3.push_back({H + (long long)t * b * K, Zt + kA, Yo + ooff[t], ri, ld, ri, ri, width, K, 0,
                        0, -1.0, 1.0, 0, 0});
      } else {
        // Z1 = UA^T X ; Z2 = H^T X ; B = VA Z1 - Ucat Z2
        if (kA) p1.push_back({M.U[q], Xt, Zt, ri, ri, ld, kA, width, ri, 1, 0, 1.0, 0.0, 0, 0});
        if (K)
          p1.push_back({H + (long long)t * b * K, Xt, Zt + kA, ri, ri, ld, K, width, ri, 1, 0, 1.0,
                        0.0, 0, 0});
        p2.push_back({kA ? M.V[q] : Yo, kA ? Zt : Yo, Yo + ooff[t], rk, ld, rk, rk, width, kA, 0, 0,
                      1.0, 0.0, 0, 0});
        if (K)
          p3.push_back({cs.Ucat, Zt + kA, Yo + ooff[t], rk, ld, rk, rk, width, K, 0, 0, -1.0, 1.0, 0,
                        0});
      }
    }
    C.gemm(p1);
    C.gemm(p2);
    C.gemm(p3);
    TLRG_CUDA(cudaMemcpyAsync(out, Yo, 8 * otot, cudaMemcpyDeviceToHost, C.st));
    C.sync();
  });
}

int tlrg_chol_ara_update(tlrg_matrix mh, const double* dd, const double* de, const uint8_t* ds2,
                         int32_t k, const tlrg_ara_config* cfg, const tlrg_workspace* ws,
                         tlrg_ara* out, tlrg_status* st) {
  (void)ws;
  return guarded(st, [&] {
    const Matrix& M = *mh->m;
    Ctx& C = *M.ctx;
    AraCfg c = to_cfg(cfg);
    if (!(c.eps > 0)) config_error("chol_ara_update: eps must be positive");
    DUpload du;
    upload_d(du, M, dd, de, ds2);
    cudaEvent_t ev0, ev1;
    TLRG_CUDA(cudaEventCreate(&ev0));
    TLRG_CUDA(cudaEventCreate(&ev1));
    TLRG_CUDA(cudaEventRecord(ev0, C.st));
    ColumnSetup cs;
    column_setup(C, M, k, du.D, cs);
    auto store = std::make_shared<Store>();
    store->st = C.st_main;
    store->owner = &C;
    ColumnStats cst;
    auto res = column_ara(C, M, k, cs, c, *store, cst);
    TLRG_CUDA(cudaEventRecord(ev1, C.st));
    C.sync();
    column_stats_resolve(cst);
    auto* a = new tlrg_ara_s;
    {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev0, ev1);
      a->t_device = ms * 1e-3;
      cudaEventDestroy(ev0);
      cudaEventDestroy(ev1);
      a->t_fused = cst.t_fused;
      a->flops_fused = cst.flops_fused;
      a->flops_ref = cst.flops_ref;
      a->tile_rounds = cst.tile_rounds;
    }
    int rk = M.rows(k);
    for (auto& r : res) {
      a->i.push_back(r.i);
      a->rank.push_back(r.rank);
      a->conv.push_back(r.converged);
      a->rounds.push_back(r.rounds);
      std::vector<double> Q((size_t)M.rows(r.i) * r.rank), B((size_t)rk * r.rank);
      if (r.rank) {
        TLRG_CUDA(cudaMemcpy(Q.data(), r.U, 8 * Q.size(), cudaMemcpyDeviceToHost));
        TLRG_CUDA(cudaMemcpy(B.data(), r.V, 8 * B.size(), cudaMemcpyDeviceToHost));
      }
      a->Q.push_back(std::move(Q));
      a->B.push_back(std::move(B));
    }
    *out = a;
  });
}
int tlrg_ara_count(tlrg_ara a) { return (int)a->i.size(); }
int tlrg_ara_tile(tlrg_ara a, int32_t t, int32_t* info, double* Q, double* B) {
  info[0] = a->i[t];
  info[1] = a->rank[t];
  info[2] = a->conv[t];
  info[3] = a->rounds[t];
  if (Q) std::memcpy(Q, a->Q[t].data(), 8 * a->Q[t].size());
  if (B) std::memcpy(B, a->B[t].data(), 8 * a->B[t].size());
  return 0;
}
void tlrg_ara_free(tlrg_ara a) { delete a; }
void tlrg_ara_stats(tlrg_ara a, double* out5) {
  out5[0] = a->t_device;  // CUDA-event time of the column's ARA (setup .. panel written)
  out5[1] = (double)a->tile_rounds;
  out5[2] = a->flops_ref;    // reference-formulation sampling + projection flops
  out5[3] = a->t_fused;      // fused-kernel event time (0 on the graph path)
  out5[4] = a->flops_fused;  // algorithmic flops executed in the fused kernel
}

int tlrg_rng_gaussians(tlrg_ctx ctx, uint64_t seed, int64_t n, double* out, tlrg_status* st) {
  return guarded(st, [&] {
    Ctx& C = ctx->c;
    // through the stream generator used by the factorization
    GaussStreams G;
    G.cap = (n + 2) & ~1LL;
    G.st = C.buf<RngState>("t_rng", 1);
    G.buf = C.buf<double>("t_rng_out", (size_t)G.cap + 2);
    long long* gl = C.buf<long long>("t_rng_cur", 2);
    G.avail = gl;
    G.cursor = gl + 1;
    TLRG_CUDA(cudaMemsetAsync(gl, 0, sizeof(long long) * 2, C.st));
    std::vector<uint64_t> s1{seed};
    rng_seed(G.st, C.push(s1), 1, C.st);
    std::vector<int> slot{0};
    std::vector<long long> want{G.cap};
    gauss_generate(G, C.push(slot), C.push(want), 1, C.st);
    TLRG_CUDA(cudaMemcpyAsync(out, G.buf, 8 * n, cudaMemcpyDeviceToHost, C.st));
    C.sync();
  });
}

int tlrg_orthog(tlrg_ctx ctx, const double* Q, int32_t rows, int32_t q, double* Y, int32_t k,
                uint64_t seed, double* R, double* col_norms, double* new_mass, double* next_draw,
                tlrg_status* st) {
  return guarded(st, [&] {
    Ctx& C = ctx->c;
    if (k == 0) return;
    double* dQ = C.buf<double>("o_Q", (size_t)rows * q + 1);
    double* dY = C.buf<double>("o_Y", (size_t)rows * k);
    double* dC = C.buf<double>("o_C", (size_t)q * k + 1);
    double* dR = C.buf<double>("o_R", (size_t)k * k);
    double* dRp = C.buf<double>("o_Rp", (size_t)2 * k * k);
    double* vec = C.buf<double>("o_vec", (size_t)4 * k);
    uint8_t* df = C.buf<uint8_t>("o_df", (size_t)k);
    GaussStreams G;
    G.cap = (2LL * k * rows + 4) & ~1LL;
    G.st = C.buf<RngState>("o_rng", 1);
    G.buf = C.buf<double>("o_gbuf", (size_t)G.cap);
    long long* gl = C.buf<long long>("o_gcur", 2);
    G.avail = gl;
    G.cursor = gl + 1;
    TLRG_CUDA(cudaMemsetAsync(gl, 0, sizeof(long long) * 2, C.st));
    std::vector<uint64_t> s1{seed};
    rng_seed(G.st, C.push(s1), 1, C.st);
    std::vector<int> slot{0};
    std::vector<long long> want{G.cap};
    gauss_generate(G, C.push(slot), C.push(want), 1, C.st);
    if (q) TLRG_CUDA(cudaMemcpyAsync(dQ, Q, 8 * (size_t)rows * q, cudaMemcpyHostToDevice, C.st));
    TLRG_CUDA(cudaMemcpyAsync(dY, Y, 8 * (size_t)rows * k, cudaMemcpyHostToDevice, C.st));
    std::vector<PanelTask> t(1);
    PanelTask& P = t[0];
    P = PanelTask{};
    P.Y = dY; P.Q = q ? dQ : nullptr; P.R = dR; P.Rp = dRp; P.tiny = vec;
    P.col_norms = vec + k; P.new_mass = vec + 2 * k; P.deficient = df;
    P.gbuf = G.buf; P.gcursor = G.cursor; P.gcap = G.cap;
    P.rep = C.buf<double>("o_rep", (size_t)rows * k);
    P.repC = C.buf<double>("o_repC", (size_t)(q + 1) * k);
    P.rows = rows; P.width = k; P.q = q;
    PanelTask* d = C.push(t);
    panel_tau(d, 1, C.st);
    for (int sweep = 0; sweep < 2; ++sweep) {
      if (q) {
        std::vector<GemmProblem> a(1), b(1);
        a[0] = {dQ, dY, dC, rows, rows, q, q, k, rows, 1, 0, 1.0, 0.0, 0, 0};
        b[0] = {dQ, dC, dY, rows, q, rows, rows, k, q, 0, 0, -1.0, 1.0, 0, 0};
        C.gemm(a);
        C.gemm(b);
      }
      panel_mgs(d, 1, sweep, sweep == 1, k, rows, C.st);
    }
    long long cur = 0;
    TLRG_CUDA(cudaMemcpyAsync(Y, dY, 8 * (size_t)rows * k, cudaMemcpyDeviceToHost, C.st));
    TLRG_CUDA(cudaMemcpyAsync(R, dR, 8 * (size_t)k * k, cudaMemcpyDeviceToHost, C.st));
    TLRG_CUDA(cudaMemcpyAsync(col_norms, vec + k, 8 * k, cudaMemcpyDeviceToHost, C.st));
    TLRG_CUDA(cudaMemcpyAsync(new_mass, vec + 2 * k, 8 * k, cudaMemcpyDeviceToHost, C.st));
    TLRG_CUDA(cudaMemcpyAsync(&cur, G.cursor, 8, cudaMemcpyDeviceToHost, C.st));
    C.sync();
    if (next_draw) TLRG_CUDA(cudaMemcpy(next_draw, G.buf + cur, 8, cudaMemcpyDeviceToHost));
  });
}

int tlrg_potrf(tlrg_ctx ctx, const double* A, int32_t n, double* L, int32_t* fail,
               tlrg_status* st) {
  return guarded(st, [&] {
    Ctx& C = ctx->c;
    double* d = C.buf<double>("t_potrf", (size_t)n * n);
    TLRG_CUDA(cudaMemcpy(d, A, 8 * (size_t)n * n, cudaMemcpyHostToDevice));
    int* info = C.buf<int>("potrf_info", 1);
    tlrg::potrf_impl(d, n, info, C.desc, C.st);
    TLRG_CUDA(cudaMemcpyAsync(fail, info, 4, cudaMemcpyDeviceToHost, C.st));
    TLRG_CUDA(cudaMemcpyAsync(L, d, 8 * (size_t)n * n, cudaMemcpyDeviceToHost, C.st));
    C.sync();
  });
}

int tlrg_dense_ldl(tlrg_ctx ctx, const double* A, int32_t n, double* L, double* d, double* e,
                   uint8_t* s2, int32_t* perm, int32_t* info, tlrg_status* st) {
  return guarded(st, [&] {
    Ctx& C = ctx->c;
    double* dA = C.buf<double>("t_ldl", (size_t)n * n);
    double* dd = C.buf<double>("t_ldl_d", (size_t)n);
    double* de = C.buf<double>("t_ldl_e", (size_t)n);
    uint8_t* ds = C.buf<uint8_t>("t_ldl_s", (size_t)n);
    int* dp = C.buf<int>("t_ldl_p", (size_t)n);
    int* di = C.buf<int>("t_ldl_i", 1);
    TLRG_CUDA(cudaMemcpy(dA, A, 8 * (size_t)n * n, cudaMemcpyHostToDevice));
    sytrf_bk(dA, n, dd, de, ds, dp, di, C.st);
    C.sync();
    TLRG_CUDA(cudaMemcpy(L, dA, 8 * (size_t)n * n, cudaMemcpyDeviceToHost));
    TLRG_CUDA(cudaMemcpy(d, dd, 8 * n, cudaMemcpyDeviceToHost));
    if (n > 1) TLRG_CUDA(cudaMemcpy(e, de, 8 * (n - 1), cudaMemcpyDeviceToHost));
    TLRG_CUDA(cudaMemcpy(s2, ds, n, cudaMemcpyDeviceToHost));
    TLRG_CUDA(cudaMemcpy(perm, dp, 4 * n, cudaMemcpyDeviceToHost));
    TLRG_CUDA(cudaMemcpy(info, di, 4, cudaMemcpyDeviceToHost));
  });
}

int tlrg_schur_compensation(tlrg_ctx ctx, const double* Dk, int32_t n, double eps,
                            double* diag_out, double* frob, tlrg_status* st) {
  return guarded(st, [&] {
    Ctx& C = ctx->c;
    double* dD = C.buf<double>("t_sc_D", (size_t)n * n);
    double* corr = C.buf<double>("t_sc_c", (size_t)n);
    double* fr = C.buf<double>("t_sc_f", 1);
    TLRG_CUDA(cudaMemcpy(dD, Dk, 8 * (size_t)n * n, cudaMemcpyHostToDevice));
    int hint = 0;
    schur_compensation_device(C, dD, n, eps, 12345, corr, fr, hint);
    C.sync();
    TLRG_CUDA(cudaMemcpy(diag_out, corr, 8 * n, cudaMemcpyDeviceToHost));
    double f2 = 0;
    TLRG_CUDA(cudaMemcpy(&f2, fr, 8, cudaMemcpyDeviceToHost));
    if (frob) *frob = std::sqrt(f2);
  });
}

int tlrg_jacobi_svd(tlrg_ctx ctx, const double* A, int32_t m, int32_t n, double cut,
                    int32_t force_single, double* US, double* V, double* sig, int32_t* rank,
                    tlrg_status* st) {
  return guarded(st, [&] {
    if (m < 1 || n < 1) config_error("jacobi_svd: empty matrix");
    Ctx& C = ctx->c;
    double* dA = C.buf<double>("t_js_A", (size_t)m * n);
    double* dV = C.buf<double>("t_js_V", (size_t)n * n);
    double* dS = C.buf<double>("t_js_S", (size_t)n);
    double* dW = C.buf<double>("t_js_W", (size_t)n * (m + n));
    int* dR = C.buf<int>("t_js_R", 1);
    TLRG_CUDA(cudaMemcpy(dA, A, 8 * (size_t)m * n, cudaMemcpyHostToDevice));
    SvdTask t{};
    t.A = dA;
    t.V = dV;
    t.sig = dS;
    t.work = dW;
    t.rank_out = dR;
    t.n = n;
    t.m = m;
    t.cut = cut;
    const bool wide = !force_single && n > jacobi_staged_max_n() && n <= 1024 && m <= 1024;
    if (wide) jacobi_svd_wide(C.push(std::vector<SvdTask>{t}), 1, n, C.st, m);
    else jacobi_svd(C.push(std::vector<SvdTask>{t}), 1, n, C.st, m);
    C.sync();
    TLRG_CUDA(cudaMemcpy(US, dA, 8 * (size_t)m * n, cudaMemcpyDeviceToHost));
    TLRG_CUDA(cudaMemcpy(V, dV, 8 * (size_t)n * n, cudaMemcpyDeviceToHost));
    TLRG_CUDA(cudaMemcpy(sig, dS, 8 * (size_t)n, cudaMemcpyDeviceToHost));
    TLRG_CUDA(cudaMemcpy(rank, dR, 4, cudaMemcpyDeviceToHost));
  });
}

int tlrg_gemm(tlrg_ctx ctx, int32_t M, int32_t N, int32_t K, int32_t ta, int32_t tb, double alpha,
              const double* A, const double* B, double beta, double* Cm, tlrg_status* st) {
  return guarded(st, [&] {
    Ctx& C = ctx->c;
    size_t na = (size_t)M * K, nbb = (size_t)K * N, nc = (size_t)M * N;
    double* dA = C.buf<double>("t_gA", na + 1);
    double* dB = C.buf<double>("t_gB", nbb + 1);
    double* dC = C.buf<double>("t_gC", nc + 1);
    TLRG_CUDA(cudaMemcpy(dA, A, 8 * na, cudaMemcpyHostToDevice));
    TLRG_CUDA(cudaMemcpy(dB, B, 8 * nbb, cudaMemcpyHostToDevice));
    TLRG_CUDA(cudaMemcpy(dC, Cm, 8 * nc, cudaMemcpyHostToDevice));
    std::vector<GemmProblem> p(1);
    p[0] = GemmProblem{};
    p[0].A = dA; p[0].lda = ta ? K : M; p[0].transA = ta;
    p[0].B = dB; p[0].ldb = tb ? N : K; p[0].transB = tb;
    p[0].C = dC; p[0].ldc = M; p[0].M = M; p[0].N = N; p[0].K = K;
    p[0].alpha = alpha; p[0].beta = beta;
    C.gemm(p);
    C.sync();
    TLRG_CUDA(cudaMemcpy(Cm, dC, 8 * nc, cudaMemcpyDeviceToHost));
  });
}

int tlrg_build(tlrg_ctx ctx, int32_t dim, int64_t n, const double* coords, int32_t kernel_kind,
               double ell, double nugget, int32_t b, double eps, int32_t compressor,
               const tlrg_ara_config* cfg, tlrg_matrix* out, tlrg_status* st) {
  return guarded(st, [&] {
    auto* h = new tlrg_matrix_s;
    h->m = build_tlr_device(ctx->c, dim, n, coords, kernel_kind, ell, nugget, b, eps, compressor,
                            to_cfg(cfg));
    *out = h;
  });
}

}  // extern "C"
