// Multi-GPU exchange for the intra-column tile split.
//
// Every rank holds the whole factor (L is replicated) and runs the diagonal
// path redundantly; the rank-sorted active tiles of each column are dealt
// round-robin over the ranks, each rank runs the fused ARA + recompression +
// TRSM on its share, and one variable-size all-gather per column
// (counts all-gather + one broadcast per root, grouped) replicates the new
// U/V panel.  Per-tile gaussian streams are seeded by (root, i, k), so the
// factor is bitwise identical for any number of ranks.
//
// Two transports behind one interface:
//   * NCCL (one process per GPU; libnccl.so.2 is dlopen'ed on first use, so
//     the library has no link-time NCCL dependency);
//   * in-process ranks driven by host threads (device -> host -> device
//     copies through a shared staging area): exercises the exact split /
//     pack / unpack path with several contexts on one GPU (tests).
#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <mutex>

#include "../../include/tlrg.h"
#include "core.h"

namespace tlrg {

// ------------------------------------------------------------------ NCCL ---
namespace nccl {
typedef struct {
  char internal[128];
} UniqueId;
typedef void* Comm;
enum { ncclInt32 = 2, ncclFloat64 = 8 };
struct Api {
  bool ok = false;
  std::string why;
  int (*GetUniqueId)(UniqueId*);
  int (*CommInitRank)(Comm*, int, UniqueId, int);
  int (*CommDestroy)(Comm);
  int (*Broadcast)(const void*, void*, size_t, int, int, Comm, cudaStream_t);
  int (*AllGather)(const void*, void*, size_t, int, Comm, cudaStream_t);
  int (*GroupStart)();
  int (*GroupEnd)();
  const char* (*GetErrorString)(int);
};
Api& api() {
  static Api a = [] {
    Api x;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      x.why = "libnccl.so.2 not found";
      return x;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    x.GetUniqueId = (int (*)(UniqueId*))sym("ncclGetUniqueId");
    x.CommInitRank = (int (*)(Comm*, int, UniqueId, int))sym("ncclCommInitRank");
    x.CommDestroy = (int (*)(Comm))sym("ncclCommDestroy");
    x.Broadcast = (int (*)(const void*, void*, size_t, int, int, Comm, cudaStream_t))sym(
        "ncclBroadcast");
    x.AllGather =
        (int (*)(const void*, void*, size_t, int, Comm, cudaStream_t))sym("ncclAllGather");
    x.GroupStart = (int (*)())sym("ncclGroupStart");
    x.GroupEnd = (int (*)())sym("ncclGroupEnd");
    x.GetErrorString = (const char* (*)(int))sym("ncclGetErrorString");
    x.ok = x.GetUniqueId && x.CommInitRank && x.Broadcast && x.AllGather && x.GroupStart &&
           x.GroupEnd;
    if (!x.ok) x.why = "libnccl.so.2 lacks required symbols";
    return x;
  }();
  return a;
}
void check(int r, const char* what) {
  if (r != 0) {
    const char* s = api().GetErrorString ? api().GetErrorString(r) : "?";
    throw CudaError(std::string(what) + ": " + s);
  }
}
}  // namespace nccl

struct NcclComm : Comm {
  nccl::Comm c = nullptr;
  ~NcclComm() override {
    if (c && nccl::api().CommDestroy) nccl::api().CommDestroy(c);
  }
  void allgather_ints(Ctx& C, const int* send, int n, int* recv) override {
    int* d = C.buf<int>("comm_ints", (size_t)n * (world + 1));
    TLRG_CUDA(cudaMemcpyAsync(d, send, sizeof(int) * n, cudaMemcpyHostToDevice, C.st));
    nccl::check(nccl::api().AllGather(d, d + n, n, nccl::ncclInt32, c, C.st), "ncclAllGather");
    TLRG_CUDA(cudaMemcpyAsync(recv, d + n, sizeof(int) * n * world, cudaMemcpyDeviceToHost, C.st));
    C.wait();
  }
  void broadcast_all(Ctx& C, const double* mine, const std::vector<double*>& dst,
                     const std::vector<long long>& counts) override {
    nccl::check(nccl::api().GroupStart(), "ncclGroupStart");
    for (int r = 0; r < world; ++r) {
      if (counts[r] == 0) continue;
      const void* sb = r == rank ? (const void*)mine : (const void*)dst[r];
      void* rb = r == rank ? (void*)mine : (void*)dst[r];
      nccl::check(nccl::api().Broadcast(sb, rb, (size_t)counts[r], nccl::ncclFloat64, r, c, C.st),
                  "ncclBroadcast");
    }
    nccl::check(nccl::api().GroupEnd(), "ncclGroupEnd");
  }
};

// ------------------------------------------------------------ in-process ---
struct LocalHub {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  std::vector<std::vector<int>> ints;
  std::vector<std::vector<double>> data;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long g = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != g; });
    }
  }
};

struct LocalComm : Comm {
  std::shared_ptr<LocalHub> hub;
  void allgather_ints(Ctx&, const int* send, int n, int* recv) override {
    hub->ints[rank].assign(send, send + n);
    hub->barrier();
    for (int r = 0; r < world; ++r) std::memcpy(recv + (size_t)r * n, hub->ints[r].data(), 4 * n);
    hub->barrier();
  }
  void broadcast_all(Ctx& C, const double* mine, const std::vector<double*>& dst,
                     const std::vector<long long>& counts) override {
    auto& own = hub->data[rank];
    own.resize((size_t)counts[rank]);
    if (counts[rank])
      TLRG_CUDA(cudaMemcpyAsync(own.data(), mine, 8 * counts[rank], cudaMemcpyDeviceToHost, C.st));
    C.wait();
    hub->barrier();
    for (int r = 0; r < world; ++r)
      if (r != rank && counts[r])
        TLRG_CUDA(cudaMemcpyAsync(dst[r], hub->data[r].data(), 8 * counts[r],
                                  cudaMemcpyHostToDevice, C.st));
    C.wait();
    hub->barrier();
  }
};

// ------------------------------------------------- the per-column exchange ---
// res: all tiles i > k of the column (ascending i); on entry only the tiles
// this rank owns (slot s of the rank-sorted queue with s % world == rank) are
// filled, their U/V in one contiguous buffer [U panel | V panel] starting at
// `mine` (TRSM already applied).  On exit every tile is filled; received
// panels are allocated from `store` and referenced in place.
void exchange_column(Ctx& C, Comm& cm, const Matrix& M, int k, const std::vector<int>& queue,
                     std::vector<TileResult>& res, double* mine, Store& store) {
  const int P = cm.world, T = (int)queue.size(), rk = M.rows(k);
  const int per = (T + P - 1) / P;
  // owner r holds slots r, r + P, ...; its tiles travel in ascending i
  std::vector<std::vector<int>> tiles(P);
  for (int s = 0; s < T; ++s) tiles[s % P].push_back(queue[s]);
  for (auto& v : tiles) std::sort(v.begin(), v.end());
  std::vector<int> send(per, 0), recv((size_t)per * P, 0);
  for (size_t t = 0; t < tiles[cm.rank].size(); ++t) send[t] = res[tiles[cm.rank][t] - k - 1].rank;
  cm.allgather_ints(C, send.data(), per, recv.data());
  std::vector<long long> counts(P, 0), ucount(P, 0);
  for (int r = 0; r < P; ++r)
    for (size_t t = 0; t < tiles[r].size(); ++t) {
      const int q = recv[(size_t)r * per + t];
      ucount[r] += (long long)M.rows(tiles[r][t]) * q;
      counts[r] += (long long)(M.rows(tiles[r][t]) + rk) * q;
    }
  std::vector<double*> dst(P, nullptr);
  for (int r = 0; r < P; ++r)
    if (r != cm.rank && counts[r]) dst[r] = store.alloc((size_t)counts[r]);
  cm.broadcast_all(C, mine, dst, counts);
  for (int r = 0; r < P; ++r) {
    if (r == cm.rank) continue;
    long long uo = 0, vo = ucount[r];
    for (size_t t = 0; t < tiles[r].size(); ++t) {
      const int i = tiles[r][t], q = recv[(size_t)r * per + t];
      TileResult& tr = res[i - k - 1];
      tr.rank = q;
      tr.rounds = 0;  // ARA statistics stay with the owning rank
      tr.U = q ? dst[r] + uo : nullptr;
      tr.V = q ? dst[r] + vo : nullptr;
      uo += (long long)M.rows(i) * q;
      vo += (long long)rk * q;
    }
  }
}

}  // namespace tlrg

using namespace tlrg;

struct tlrg_ctx_s;  // defined in capi.cu
extern "C" {

struct tlrg_comm_s {
  std::shared_ptr<Comm> c;
};

int tlrg_comm_nccl_id(uint8_t* id, tlrg_status* st) {
  try {
    auto& a = nccl::api();
    if (!a.ok) throw Error(2, "tlrg_comm_nccl_id: " + a.why);
    nccl::UniqueId u;
    nccl::check(a.GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, u.internal, 128);
    if (st) st->code = 0;
    return 0;
  } catch (const Error& e) {
    if (st) {
      st->code = e.code;
      std::snprintf(st->msg, sizeof st->msg, "%s", e.what());
    }
    return e.code;
  } catch (const std::exception& e) {
    if (st) {
      st->code = 1;
      std::snprintf(st->msg, sizeof st->msg, "%s", e.what());
    }
    return 1;
  }
}

}  // extern "C"

namespace tlrg {
std::shared_ptr<Comm> make_nccl_comm(int rank, int world, const uint8_t* id) {
  auto& a = nccl::api();
  if (!a.ok) throw Error(2, "NCCL transport unavailable: " + a.why);
  auto c = std::make_shared<NcclComm>();
  c->rank = rank;
  c->world = world;
  nccl::UniqueId u;
  std::memcpy(u.internal, id, 128);
  nccl::check(a.CommInitRank(&c->c, world, u, rank), "ncclCommInitRank");
  return c;
}
std::vector<std::shared_ptr<Comm>> make_local_comms(int world) {
  auto hub = std::make_shared<LocalHub>();
  hub->world = world;
  hub->ints.resize(world);
  hub->data.resize(world);
  std::vector<std::shared_ptr<Comm>> out;
  for (int r = 0; r < world; ++r) {
    auto c = std::make_shared<LocalComm>();
    c->rank = r;
    c->world = world;
    c->hub = hub;
    out.push_back(c);
  }
  return out;
}
}  // namespace tlrg
