// Communicators for the row-partitioned mode (comm.h) and their C ABI.
//
//   NcclComm  one rank per GPU (one process each), ncclAllReduce on the
//             compute stream; capturable, so the LSMR graphs keep the
//             exchange inside them.  NCCL is resolved at run time (dlopen of
//             the libnccl.so.2 that torch already loaded, else the system
//             one), so the library has no link-time NCCL dependency.
//   LocalComm `world` shards on ONE device, one host thread each: the
//             exchange is a host barrier around a fixed-order sum kernel.
//             No kernel ever waits on another shard's kernel; used to run
//             and test the partitioned algorithm for world > 1 on one GPU.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "comm.h"
#include "qg_common.cuh"

namespace qg {

namespace {

// ----------------------------------------------------------------- NCCL --
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char *(*error_string)(ncclResult_t) = nullptr;
  std::string why;
};

const NcclApi &nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW);
    if (!h) {
      a.why = "libnccl.so.2 not found";
      return a;
    }
    a.get_unique_id = (decltype(a.get_unique_id))dlsym(h, "ncclGetUniqueId");
    a.comm_init_rank = (decltype(a.comm_init_rank))dlsym(h, "ncclCommInitRank");
    a.all_reduce = (decltype(a.all_reduce))dlsym(h, "ncclAllReduce");
    a.comm_destroy = (decltype(a.comm_destroy))dlsym(h, "ncclCommDestroy");
    a.error_string = (decltype(a.error_string))dlsym(h, "ncclGetErrorString");
    if (!a.get_unique_id || !a.comm_init_rank || !a.all_reduce || !a.comm_destroy) a.why = "NCCL symbols missing";
    return a;
  }();
  if (!api.why.empty()) throw Error{QG_ERR_CUDA, "NCCL unavailable: " + api.why};
  return api;
}

void nccl_check(ncclResult_t r, const char *what) {
  if (r != ncclSuccess) {
    const NcclApi &a = nccl();
    throw Error{QG_ERR_CUDA, std::string(what) + ": " + (a.error_string ? a.error_string(r) : "NCCL error")};
  }
}

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) nccl().comm_destroy(comm);
  }
  void allreduce(double *buf, int64_t n, cudaStream_t st) override {
    if (n <= 0) return;
    nccl_check(nccl().all_reduce(buf, buf, (size_t)n, ncclFloat64, ncclSum, comm, st), "ncclAllReduce");
  }
  bool capturable() const override { return true; }
};

// ---------------------------------------------------------------- local --
struct LocalGroup {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int count = 0;
  long long gen = 0;
  std::vector<double *> bufs;
  void barrier() {
    std::unique_lock<std::mutex> l(mu);
    const long long g = gen;
    if (++count == world) {
      count = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(l, [&] { return gen != g; });
    }
  }
};

constexpr int kMaxLocal = 8;
struct RankPtrs {
  const double *p[kMaxLocal];
};

// out = buf_0 + buf_1 + ... in rank order (identical bits on every shard)
__global__ void k_sum_ranks(RankPtrs r, int world, int64_t n, double *out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = r.p[0][i];
    for (int k = 1; k < world; ++k) s += r.p[k][i];
    out[i] = s;
  }
}

struct LocalComm : Comm {
  std::shared_ptr<LocalGroup> g;
  double *tmp = nullptr;
  int64_t tmp_n = 0;
  ~LocalComm() override {
    if (tmp) cudaFree(tmp);
  }
  void allreduce(double *buf, int64_t n, cudaStream_t st) override {
    if (world == 1) return;
    if (n > tmp_n) {
      QG_CUDA(cudaStreamSynchronize(st));
      if (tmp) QG_CUDA(cudaFree(tmp));
      QG_CUDA(cudaMalloc(&tmp, sizeof(double) * (size_t)n));
      tmp_n = n;
    }
    QG_CUDA(cudaStreamSynchronize(st));  // this shard's partials are final
    g->bufs[rank] = buf;
    g->barrier();                        // ... and every other shard's
    RankPtrs rp{};
    for (int k = 0; k < world; ++k) rp.p[k] = g->bufs[k];
    if (n > 0) {
      const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8);
      k_sum_ranks<<<grid, 256, 0, st>>>(rp, world, n, tmp);
      QG_LAUNCHED();
    }
    QG_CUDA(cudaStreamSynchronize(st));
    g->barrier();                        // nobody reads the partials any more
    if (n > 0) QG_CUDA(cudaMemcpyAsync(buf, tmp, sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, st));
  }
  bool capturable() const override { return false; }
};

}  // namespace
}  // namespace qg

using namespace qg;

#define QG_COMM_TRY try {
#define QG_COMM_END                                                  \
  return QG_OK;                                                      \
  }                                                                  \
  catch (const qg::Error &e) { return qg::fail(e.code, e.msg); }      \
  catch (const std::exception &e) { return qg::fail(QG_ERR_CUDA, e.what()); }

extern "C" {

int qg_comm_nccl_id(unsigned char id[128]) {
  QG_COMM_TRY
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId u;
  nccl_check(nccl().get_unique_id(&u), "ncclGetUniqueId");
  std::memcpy(id, &u, 128);
  QG_COMM_END
}

int qg_comm_create_nccl(qg_comm **out, const unsigned char id[128], int world, int rank) {
  QG_COMM_TRY
  if (world < 1 || rank < 0 || rank >= world) throw Error{QG_ERR_VALIDATION, "bad rank / world size"};
  auto c = std::make_unique<NcclComm>();
  c->rank = rank;
  c->world = world;
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  nccl_check(nccl().comm_init_rank(&c->comm, world, u, rank), "ncclCommInitRank");
  *out = reinterpret_cast<qg_comm *>(static_cast<Comm *>(c.release()));
  QG_COMM_END
}

int qg_comm_create_local(qg_comm **out, int world) {
  QG_COMM_TRY
  if (world < 1 || world > kMaxLocal) throw Error{QG_ERR_VALIDATION, "local group size must be 1..8"};
  auto g = std::make_shared<LocalGroup>();
  g->world = world;
  g->bufs.assign(world, nullptr);
  for (int r = 0; r < world; ++r) {
    auto *c = new LocalComm();
    c->rank = r;
    c->world = world;
    c->g = g;
    out[r] = reinterpret_cast<qg_comm *>(static_cast<Comm *>(c));
  }
  QG_COMM_END
}

int qg_comm_destroy(qg_comm *c) {
  QG_COMM_TRY
  delete reinterpret_cast<Comm *>(c);
  QG_COMM_END
}

int qg_comm_rank(const qg_comm *c, int *rank, int *world) {
  QG_COMM_TRY
  const Comm *k = reinterpret_cast<const Comm *>(c);
  *rank = k->rank;
  *world = k->world;
  QG_COMM_END
}

int qg_comm_allreduce(qg_comm *c, double *buf, int64_t n, void *stream) {
  QG_COMM_TRY
  cudaStream_t st = (cudaStream_t)stream;
  reinterpret_cast<Comm *>(c)->allreduce(buf, n, st);
  QG_CUDA(cudaStreamSynchronize(st));
  QG_COMM_END
}

}  // extern "C"
