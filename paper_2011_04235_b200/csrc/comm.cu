// Communicators of a sharded solve (comm.cuh): NCCL loaded at run time (the libnccl.so.2 that
// torch already mapped, so the library links without it), or a host callback.
#include <dlfcn.h>
#include <nccl.h>

#include "capi_guard.cuh"
#include "comm.cuh"

namespace fpi {
namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
      a.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return a;
    }
    auto sym = [&](const char* n) { return dlsym(lib, n); };
    a.get_unique_id = (decltype(a.get_unique_id))sym("ncclGetUniqueId");
    a.comm_init_rank = (decltype(a.comm_init_rank))sym("ncclCommInitRank");
    a.comm_destroy = (decltype(a.comm_destroy))sym("ncclCommDestroy");
    a.all_reduce = (decltype(a.all_reduce))sym("ncclAllReduce");
    a.all_gather = (decltype(a.all_gather))sym("ncclAllGather");
    a.reduce = (decltype(a.reduce))sym("ncclReduce");
    a.group_start = (decltype(a.group_start))sym("ncclGroupStart");
    a.group_end = (decltype(a.group_end))sym("ncclGroupEnd");
    a.error_string = (decltype(a.error_string))sym("ncclGetErrorString");
    a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.all_reduce && a.all_gather && a.reduce &&
           a.group_start && a.group_end && a.error_string;
    if (!a.ok) a.why = "libnccl.so.2 lacks an expected symbol";
    return a;
  }();
  return api;
}

#define FPI_NCCL(call)                                                                              \
  do {                                                                                              \
    ncclResult_t _r = (call);                                                                       \
    if (_r != ncclSuccess)                                                                          \
      throw ::fpi::Error(FPI_ECUDA, std::string("NCCL: ") + #call + ": " + nccl().error_string(_r)); \
  } while (0)

struct NcclComm final : Comm {
  ncclComm_t c = nullptr;
  ~NcclComm() override {
    if (c) nccl().comm_destroy(c);
  }
  void allreduce(double* buf, int64_t n, int op, cudaStream_t s) override {
    if (n > 0) FPI_NCCL(nccl().all_reduce(buf, buf, (size_t)n, ncclFloat64, op ? ncclMax : ncclSum, c, s));
  }
  void allgather(const double* send, double* recv, int64_t n, cudaStream_t s) override {
    if (n > 0) FPI_NCCL(nccl().all_gather(send, recv, (size_t)n, ncclFloat64, c, s));
  }
  void reduce(const double* send, double* recv, int64_t n, int root, cudaStream_t s) override {
    if (n > 0) FPI_NCCL(nccl().reduce(send, recv, (size_t)n, ncclFloat64, ncclSum, root, c, s));
  }
  void group_begin() override { FPI_NCCL(nccl().group_start()); }
  void group_end() override { FPI_NCCL(nccl().group_end()); }
};

// fpi_comm_fn (fastpi_b200.h): op 0 all-reduce sum (in place), 1 all-reduce max, 2 all-gather,
// 3 reduce to root; the library has synchronised its stream before the call.
struct CallbackComm final : Comm {
  fpi_comm_fn fn = nullptr;
  void* user = nullptr;
  void call(int op, const void* send, void* recv, int64_t n, int root, cudaStream_t s) {
    if (n <= 0) return;
    FPI_CUDA(cudaStreamSynchronize(s));
    const int rc = fn(user, op, send, recv, n, root);
    FPI_REQUIRE(rc == 0, FPI_ECUDA, "communicator callback failed (op " + std::to_string(op) + ")");
  }
  void allreduce(double* buf, int64_t n, int op, cudaStream_t s) override { call(op ? 1 : 0, buf, buf, n, 0, s); }
  void allgather(const double* send, double* recv, int64_t n, cudaStream_t s) override {
    call(2, send, recv, n, 0, s);
  }
  void reduce(const double* send, double* recv, int64_t n, int root, cudaStream_t s) override {
    call(3, send, recv, n, root, s);
  }
};

// world of one: every exchange is the identity (the sharded engine run on a single rank)
struct SelfComm final : Comm {
  void allreduce(double*, int64_t, int, cudaStream_t) override {}
  void allgather(const double* send, double* recv, int64_t n, cudaStream_t s) override {
    if (n > 0 && send != recv) FPI_CUDA(cudaMemcpyAsync(recv, send, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  }
  void reduce(const double* send, double* recv, int64_t n, int, cudaStream_t s) override {
    if (n > 0 && send != recv) FPI_CUDA(cudaMemcpyAsync(recv, send, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  }
};

}  // namespace

void comm_free(fpi_context* h) {
  delete h->comm;
  h->comm = nullptr;
}

}  // namespace fpi

extern "C" {

/* A fresh NCCL unique id (rank 0 creates it, the ranks exchange it out of band). */
int fpi_comm_nccl_id(char* h_out128, char* h_err, int64_t err_cap) {
  const auto& a = fpi::nccl();
  if (!a.ok) {
    if (h_err && err_cap > 0) snprintf(h_err, (size_t)err_cap, "%s", a.why.c_str());
    return FPI_ECUDA;
  }
  ncclUniqueId id;
  if (a.get_unique_id(&id) != ncclSuccess) return FPI_ECUDA;
  memcpy(h_out128, id.internal, NCCL_UNIQUE_ID_BYTES);
  return FPI_OK;
}

int fpi_comm_init_nccl(fpi_handle h, const char* h_id128, int rank, int world) {
  FPI_API_BEGIN(h)
  FPI_REQUIRE(world >= 1 && rank >= 0 && rank < world, FPI_EDOMAIN, "bad rank / world");
  const auto& a = fpi::nccl();
  FPI_REQUIRE(a.ok, FPI_ECUDA, a.why);
  fpi::comm_free(h);
  auto* c = new fpi::NcclComm();
  ncclUniqueId id;
  memcpy(id.internal, h_id128, NCCL_UNIQUE_ID_BYTES);
  const ncclResult_t r = a.comm_init_rank(&c->c, world, id, rank);
  if (r != ncclSuccess) {
    c->c = nullptr;
    delete c;
    throw fpi::Error(FPI_ECUDA, std::string("ncclCommInitRank: ") + a.error_string(r));
  }
  c->rank = rank;
  c->world = world;
  h->comm = c;
  FPI_API_END(h)
}

int fpi_comm_init_callback(fpi_handle h, int rank, int world, fpi_comm_fn fn, void* user) {
  FPI_API_BEGIN(h)
  FPI_REQUIRE(world >= 1 && rank >= 0 && rank < world && fn, FPI_EDOMAIN, "bad rank / world / callback");
  fpi::comm_free(h);
  auto* c = new fpi::CallbackComm();
  c->fn = fn;
  c->user = user;
  c->rank = rank;
  c->world = world;
  h->comm = c;
  FPI_API_END(h)
}

int fpi_comm_init_self(fpi_handle h) {
  FPI_API_BEGIN(h)
  fpi::comm_free(h);
  h->comm = new fpi::SelfComm();
  FPI_API_END(h)
}

int fpi_comm_free(fpi_handle h) {
  FPI_API_BEGIN(h)
  fpi::comm_free(h);
  FPI_API_END(h)
}

/* rank / world of the handle's communicator (0 / 1 without one) */
int fpi_comm_info(fpi_handle h, int* h_rank, int* h_world) {
  FPI_API_BEGIN(h)
  *h_rank = h->comm ? h->comm->rank : 0;
  *h_world = h->comm ? h->comm->world : 1;
  FPI_API_END(h)
}

/* In-place sum over the ranks of n doubles (device) -- the exchange primitive, exposed for tests. */
int fpi_comm_allreduce(fpi_handle h, double* d_buf, int64_t n) {
  FPI_API_BEGIN(h)
  FPI_REQUIRE(h->comm, FPI_EDOMAIN, "handle has no communicator");
  h->comm->allreduce(d_buf, n, 0, h->stream);
  FPI_API_END(h)
}

}  // extern "C"
