// gsot_comm.cu — the column-sharded solve's collective.
//
// The reference has no multi-process path: its solve runs on one host
// (solver.hpp:284-293) and the only decomposition SURVEY.md §8(e) allows is
// by column. A sharded context (gsot_create_shard[_device]: cost[:, J_p],
// a on rank 0 and zeros elsewhere, b[J_p]) with a communicator attached runs
// the ordinary device solve (gsot_solver.cu) and sums, per device sequence,
// the gradient head and a 16-double scalar tail over the ranks, plus the
// L-BFGS dots inside every direction update. Two transports:
//  * NCCL (loaded with dlopen; the process's own libnccl.so.2 when torch has
//    loaded one): ncclAllReduce on the context stream, captured into the
//    solver's CUDA graphs like any kernel;
//  * a host callback (tests, hosts without NCCL): the stream is synchronised,
//    the doubles reduced in pinned host memory by the caller, copied back.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "gsot_ctx.cuh"

namespace gsot {

namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // the copy already in the process (torch's) first, then the loader's
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.why = std::string("libnccl.so.2 not loadable: ") + (e ? e : "?");
      return;
    }
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p && api.why.empty()) api.why = std::string("libnccl lacks ") + name;
      return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.ok = api.why.empty();
  });
  if (!api.ok) throw Error(GSOT_ERR_CUDA, "NCCL unavailable: " + api.why);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(GSOT_ERR_CUDA, std::string(what) + " failed: " + nccl().GetErrorString(r));
}

}  // namespace

ShardComm::~ShardComm() {
  if (nccl_comm) nccl().CommDestroy(static_cast<ncclComm_t>(nccl_comm));
  if (host_buf) cudaFreeHost(host_buf);
  if (d_tail) cudaFree(d_tail);
  if (d_red) cudaFree(d_red);
  if (d_n) cudaFree(d_n);
}

void ShardComm::group_begin() {
  if (kind == kNccl) nccl_check(nccl().GroupStart(), "ncclGroupStart");
}

void ShardComm::group_end() {
  if (kind == kNccl) nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
}

void ShardComm::allreduce(double* d, int64_t count, int op, cudaStream_t s) {
  if (count <= 0) return;
  if (kind == kNccl) {
    nccl_check(nccl().AllReduce(d, d, static_cast<size_t>(count), ncclFloat64,
                                op == GSOT_REDUCE_MAX ? ncclMax : ncclSum,
                                static_cast<ncclComm_t>(nccl_comm), s),
               "ncclAllReduce");
    return;
  }
  if (static_cast<size_t>(count) > host_cap) {
    if (host_buf) cudaFreeHost(host_buf);
    host_buf = nullptr;
    GSOT_CUDA_CHECK(cudaMallocHost(&host_buf, sizeof(double) * count));
    host_cap = static_cast<size_t>(count);
  }
  GSOT_CUDA_CHECK(cudaMemcpyAsync(host_buf, d, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
  GSOT_CUDA_CHECK(cudaStreamSynchronize(s));
  if (fn(host_buf, count, op, user) != 0)
    throw Error(GSOT_ERR_CUDA, "host all-reduce callback failed");
  GSOT_CUDA_CHECK(cudaMemcpyAsync(d, host_buf, sizeof(double) * count, cudaMemcpyHostToDevice, s));
}

// Attach: allocate the device buffers, then one all-reduce of the shard's
// column count gives n_global (GradStats of dense calls, solver.hpp:117-119).
void comm_attach(gsot_ctx* c, std::unique_ptr<ShardComm> cm) {
  if (cm->world < 1 || cm->rank < 0 || cm->rank >= cm->world)
    throw Error(GSOT_ERR_INVALID_ARGUMENT, "bad rank / world size");
  GSOT_CUDA_CHECK(cudaMalloc(&cm->d_tail, sizeof(double) * kShardTail));
  GSOT_CUDA_CHECK(cudaMalloc(&cm->d_red, sizeof(double) * (kMaxMemory + 1) * 5));
  GSOT_CUDA_CHECK(cudaMalloc(&cm->d_n, sizeof(double)));
  const double nl = static_cast<double>(c->n);
  GSOT_CUDA_CHECK(cudaMemcpyAsync(cm->d_n, &nl, sizeof(double), cudaMemcpyHostToDevice, c->stream));
  cm->allreduce(cm->d_n, 1, GSOT_REDUCE_SUM, c->stream);
  double ng = 0.0;
  GSOT_CUDA_CHECK(cudaMemcpyAsync(&ng, cm->d_n, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  GSOT_CUDA_CHECK(cudaStreamSynchronize(c->stream));
  cm->n_global = static_cast<int64_t>(ng);
  c->comm = std::move(cm);
  c->pending_grad = nullptr;
  ++c->graph_epoch;  // captured graphs never mix transports
}

}  // namespace gsot

using gsot::Error;

namespace {
template <typename F>
int comm_guard(F&& f) {
  return gsot_guard_call(std::function<void()>(std::forward<F>(f)));
}
}  // namespace

GSOT_API int gsot_comm_unique_id(unsigned char id[128]) {
  return comm_guard([&] {
    if (!id) throw Error(GSOT_ERR_INVALID_ARGUMENT, "null id");
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL_UNIQUE_ID_BYTES");
    ncclUniqueId u;
    gsot::nccl_check(gsot::nccl().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
  });
}

GSOT_API int gsot_comm_attach_nccl(gsot_ctx* ctx, const unsigned char id[128], int32_t world,
                                   int32_t rank) {
  return comm_guard([&] {
    if (!ctx || !id) throw Error(GSOT_ERR_INVALID_ARGUMENT, "null argument");
    if (world < 1 || rank < 0 || rank >= world)
      throw Error(GSOT_ERR_INVALID_ARGUMENT, "bad rank / world size");
    std::unique_ptr<gsot::ShardComm> cm(new gsot::ShardComm());
    cm->kind = gsot::ShardComm::kNccl;
    cm->world = world;
    cm->rank = rank;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    ncclComm_t comm = nullptr;
    GSOT_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    gsot::nccl_check(gsot::nccl().CommInitRank(&comm, world, u, rank), "ncclCommInitRank");
    cm->nccl_comm = comm;
    gsot::comm_attach(ctx, std::move(cm));
  });
}

GSOT_API int gsot_comm_attach_host(gsot_ctx* ctx, int32_t world, int32_t rank,
                                   gsot_allreduce_fn fn, void* user) {
  return comm_guard([&] {
    if (!ctx || !fn) throw Error(GSOT_ERR_INVALID_ARGUMENT, "null argument");
    std::unique_ptr<gsot::ShardComm> cm(new gsot::ShardComm());
    cm->kind = gsot::ShardComm::kHost;
    cm->world = world;
    cm->rank = rank;
    cm->fn = fn;
    cm->user = user;
    gsot::comm_attach(ctx, std::move(cm));
  });
}

GSOT_API int gsot_comm_detach(gsot_ctx* ctx) {
  return comm_guard([&] {
    if (!ctx) throw Error(GSOT_ERR_INVALID_ARGUMENT, "null context");
    if (!ctx->comm) return;
    GSOT_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    ctx->comm.reset();
    ctx->pending_grad = nullptr;
    ++ctx->graph_epoch;
  });
}
