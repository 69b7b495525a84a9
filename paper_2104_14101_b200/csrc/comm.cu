// Row-shard exchanges inside libadask.  One process per
// GPU; the context owns (or borrows) an NCCL communicator and every exchange
// of the sharded solve is issued on the solve's stream from native code:
//
//   per loop pass   all-reduce of the d*c partial A_g^T (A_g x)  (problem.py:89-95)
//                   (PCG proposals: ONE all-reduce of the 2d pair [A_g^T A_g p, A_g^T A_g x])
//   per resketch    reduce-scatter of the m x d partial S_g A_g (embeddings.py:117-129),
//                   partial Gram of this rank's m/G rows, all-reduce of the d x d Gram
//                   (dense path); the Woodbury path all-reduces SA (its apply needs all of it)
//
// NCCL is resolved at run time (dlopen of libnccl.so.2 -- the copy torch
// loads when it is already in the process), so libadask has no link-time
// NCCL dependency and single-GPU use never touches it.  A problem may instead
// carry a host all-reduce hook (adask_problem.allreduce): the CPU-side tests
// drive the same sharded code through torch.distributed gloo with it.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "comm.cuh"

namespace adask {
namespace {

struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*reduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  std::string why;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (api.tried) return api;
  api.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    api.why = dlerror() ? dlerror() : "dlopen(libnccl.so.2) failed";
    return api;
  }
#define ADASK_SYM(field, name)                                  \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name)); \
  if (!api.field) {                                             \
    api.why = "libnccl lacks " name;                            \
    return api;                                                 \
  }
  ADASK_SYM(getUniqueId, "ncclGetUniqueId");
  ADASK_SYM(commInitRank, "ncclCommInitRank");
  ADASK_SYM(commDestroy, "ncclCommDestroy");
  ADASK_SYM(allReduce, "ncclAllReduce");
  ADASK_SYM(reduceScatter, "ncclReduceScatter");
  ADASK_SYM(getErrorString, "ncclGetErrorString");
#undef ADASK_SYM
  api.ok = true;
  return api;
}

int nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return ADASK_OK;
  return fail(ADASK_E_CUDA, "%s: %s", what, nccl().getErrorString ? nccl().getErrorString(r) : "nccl error");
}

ncclDataType_t nccl_type(int dtype) { return dtype == ADASK_F64 ? ncclFloat64 : ncclFloat32; }

}  // namespace

bool problem_sharded(const adask_ctx* ctx, const adask_problem* pb) {
  return pb->allreduce != nullptr || (pb->use_ctx_comm && ctx->comm.nccl != nullptr);
}

int comm_rank(const adask_ctx* ctx, const adask_problem* pb) {
  return pb->allreduce ? pb->comm_rank : ctx->comm.rank;
}
int comm_world(const adask_ctx* ctx, const adask_problem* pb) {
  if (pb->allreduce) return pb->comm_world > 0 ? pb->comm_world : 1;
  return pb->use_ctx_comm && ctx->comm.nccl ? ctx->comm.world : 1;
}

int problem_allreduce(adask_ctx* ctx, const adask_problem* pb, void* buf, int64_t count, int dtype,
                      cudaStream_t st) {
  if (count <= 0) return ADASK_OK;
  if (pb->allreduce) {
    if (pb->allreduce(buf, count, dtype, pb->allreduce_user, (void*)st) != 0)
      return fail(ADASK_E_CUDA, "all-reduce hook failed");
    return ADASK_OK;
  }
  if (!(pb->use_ctx_comm && ctx->comm.nccl)) return ADASK_OK;  // not sharded
  return nccl_check(nccl().allReduce(buf, buf, (size_t)count, nccl_type(dtype), ncclSum,
                                     (ncclComm_t)ctx->comm.nccl, st),
                    "ncclAllReduce");
}

// Sum over ranks of send (world * count elements); this rank's slice
// [rank*count, (rank+1)*count) of the sum lands in *recv.  NCCL: a
// reduce-scatter into `scratch`; hook: an all-reduce of send in place, *recv
// points into it.
int problem_reduce_scatter(adask_ctx* ctx, const adask_problem* pb, void* send, void* scratch, int64_t count,
                           int dtype, void** recv, cudaStream_t st) {
  const size_t esz = dtype == ADASK_F64 ? 8 : 4;
  if (pb->allreduce) {
    ADASK_TRY(problem_allreduce(ctx, pb, send, count * comm_world(ctx, pb), dtype, st));
    *recv = (char*)send + (size_t)comm_rank(ctx, pb) * count * esz;
    return ADASK_OK;
  }
  if (!(pb->use_ctx_comm && ctx->comm.nccl)) {
    *recv = send;
    return ADASK_OK;
  }
  ADASK_TRY(nccl_check(nccl().reduceScatter(send, scratch, (size_t)count, nccl_type(dtype), ncclSum,
                                            (ncclComm_t)ctx->comm.nccl, st),
                       "ncclReduceScatter"));
  *recv = scratch;
  return ADASK_OK;
}

void comm_release(adask_ctx* ctx) {
  if (ctx->comm.nccl && ctx->comm.owned && nccl().ok) nccl().commDestroy((ncclComm_t)ctx->comm.nccl);
  ctx->comm = CommState{};
}

}  // namespace adask

using namespace adask;

extern "C" int adask_nccl_available(void) { return nccl().ok ? 1 : 0; }

extern "C" int adask_nccl_unique_id(void* id_out) {
  if (!id_out) return fail(ADASK_E_ARG, "null id buffer");
  if (!nccl().ok) return fail(ADASK_E_CUDA, "NCCL unavailable: %s", nccl().why.c_str());
  ncclUniqueId id;
  ADASK_TRY(nccl_check(nccl().getUniqueId(&id), "ncclGetUniqueId"));
  memcpy(id_out, &id, sizeof(id));
  return ADASK_OK;
}

extern "C" int adask_comm_init_nccl(adask_ctx* ctx, const void* id, int rank, int world) {
  ADASK_TRY(use_device(ctx));
  if (!id || world < 1 || rank < 0 || rank >= world) return fail(ADASK_E_ARG, "comm_init: bad rank / world");
  if (!nccl().ok) return fail(ADASK_E_CUDA, "NCCL unavailable: %s", nccl().why.c_str());
  comm_release(ctx);
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  ADASK_TRY(nccl_check(nccl().commInitRank(&c, world, uid, rank), "ncclCommInitRank"));
  ctx->comm.nccl = c;
  ctx->comm.rank = rank;
  ctx->comm.world = world;
  ctx->comm.owned = true;
  return ADASK_OK;
}

extern "C" int adask_set_comm(adask_ctx* ctx, void* nccl_comm, int rank, int world) {
  if (!ctx) return fail(ADASK_E_ARG, "null ctx");
  if (world < 1 || rank < 0 || rank >= world) return fail(ADASK_E_ARG, "set_comm: bad rank / world");
  comm_release(ctx);
  ctx->comm.nccl = nccl_comm;
  ctx->comm.rank = rank;
  ctx->comm.world = world;
  ctx->comm.owned = false;
  return ADASK_OK;
}

extern "C" int adask_comm_destroy(adask_ctx* ctx) {
  if (!ctx) return ADASK_OK;
  comm_release(ctx);
  return ADASK_OK;
}

extern "C" int adask_comm_allreduce(adask_ctx* ctx, void* buf, int64_t count, int dtype, void* stream) {
  ADASK_TRY(use_device(ctx));
  if (!ctx->comm.nccl) return ADASK_OK;
  return nccl_check(nccl().allReduce(buf, buf, (size_t)count, nccl_type(dtype), ncclSum, (ncclComm_t)ctx->comm.nccl,
                                     S(stream)),
                    "ncclAllReduce");
}
