// Row-shard exchanges of the sharded solve (comm.cu).
#pragma once
#include "common.cuh"

namespace adask {
// true when the problem's A is one row shard (NCCL communicator on the ctx or
// a host all-reduce hook on the problem)
bool problem_sharded(const adask_ctx* ctx, const adask_problem* pb);
int comm_rank(const adask_ctx* ctx, const adask_problem* pb);
int comm_world(const adask_ctx* ctx, const adask_problem* pb);
// in-place sum over ranks (no-op when not sharded)
int problem_allreduce(adask_ctx* ctx, const adask_problem* pb, void* buf, int64_t count, int dtype, cudaStream_t st);
// this rank's `count`-element slice of the sum of `send` (world * count elements)
int problem_reduce_scatter(adask_ctx* ctx, const adask_problem* pb, void* send, void* scratch, int64_t count,
                           int dtype, void** recv, cudaStream_t st);
void comm_release(adask_ctx* ctx);
}  // namespace adask
