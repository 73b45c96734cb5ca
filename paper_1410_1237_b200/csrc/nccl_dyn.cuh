// nccl_dyn.cuh -- the NCCL calls of the partitioned phase engine (nccl_dyn.cu
// binds them at run time; nccl.h supplies only the types).
#pragma once
#include "common.cuh"
#include <nccl.h>
#include <cstring>

namespace plv {

void nccl_group_start();
void nccl_group_end();
// In-place broadcast of `count` elements from `root` (capturable).
void nccl_bcast_inplace(void *buf, size_t count, ncclDataType_t type, int root, void *comm,
                        cudaStream_t s);

// In-place all-gather: rank r's bytes_per_rank bytes sit at buf + r * bytes_per_rank.
void nccl_allgather_inplace(void *buf, size_t bytes_per_rank, int rank, void *comm,
                            cudaStream_t s);

}  // namespace plv
