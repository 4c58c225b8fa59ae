// comm.cuh -- NCCL all-gather of the multi-GPU step (see comm.cu).
#pragma once

#include "common.cuh"

namespace rkfac_b200 {

size_t nccl_unique_id_bytes();
void nccl_unique_id(void* out);                                   // ncclGetUniqueId
void* nccl_comm_init(const void* id, int nranks, int rank);       // ncclCommInitRank (collective over the clique)
void nccl_comm_destroy(void* comm);
void nccl_allgather(void* comm, const float* send, float* recv, long long count, cudaStream_t s);

}  // namespace rkfac_b200
