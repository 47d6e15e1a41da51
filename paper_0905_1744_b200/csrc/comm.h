// libsa's NCCL communicator (comm.cpp): run-time resolved NCCL, the
// collectives Algorithm 2 needs (allgather, personalised all-to-all).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "../../include/sa.h"

namespace sa {
bool nccl_available();
sa_status nccl_unique_id(void* id_h);   // 128 bytes
sa_status nccl_init(void** comm_out, const void* id_h, int nranks, int rank);
void nccl_destroy(void* comm);
sa_status nccl_check(void* comm);       // asynchronous communicator errors
sa_status nccl_allgather(void* comm, const void* send, void* recv, int64_t bytes, cudaStream_t st);
sa_status nccl_alltoallv(void* comm, int nranks, int rank, const void* send, const int64_t* send_bytes,
                         const int64_t* send_displs, void* recv, const int64_t* recv_bytes,
                         const int64_t* recv_displs, cudaStream_t st);
}  // namespace sa
