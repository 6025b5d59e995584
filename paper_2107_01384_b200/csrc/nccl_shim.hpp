// NCCL entry points used by the sharded compress (loaded at run time, nccl_shim.cpp).
#pragma once

#include <nccl.h>

#include <cstring>

#include "common.cuh"

namespace tcb {

void nccl_unique_id(unsigned char out[128]);
void* nccl_comm_init(const unsigned char id[128], int world, int rank);
void nccl_comm_destroy(void* comm);
// in place, fp64 sum over the communicator, ordered on `s`
void nccl_allreduce_sum_f64(double* buf, u64 count, void* comm, cudaStream_t s);
// recv = the ranks' `send` blocks of count_per_rank doubles, rank-major
void nccl_allgather_f64(const double* send, double* recv, u64 count_per_rank, void* comm, cudaStream_t s);
void nccl_allgather_bytes(const void* send, void* recv, u64 bytes_per_rank, void* comm, cudaStream_t s);

}  // namespace tcb
