// comm.h — internal interface of comm.cpp (the exchange step's NCCL calls)
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace hsf {
struct Comm;
int comm_nranks(const Comm* c);
int comm_rank(const Comm* c);
int comm_device(const Comm* c);
uint64_t comm_serial(const Comm* c);
bool comm_same_hash(Comm* c, uint64_t hash, cudaStream_t st);
void comm_allreduce(Comm* c, void* buf, size_t count, bool f64, cudaStream_t st);
void comm_reduce_scatter(Comm* c, const void* in, void* out, size_t count_per_rank, bool f64, cudaStream_t st);
void comm_check_async(Comm* c);
}  // namespace hsf
