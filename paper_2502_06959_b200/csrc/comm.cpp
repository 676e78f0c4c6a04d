// comm.cpp — the exchange step of multi-GPU HSF behind the C ABI (P:109:
// the paths are independent, their contributions are "added up"): an NCCL
// communicator owned by libhsf.so, and the sum over ranks of the partial
// amplitude vectors (all-reduce) or of the row shards (reduce-scatter)
// enqueued by hsf_run on its stream right after the path-sum -- inside the
// run's captured CUDA graph.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2: inside a process that
// already loaded PyTorch's NCCL this returns that same library), so the
// library links and loads without it; hsf_comm_* report HSF_ERR_NCCL when it
// is missing.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>

#include "comm.h"
#include "hsf_internal.h"

namespace hsf {

namespace {
// the few NCCL declarations used (nccl.h, ABI-stable since 2.x)
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;  // 0 = ncclSuccess
enum { ncclFloat32 = 7, ncclFloat64 = 8, ncclUint64 = 5 };
enum { ncclSum = 0 };

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, void*) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, int, int, ncclComm_t, void*) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, void*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string err;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (n.h) break;
    }
    if (!n.h) {
      const char* e = dlerror();
      n.err = std::string("libnccl.so.2 not loadable: ") + (e ? e : "?");
      return;
    }
    auto sym = [&](const char* s) {
      void* p = dlsym(n.h, s);
      if (!p && n.err.empty()) n.err = std::string("NCCL symbol missing: ") + s;
      return p;
    };
    n.GetUniqueId = (decltype(n.GetUniqueId))sym("ncclGetUniqueId");
    n.CommInitRank = (decltype(n.CommInitRank))sym("ncclCommInitRank");
    n.CommDestroy = (decltype(n.CommDestroy))sym("ncclCommDestroy");
    n.CommGetAsyncError = (decltype(n.CommGetAsyncError))sym("ncclCommGetAsyncError");
    n.AllReduce = (decltype(n.AllReduce))sym("ncclAllReduce");
    n.ReduceScatter = (decltype(n.ReduceScatter))sym("ncclReduceScatter");
    n.AllGather = (decltype(n.AllGather))sym("ncclAllGather");
    n.GetErrorString = (decltype(n.GetErrorString))sym("ncclGetErrorString");
  });
  if (!n.err.empty()) fail(HSF_ERR_NCCL, n.err);
  return n;
}

void nck(ncclResult_t r, const char* what) {
  if (r != 0) {
    Nccl& n = nccl();
    fail(HSF_ERR_NCCL, std::string(what) + ": " + (n.GetErrorString ? n.GetErrorString(r) : "error"));
  }
}
}  // namespace

struct Comm {
  ncclComm_t c = nullptr;
  int nranks = 1, rank = 0, device = -1;
  uint64_t serial = 0;  // distinguishes communicators for the plans' hash-check cache
};

void comm_unique_id(void* out128) {
  ncclUniqueId id;
  nck(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
}

Comm* comm_create(const void* id128, int nranks, int rank, int device) {
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(HSF_ERR_INVALID_ARG, "bad nranks / rank");
  static uint64_t serial = 0;
  Nccl& n = nccl();
  int cur = -1;
  cudaGetDevice(&cur);
  if (device >= 0 && cudaSetDevice(device) != cudaSuccess) fail(HSF_ERR_CUDA, "cudaSetDevice");
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  auto* c = new Comm();
  c->nranks = nranks;
  c->rank = rank;
  cudaGetDevice(&c->device);
  const ncclResult_t r = n.CommInitRank(&c->c, nranks, id, rank);
  if (cur >= 0) cudaSetDevice(cur);
  if (r != 0) {
    delete c;
    nck(r, "ncclCommInitRank");
  }
  c->serial = ++serial;
  return c;
}

void comm_free(Comm* c) {
  if (!c) return;
  if (c->c) {
    Nccl& n = nccl();
    n.CommDestroy(c->c);
  }
  delete c;
}

int comm_nranks(const Comm* c) { return c->nranks; }
int comm_rank(const Comm* c) { return c->rank; }
int comm_device(const Comm* c) { return c->device; }
uint64_t comm_serial(const Comm* c) { return c->serial; }

// every rank's plan hash equal? (one all-gather; synchronises the stream)
bool comm_same_hash(Comm* c, uint64_t hash, cudaStream_t st) {
  if (c->nranks == 1) return true;
  Nccl& n = nccl();
  uint64_t* d = nullptr;
  if (cudaMalloc(&d, sizeof(uint64_t) * (c->nranks + 1)) != cudaSuccess) fail(HSF_ERR_OUT_OF_MEMORY, "hash buffer");
  bool ok = true;
  try {
    if (cudaMemcpyAsync(d, &hash, 8, cudaMemcpyHostToDevice, st) != cudaSuccess) fail(HSF_ERR_CUDA, "hash H2D");
    nck(n.AllGather(d, d + 1, 1, ncclUint64, c->c, st), "ncclAllGather (plan hash)");
    std::string buf(8 * c->nranks, '\0');
    if (cudaMemcpyAsync(&buf[0], d + 1, 8 * c->nranks, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      fail(HSF_ERR_CUDA, "hash D2H");
    for (int r = 0; r < c->nranks; ++r) {
      uint64_t v;
      std::memcpy(&v, &buf[8 * r], 8);
      ok = ok && v == hash;
    }
  } catch (...) {
    cudaFree(d);
    throw;
  }
  cudaFree(d);
  return ok;
}

// sum over ranks: in place (all-reduce) or into each rank's shard (reduce-scatter);
// `count` real elements (2 per complex), fp32 or fp64
void comm_allreduce(Comm* c, void* buf, size_t count, bool f64, cudaStream_t st) {
  nck(nccl().AllReduce(buf, buf, count, f64 ? ncclFloat64 : ncclFloat32, ncclSum, c->c, st), "ncclAllReduce");
}
void comm_reduce_scatter(Comm* c, const void* in, void* out, size_t count_per_rank, bool f64, cudaStream_t st) {
  nck(nccl().ReduceScatter(in, out, count_per_rank, f64 ? ncclFloat64 : ncclFloat32, ncclSum, c->c, st),
      "ncclReduceScatter");
}
void comm_check_async(Comm* c) {
  ncclResult_t a = 0;
  nck(nccl().CommGetAsyncError(c->c, &a), "ncclCommGetAsyncError");
  nck(a, "NCCL asynchronous error");
}

}  // namespace hsf

using namespace hsf;

extern "C" {

hsf_status hsf_comm_unique_id(void* out128) {
  try {
    if (!out128) fail(HSF_ERR_INVALID_ARG, "NULL argument");
    comm_unique_id(out128);
    return HSF_OK;
  } catch (const Error& e) {
    set_last_error(e.msg);
    return e.st;
  } catch (...) {
    set_last_error("unknown C++ exception");
    return HSF_ERR_INVALID_ARG;
  }
}

hsf_status hsf_comm_create(const void* id128, int32_t nranks, int32_t rank, int32_t device, hsf_comm_t** out) {
  try {
    if (!id128 || !out) fail(HSF_ERR_INVALID_ARG, "NULL argument");
    *out = nullptr;
    *out = reinterpret_cast<hsf_comm_t*>(comm_create(id128, nranks, rank, device));
    return HSF_OK;
  } catch (const Error& e) {
    set_last_error(e.msg);
    return e.st;
  } catch (...) {
    set_last_error("unknown C++ exception");
    return HSF_ERR_INVALID_ARG;
  }
}

void hsf_comm_free(hsf_comm_t* c) {
  try {
    comm_free(reinterpret_cast<Comm*>(c));
  } catch (...) {
  }
}

}  // extern "C"
