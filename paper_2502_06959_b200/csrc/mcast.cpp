// mcast.cpp — NVLink SHARP (NVLS) multicast buffers for the fused exchange of
// bitstring runs (the paths' contributions are
// added up).  Every rank binds `bytes` of its own device memory to one
// multicast object; a kernel's `multimem.red.add` on the multicast address
// adds into every rank's copy inside the NVSwitch, so after all ranks'
// block gathers every rank holds the whole sum -- an all-reduce with no
// collective call and no partial vector.
//
// Set-up (collective, in this order on every rank): rank 0
// hsf_mcast_create (exports a 64-byte fabric handle), the others
// hsf_mcast_import it; every rank hsf_mcast_add_device; barrier (all devices
// added before any bind); every rank hsf_mcast_bind; barrier.  One rank
// alone is a valid team (the box has one GPU: the tests run G = 1).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "hsf_internal.h"

namespace hsf {

namespace {
template <typename F>
F drv(const char* name) {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
      !f)
    fail(HSF_ERR_UNSUPPORTED, std::string("driver entry point unavailable: ") + name);
  return reinterpret_cast<F>(f);
}
#define HSF_DRV(fn) static auto p_##fn = drv<decltype(&fn)>(#fn)

void cu(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) {
    const char* s = nullptr;
    static auto p_err = drv<decltype(&cuGetErrorString)>("cuGetErrorString");
    p_err(r, &s);
    fail(r == CUDA_ERROR_NOT_SUPPORTED ? HSF_ERR_UNSUPPORTED : HSF_ERR_CUDA,
         std::string(what) + ": " + (s ? s : "CUDA driver error"));
  }
}
}  // namespace

struct Mcast {
  CUmemGenericAllocationHandle mc = 0, mem = 0;
  CUdeviceptr local = 0, multi = 0;
  size_t size = 0;  // granularity-rounded bytes
  int device = 0;
  bool bound = false, mapped_local = false, mapped_mc = false;
};

static size_t mc_granule(int nranks, size_t bytes, unsigned long long htypes) {
  HSF_DRV(cuMulticastGetGranularity);
  CUmulticastObjectProp pr{};
  pr.numDevices = (unsigned)nranks;
  pr.size = bytes;
  pr.handleTypes = htypes;
  size_t g = 0;
  cu(p_cuMulticastGetGranularity(&g, &pr, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity");
  return g ? g : (size_t)2 << 20;
}

static void set_dev(int device) {
  if (device >= 0 && cudaSetDevice(device) != cudaSuccess) fail(HSF_ERR_CUDA, "cudaSetDevice");
}

static Mcast* mcast_create(size_t bytes, int nranks, int device, void* handle64) {
  HSF_DRV(cuMulticastCreate);
  HSF_DRV(cuMemExportToShareableHandle);
  HSF_DRV(cuDeviceGetAttribute);
  set_dev(device);
  int attr = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  cu(p_cuDeviceGetAttribute(&attr, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, (CUdevice)dev), "cuDeviceGetAttribute");
  if (!attr) fail(HSF_ERR_UNSUPPORTED, "multicast objects are not supported on this device");
  auto* m = new Mcast();
  m->device = dev;
  // exportable as a fabric handle (multi-rank teams: the importers need it);
  // a team of one needs no export, so it falls back to a plain object where
  // fabric handles are unavailable (no IMEX channel)
  CUresult r = CUDA_ERROR_UNKNOWN;
  for (unsigned long long ht : {(unsigned long long)CU_MEM_HANDLE_TYPE_FABRIC, 0ull}) {
    if (ht == 0 && nranks > 1) break;
    const size_t g = mc_granule(nranks, bytes, ht);
    m->size = (bytes + g - 1) / g * g;
    CUmulticastObjectProp pr{};
    pr.numDevices = (unsigned)nranks;
    pr.size = m->size;
    pr.handleTypes = ht;
    r = p_cuMulticastCreate(&m->mc, &pr);
    if (r != CUDA_SUCCESS) continue;
    std::memset(handle64, 0, 64);
    if (ht) {
      CUmemFabricHandle fh;
      r = p_cuMemExportToShareableHandle(&fh, m->mc, CU_MEM_HANDLE_TYPE_FABRIC, 0);
      if (r != CUDA_SUCCESS) {
        HSF_DRV(cuMemRelease);
        p_cuMemRelease(m->mc);
        m->mc = 0;
        continue;
      }
      std::memcpy(handle64, &fh, sizeof(fh));
    }
    return m;
  }
  delete m;
  // (a single-GPU partition of an NVSwitch system reports multicast support
  // yet rejects every multicast object: scripts/probe/mcast_probe.py)
  if (r == CUDA_ERROR_INVALID_VALUE || r == CUDA_ERROR_NOT_SUPPORTED)
    fail(HSF_ERR_UNSUPPORTED, "cuMulticastCreate rejected the multicast object (no NVLS resources for this "
                              "process's GPUs)");
  cu(r, "cuMulticastCreate");
  return nullptr;
}

static Mcast* mcast_import(const void* handle64, size_t bytes, int nranks, int device) {
  HSF_DRV(cuMemImportFromShareableHandle);
  set_dev(device);
  auto* m = new Mcast();
  cudaGetDevice(&m->device);
  const size_t g = mc_granule(nranks, bytes, CU_MEM_HANDLE_TYPE_FABRIC);
  m->size = (bytes + g - 1) / g * g;
  CUmemFabricHandle fh;
  std::memcpy(&fh, handle64, sizeof(fh));
  try {
    cu(p_cuMemImportFromShareableHandle(&m->mc, &fh, CU_MEM_HANDLE_TYPE_FABRIC), "cuMemImportFromShareableHandle");
  } catch (...) {
    delete m;
    throw;
  }
  return m;
}

static void mcast_add_device(Mcast* m) {
  HSF_DRV(cuMulticastAddDevice);
  cu(p_cuMulticastAddDevice(m->mc, (CUdevice)m->device), "cuMulticastAddDevice");
}

// this rank's memory: allocate, bind to the multicast object, map both the
// local (unicast) and the multicast address
static void mcast_bind(Mcast* m) {
  HSF_DRV(cuMemCreate);
  HSF_DRV(cuMulticastBindMem);
  HSF_DRV(cuMemAddressReserve);
  HSF_DRV(cuMemMap);
  HSF_DRV(cuMemSetAccess);
  set_dev(m->device);
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = m->device;
  cu(p_cuMemCreate(&m->mem, m->size, &ap, 0), "cuMemCreate");
  cu(p_cuMulticastBindMem(m->mc, 0, m->mem, 0, m->size, 0), "cuMulticastBindMem");
  m->bound = true;
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = m->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  cu(p_cuMemAddressReserve(&m->local, m->size, m->size, 0, 0), "cuMemAddressReserve");
  cu(p_cuMemMap(m->local, m->size, 0, m->mem, 0), "cuMemMap (local)");
  m->mapped_local = true;
  cu(p_cuMemSetAccess(m->local, m->size, &acc, 1), "cuMemSetAccess (local)");
  cu(p_cuMemAddressReserve(&m->multi, m->size, m->size, 0, 0), "cuMemAddressReserve (multicast)");
  cu(p_cuMemMap(m->multi, m->size, 0, m->mc, 0), "cuMemMap (multicast)");
  m->mapped_mc = true;
  cu(p_cuMemSetAccess(m->multi, m->size, &acc, 1), "cuMemSetAccess (multicast)");
  if (cudaMemset((void*)(uintptr_t)m->local, 0, m->size) != cudaSuccess) fail(HSF_ERR_CUDA, "cudaMemset (multicast buffer)");
}

static void mcast_free(Mcast* m) {
  if (!m) return;
  try {
    HSF_DRV(cuMemUnmap);
    HSF_DRV(cuMemAddressFree);
    HSF_DRV(cuMemRelease);
    HSF_DRV(cuMulticastUnbind);
    cudaDeviceSynchronize();
    if (m->mapped_mc) p_cuMemUnmap(m->multi, m->size);
    if (m->multi) p_cuMemAddressFree(m->multi, m->size);
    if (m->mapped_local) p_cuMemUnmap(m->local, m->size);
    if (m->local) p_cuMemAddressFree(m->local, m->size);
    if (m->bound) p_cuMulticastUnbind(m->mc, (CUdevice)m->device, 0, m->size);
    if (m->mem) p_cuMemRelease(m->mem);
    if (m->mc) p_cuMemRelease(m->mc);
  } catch (...) {
  }
  delete m;
}

}  // namespace hsf

using namespace hsf;

#define MC_GUARD(...)                         \
  try {                                       \
    __VA_ARGS__;                              \
    return HSF_OK;                            \
  } catch (const Error& e) {                  \
    set_last_error(e.msg);                    \
    return e.st;                              \
  } catch (...) {                             \
    set_last_error("unknown C++ exception");  \
    return HSF_ERR_INVALID_ARG;               \
  }

extern "C" {

hsf_status hsf_mcast_create(size_t bytes, int32_t nranks, int32_t device, void* handle_out64, hsf_mcast_t** out) {
  MC_GUARD({
    if (!handle_out64 || !out || bytes == 0 || nranks < 1) fail(HSF_ERR_INVALID_ARG, "bad argument");
    *out = reinterpret_cast<hsf_mcast_t*>(mcast_create(bytes, nranks, device, handle_out64));
  })
}

hsf_status hsf_mcast_import(const void* handle64, size_t bytes, int32_t nranks, int32_t device, hsf_mcast_t** out) {
  MC_GUARD({
    if (!handle64 || !out || bytes == 0 || nranks < 1) fail(HSF_ERR_INVALID_ARG, "bad argument");
    *out = reinterpret_cast<hsf_mcast_t*>(mcast_import(handle64, bytes, nranks, device));
  })
}

hsf_status hsf_mcast_add_device(hsf_mcast_t* m) {
  MC_GUARD({
    if (!m) fail(HSF_ERR_INVALID_ARG, "NULL argument");
    mcast_add_device(reinterpret_cast<Mcast*>(m));
  })
}

hsf_status hsf_mcast_bind(hsf_mcast_t* m, void** local_out, void** multicast_out) {
  MC_GUARD({
    if (!m || !local_out || !multicast_out) fail(HSF_ERR_INVALID_ARG, "NULL argument");
    Mcast* mc = reinterpret_cast<Mcast*>(m);
    mcast_bind(mc);
    *local_out = (void*)(uintptr_t)mc->local;
    *multicast_out = (void*)(uintptr_t)mc->multi;
  })
}

void hsf_mcast_free(hsf_mcast_t* m) { mcast_free(reinterpret_cast<Mcast*>(m)); }

}  // extern "C"
