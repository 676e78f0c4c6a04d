// HBM write bandwidth: constant vs incompressible (hashed) data, 16 GiB,
// float4 stores, grid-stride; context for c4's output-write roofline.
#include <cuda_runtime.h>
#include <cstdio>
__device__ __forceinline__ unsigned hsh(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__global__ void wr(float4* p, size_t n, int mode, unsigned salt) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 v;
    if (mode == 0) v = make_float4(1.f, 1.f, 1.f, 1.f);
    else {
      unsigned h = hsh((unsigned)i ^ salt);
      v = make_float4(__uint_as_float(0x3f800000u | (h & 0x7fffff)), __uint_as_float(0x3f800000u | (hsh(h) & 0x7fffff)),
                      __uint_as_float(0x3f800000u | (hsh(h + 1) & 0x7fffff)), __uint_as_float(0x3f800000u | (hsh(h + 2) & 0x7fffff)));
    }
    __stcs(&p[i], v);
  }
}
int main() {
  size_t bytes = (size_t)16 << 30, n = bytes / 16;
  float4* p; cudaMalloc(&p, bytes);
  cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
  for (int mode = 0; mode < 2; ++mode) {
    wr<<<148 * 8, 512>>>(p, n, mode, 1);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(s); wr<<<148 * 8, 512>>>(p, n, mode, 7 + r); cudaEventRecord(e); cudaEventSynchronize(e);
      float ms; cudaEventElapsedTime(&ms, s, e); if (ms < best) best = ms;
    }
    printf("write 16 GiB %s: %.3f ms = %.2f TB/s\n", mode ? "hashed (incompressible)" : "constant", best, bytes / best / 1e9);
  }
  return 0;
}
