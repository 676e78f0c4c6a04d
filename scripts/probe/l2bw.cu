// L2-resident read bandwidth: every CTA streams slices of a 32 MiB buffer
// (L2-resident after the first pass) with 16 B __ldcg loads, 8 in flight per
// thread; context for roofline numbers of L2-resident kernels (c3's gather).
#include <cuda_runtime.h>
#include <cstdio>
__global__ void l2read(const uint4* __restrict__ buf, unsigned n16, int reps, unsigned* out) {
  unsigned acc = 0;
  const unsigned stride = gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    unsigned i = (blockIdx.x * blockDim.x + threadIdx.x + (unsigned)r * 4099u * 16u) & (n16 - 1);
#pragma unroll 8
    for (unsigned k = 0; k < n16 / stride; ++k) {
      const uint4 v = __ldcg(&buf[i]);
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
      i = (i + stride) & (n16 - 1);
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}
int main() {
  for (size_t mb : {16, 32, 64}) {
    size_t bytes = mb << 20;
    unsigned n16 = (unsigned)(bytes / 16);
    uint4* b; unsigned* o;
    cudaMalloc(&b, bytes); cudaMalloc(&o, 4);
    cudaMemset(b, 1, bytes);
    const int reps = 40;
    l2read<<<148 * 4, 512>>>(b, n16, 2, o);
    cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
    float best = 1e9;
    for (int t = 0; t < 3; ++t) {
      cudaEventRecord(s);
      l2read<<<148 * 4, 512>>>(b, n16, reps, o);
      cudaEventRecord(e); cudaEventSynchronize(e);
      float ms; cudaEventElapsedTime(&ms, s, e); if (ms < best) best = ms;
    }
    printf("L2 read %zu MiB x %d: %.3f ms = %.2f TB/s\n", mb, reps, best, (double)bytes * reps / best / 1e9);
    cudaFree(b); cudaFree(o);
  }
  return 0;
}
