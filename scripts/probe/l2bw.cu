// L2-resident read bandwidth probe: every CTA streams a 32 MiB buffer
// (L2-resident after the first pass) with 16 B loads, `reps` times.
#include <cuda_runtime.h>
#include <cstdio>
__global__ void l2read(const uint4* __restrict__ buf, size_t n16, int reps, unsigned* out) {
  unsigned acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x + (size_t)r * 977; i < n16 + (size_t)r * 977; i += stride) {
      const uint4 v = __ldcg(&buf[i % n16]);
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  if (acc == 0x12345678u) out[0] = acc;
}
int main() {
  for (size_t mb : {16, 32, 64}) {
    size_t bytes = mb << 20, n16 = bytes / 16;
    uint4* b; unsigned* o;
    cudaMalloc(&b, bytes); cudaMalloc(&o, 4);
    cudaMemset(b, 1, bytes);
    int reps = 20;
    l2read<<<148 * 4, 512>>>(b, n16, 2, o);
    cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
    cudaEventRecord(s);
    l2read<<<148 * 4, 512>>>(b, n16, reps, o);
    cudaEventRecord(e); cudaEventSynchronize(e);
    float ms; cudaEventElapsedTime(&ms, s, e);
    printf("L2 read %zu MiB x %d: %.3f ms = %.2f TB/s\n", mb, reps, ms, (double)bytes * reps / ms / 1e9);
    cudaFree(b); cudaFree(o);
  }
  return 0;
}
