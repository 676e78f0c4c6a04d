// Random-row gather bandwidth on the box (the bitstring path-sum's access
// pattern): rows of R bytes at uniformly random row indices of a 2 GiB
// buffer, one warp per row, 16 B per lane per load, U rows in flight per warp,
// summed into one float per warp (no write traffic).  Prints GB/s of row
// bytes read for R = 256 B .. 4 KiB and U = 1, 2, 4, 8.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a rowgather.cu -o rowgather
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

template <int U>
__global__ void gather_rows(const float4* __restrict__ buf, const uint32_t* __restrict__ idx, long long n_rows,
                            int r16, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  for (long long s = w * U; s < n_rows; s += nw * U) {
    float4 v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long r = s + u < n_rows ? idx[s + u] : idx[s];
#pragma unroll
      for (int t = 0; t < 8; ++t)
        v[u][t] = (lane + 32 * t < r16) ? __ldg(&buf[r * r16 + lane + 32 * t]) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int t = 0; t < 8; ++t) acc += v[u][t].x + v[u][t].y + v[u][t].z + v[u][t].w;
  }
  if (acc == 12345.f) out[w] = acc;
}

int main() {
  const size_t bytes = 2ull << 30;
  float4* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  float* out;
  cudaMalloc(&out, 1 << 24);
  const long long n_samples = 1 << 22;
  uint32_t* idx;
  cudaMalloc(&idx, n_samples * 4);
  std::mt19937_64 rng(1);
  for (int R : {256, 512, 1024, 2048, 4096}) {
    const long long rows = bytes / R;
    std::vector<uint32_t> h(n_samples);
    for (auto& x : h) x = (uint32_t)(rng() % rows);
    cudaMemcpy(idx, h.data(), n_samples * 4, cudaMemcpyHostToDevice);
    const long long ns = R >= 2048 ? n_samples / (R / 1024) : n_samples;
    for (int U : {1, 2, 4, 8}) {
      auto run = [&]() {
        const int grid = 148 * 8;
        if (U == 1) gather_rows<1><<<grid, 256>>>(buf, idx, ns, R / 16, out);
        if (U == 2) gather_rows<2><<<grid, 256>>>(buf, idx, ns, R / 16, out);
        if (U == 4) gather_rows<4><<<grid, 256>>>(buf, idx, ns, R / 16, out);
        if (U == 8) gather_rows<8><<<grid, 256>>>(buf, idx, ns, R / 16, out);
      };
      run();
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      float best = 1e9;
      for (int i = 0; i < 5; ++i) {
        cudaEventRecord(a);
        run();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
      }
      printf("row %5d B, %d rows in flight per warp: %7.1f GB/s (%.3f ms)\n", R, U, ns * (double)R / best / 1e6, best);
    }
  }
  return 0;
}
