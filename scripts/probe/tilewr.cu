// c4 output-pattern probe: fp32 [2^14][2^18] (16 GiB) written tile by tile
// (256 x 256 tiles, grouped raster of 16 row blocks as the c4 GEMM) with
// 32-row x 32-column boxes (128 B per row, the GEMM epilogue's TMA box) vs
// 8-row x 256-column boxes (1 KB per row) vs a linear grid-stride write.
#include <cuda_runtime.h>
#include <cstdio>
constexpr int R = 1 << 14, C = 1 << 18, TM = 256, TN = 256;
__global__ void tiles(float* p, int box_cols, int group_m, int col_fastest) {
  const int nm = R / TM, nn = C / TN, ntiles = nm * nn;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int mb, nb;
    if (group_m) { const int g = t / (group_m * nn), r = t % (group_m * nn); mb = g * group_m + r % group_m; nb = r / group_m; }
    else { mb = t % nm; nb = t / nm; }
    const int box_rows = 1024 / box_cols;  // 4 KB boxes
    const int nbox = (TM / box_rows) * (TN / box_cols);
    for (int b = warp; b < nbox; b += nw) {
      const int br = col_fastest ? b / (TN / box_cols) : b % (TM / box_rows);
      const int bc = col_fastest ? b % (TN / box_cols) : b / (TM / box_rows);
      // each lane writes 16 B; a warp instruction covers 512 B = box_cols*4 B rows
      const int lanes_per_row = box_cols / 4;
      for (int k = lane; k < box_rows * lanes_per_row; k += 32) {
        const int rr = k / lanes_per_row, cc = (k % lanes_per_row) * 4;
        const size_t row = (size_t)mb * TM + br * box_rows + rr, col = (size_t)nb * TN + bc * box_cols + cc;
        __stcs(reinterpret_cast<float4*>(p + row * C + col), make_float4(1.f + k, 2.f + t, 3.f + b, 4.f));
      }
    }
  }
}
// the GEMM epilogue's order: each CTA = 128 rows of a pair tile (2 CTAs per
// tile), warp (q = w % 4, h = w / 4) writes 32-row band q, chunks h, h+G, ...
__global__ void gemmlike(float* p, int G) {
  const int nm = R / TM, nn = C / TN, ntiles = nm * nn, group_m = 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, h = warp >> 2;
  const int rank = blockIdx.x & 1;
  for (int t = blockIdx.x >> 1; t < ntiles; t += gridDim.x >> 1) {
    const int g = t / (group_m * nn), r = t % (group_m * nn);
    const int mb = g * group_m + r % group_m, nb = r / group_m;
    for (int c = h; c < TN / 32; c += G) {
      for (int k = lane; k < 32 * 8; k += 32) {
        const int rr = k / 8, cc = (k % 8) * 4;
        const size_t row = (size_t)mb * TM + rank * 128 + q * 32 + rr, col = (size_t)nb * TN + c * 32 + cc;
        __stcs(reinterpret_cast<float4*>(p + row * C + col), make_float4(1.f + k, 2.f + t, 3.f + c, 4.f));
      }
    }
  }
}
__global__ void lin(float4* p, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(&p[i], make_float4(1.f + i, 2.f, 3.f, 4.f));
}
int main() {
  const size_t bytes = (size_t)R * C * 4;
  float* p; cudaMalloc(&p, bytes);
  cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
  auto run = [&](const char* name, auto f) {
    f(); cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 4; ++r) { cudaEventRecord(s); f(); cudaEventRecord(e); cudaEventSynchronize(e);
      float ms; cudaEventElapsedTime(&ms, s, e); if (ms < best) best = ms; }
    printf("%-44s %.3f ms = %.2f TB/s\n", name, best, bytes / best / 1e9);
  };
  run("linear grid-stride", [&] { lin<<<148 * 8, 512>>>((float4*)p, bytes / 16); });
  run("tiles, 32x32 boxes, grouped 16", [&] { tiles<<<148, 256>>>(p, 32, 16, 0); });
  run("tiles, 32x32 boxes, grouped 16, col-fastest", [&] { tiles<<<148, 256>>>(p, 32, 16, 1); });
  run("tiles, 32x32 boxes, grouped 16, 2 CTA/SM", [&] { tiles<<<296, 256>>>(p, 32, 16, 0); });
  run("tiles, 4x256 boxes (1 KB rows), grouped 16", [&] { tiles<<<148, 256>>>(p, 256, 16, 0); });
  run("tiles, 32x32 boxes, M-fastest", [&] { tiles<<<148, 256>>>(p, 32, 0, 0); });
  run("tiles, 32x32 boxes, M-fastest, col-fastest", [&] { tiles<<<148, 256>>>(p, 32, 0, 1); });
  run("tiles, 4x256 boxes, M-fastest", [&] { tiles<<<148, 256>>>(p, 256, 0, 0); });
  run("gemm-like, G=2 (8 warps)", [&] { gemmlike<<<148, 256>>>(p, 2); });
  run("gemm-like, G=4 (16 warps)", [&] { gemmlike<<<148, 512>>>(p, 4); });
  run("gemm-like, G=8 (32 warps)", [&] { gemmlike<<<148, 1024>>>(p, 8); });
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
