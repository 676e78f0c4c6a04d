// sum_kernels.cuh — Kronecker path-sum kernels:
//   psi[i_A * 2^nB + i_B] = sum_p c_p Psi_A[i_A, p] Psi_B[i_B, p]
//
//   K4t  transpose_fold : node-major leaves [K][2^m] -> row-major [2^m][K],
//                         optionally folding c_p (a3)
//   K6   gather_dot     : bitstring amplitudes (one warp per sample, two
//                         contiguous K-rows, warp-shuffle reduction)
//   K5s  simt_gemm      : full output on CUDA cores (fp32 / fp64 FMA),
//                         reading the node-major leaves directly
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "sim_kernels.cuh"

namespace hsf {

// ------------------------------------------------------------------ K4t
template <typename C>
__global__ void transpose_fold_kernel(const C* __restrict__ in, C* __restrict__ out, const C* __restrict__ cp,
                                      long long K, long long M) {
  __shared__ C tile[32][33];
  const long long m0 = (long long)blockIdx.x * 32, k0 = (long long)blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    long long k = k0 + r, m = m0 + tx;
    C v;
    v.x = 0;
    v.y = 0;
    if (k < K && m < M) {
      v = in[k * M + m];
      if (cp) v = cmul(v, cp[k]);
    }
    tile[r][tx] = v;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    long long m = m0 + r, k = k0 + tx;
    if (k < K && m < M) out[m * K + k] = tile[tx][r];
  }
}

// complex64 K4t with 16 B accesses: a 32 (k) x 64 (m) tile per CTA, loads of
// two consecutive m per thread (512 B per warp row), stores of two
// consecutive k per thread (256 B per output row). SMEM [m][16 slots][2]:
// the (k, k+1) pair of row m sits in slot (k / 2) ^ ((m / 2) & 15), so both
// the load-side 8 B writes and the store-side 16 B reads run at the minimum
// wavefront count.
__global__ void transpose_fold_c64_kernel(const float2* __restrict__ in, float2* __restrict__ out,
                                          const float2* __restrict__ cp, long long K, long long M) {
  __shared__ __align__(16) float2 S[64][32];
  const long long m0 = (long long)blockIdx.x * 64, k0 = (long long)blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = ty + 8 * i;  // k offset
    const long long k = k0 + r, m = m0 + 2 * tx;
    float2 v0 = make_float2(0.f, 0.f), v1 = v0;
    if (k < K) {
      if (m + 1 < M) {
        const float4 a = *reinterpret_cast<const float4*>(in + k * M + m);
        v0 = make_float2(a.x, a.y);
        v1 = make_float2(a.z, a.w);
      } else if (m < M) {
        v0 = in[k * M + m];
      }
      if (cp) {
        const float2 c = cp[k];
        v0 = cmul(v0, c);
        v1 = cmul(v1, c);
      }
    }
    const int slot = (r >> 1) ^ (tx & 15);  // rows 2tx, 2tx+1: (m / 2) & 15 = tx & 15
    S[2 * tx][2 * slot + (r & 1)] = v0;
    S[2 * tx + 1][2 * slot + (r & 1)] = v1;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int mr = 16 * i + 2 * ty + (tx >> 4), kp = tx & 15;
    const long long m = m0 + mr, k = k0 + 2 * kp;
    const float4 v = *reinterpret_cast<const float4*>(&S[mr][2 * (kp ^ ((mr >> 1) & 15))]);
    if (m < M) {
      if (k + 1 < K && (K & 1) == 0)
        *reinterpret_cast<float4*>(out + m * K + k) = v;
      else {
        if (k < K) out[m * K + k] = make_float2(v.x, v.y);
        if (k + 1 < K) out[m * K + k + 1] = make_float2(v.z, v.w);
      }
    }
  }
}

// --------------------------------------------- qubit relabelling (partitions)
// caller index <-> internal index for a non-contiguous partition: bit q of the
// caller's index is bit relabel[q] of the internal one.  tab[16*k .. ] holds,
// for each 16-bit chunk k of the source index, the mapped bits (4 x 2^16).
__device__ __forceinline__ unsigned long long permute_index(unsigned long long x,
                                                            const unsigned long long* __restrict__ tab) {
  return __ldg(&tab[x & 0xFFFFull]) | __ldg(&tab[65536 + ((x >> 16) & 0xFFFFull)]) |
         __ldg(&tab[131072 + ((x >> 32) & 0xFFFFull)]) | __ldg(&tab[196608 + (x >> 48)]);
}

__global__ void permute_bits_kernel(const unsigned long long* __restrict__ in, unsigned long long* __restrict__ out,
                                    long long n, const unsigned long long* __restrict__ tab) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = permute_index(in[i], tab);
}

// out[j] (caller order) = in[map(j)] (internal order), or += with accumulate
template <typename C>
__global__ void permute_out_kernel(const C* __restrict__ in, C* __restrict__ out, long long n,
                                   const unsigned long long* __restrict__ tab, int accumulate) {
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    C v = in[permute_index((unsigned long long)j, tab)];
    if (accumulate) {
      v.x += out[j].x;
      v.y += out[j].y;
    }
    out[j] = v;
  }
}

// ------------------------------------------------------------------- K6
// Folded trailing diagonal units: amp(s) *= prod_u D_u[s's bits on supp(u)]
// (block-local index, LSB = smallest support qubit; see plan.cpp).
struct TrailParams {
  int n;                               // folded units (0 => weight 1)
  unsigned long long mask[kMaxTrail];  // global support bits of unit u
  long long off[kMaxTrail];            // offset of D_u in the table
};

template <typename C>
__device__ __forceinline__ C trail_weight(const TrailParams& tw, const C* __restrict__ tab, unsigned long long s) {
  C w;
  w.x = 1;
  w.y = 0;
  for (int u = 0; u < tw.n; ++u) {
    unsigned long long m = tw.mask[u];
    uint32_t idx = 0;
    for (int j = 0; m; ++j, m &= m - 1) idx |= (uint32_t)((s >> (__ffsll((long long)m) - 1)) & 1ull) << j;
    w = cmul(w, __ldg(&tab[tw.off[u] + idx]));
  }
  return w;
}

// amp[s] = sum_p AT[s >> nB][p] * BT[s & maskB][p]   (AT already holds c_p)
template <typename C>
__global__ void gather_dot_kernel(const C* __restrict__ AT, const C* __restrict__ BT,
                                  const unsigned long long* __restrict__ bits, C* __restrict__ out,
                                  long long n_samples, long long K, int n_low, const TrailParams tw,
                                  const C* __restrict__ trail, int accumulate) {
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const unsigned long long maskB = (1ull << n_low) - 1ull;
  for (long long s = warp; s < n_samples; s += nwarps) {
    unsigned long long b = bits[s];
    const C* a = AT + (long long)(b >> n_low) * K;
    const C* bb = BT + (long long)(b & maskB) * K;
    C acc;
    acc.x = 0;
    acc.y = 0;
    for (long long p = lane; p < K; p += 32) acc = cfma(__ldg(&a[p]), __ldg(&bb[p]), acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if (lane == 0) {
      C r = tw.n ? cmul(acc, trail_weight(tw, trail, b)) : acc;
      if (accumulate) {
        r.x += out[s].x;
        r.y += out[s].y;
      }
      out[s] = r;
    }
  }
}

// Specialisation for K % 64 == 0 with complex64: 16 B loads, 2 complex per lane
// per step, 4 steps in flight.
__global__ void gather_dot_c64_vec_kernel(const float4* __restrict__ AT, const float4* __restrict__ BT,
                                          const unsigned long long* __restrict__ bits, float2* __restrict__ out,
                                          long long n_samples, long long K, int n_low, const TrailParams tw,
                                          const float2* __restrict__ trail, int accumulate) {
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const unsigned long long maskB = (1ull << n_low) - 1ull;
  const long long K2 = K >> 1;  // float4 per row
  for (long long s = warp; s < n_samples; s += nwarps) {
    unsigned long long b = bits[s];
    const float4* a = AT + (long long)(b >> n_low) * K2;
    const float4* bb = BT + (long long)(b & maskB) * K2;
    float re = 0.f, im = 0.f;
    for (long long p = lane; p < K2; p += 32) {
      float4 x = __ldg(&a[p]);
      float4 y = __ldg(&bb[p]);
      re = fmaf(x.x, y.x, fmaf(-x.y, y.y, re));
      im = fmaf(x.x, y.y, fmaf(x.y, y.x, im));
      re = fmaf(x.z, y.z, fmaf(-x.w, y.w, re));
      im = fmaf(x.z, y.w, fmaf(x.w, y.z, im));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      re += __shfl_xor_sync(0xffffffffu, re, o);
      im += __shfl_xor_sync(0xffffffffu, im, o);
    }
    if (lane == 0) {
      const float2 a = make_float2(re, im);
      float2 r = tw.n ? cmul(a, trail_weight(tw, trail, b)) : a;
      if (accumulate) {
        r.x += out[s].x;
        r.y += out[s].y;
      }
      out[s] = r;
    }
  }
}

// ------------------------------------------------------ K6, grouped by A row
// When many samples share an A row (c3: 2^20 samples over 2^15 rows, ~32 per
// row; both operands L2-resident, so the plain gather is bound by L2->SM
// traffic), the samples are bucketed by A row (counting sort: count, one-CTA
// scan, scatter of sample indices) and one warp per row keeps the row in
// registers while it streams its samples' B rows: A traffic drops from one
// row per sample to one row per distinct row.
__global__ void bucket_count_kernel(const unsigned long long* __restrict__ bits, long long n, int n_low,
                                    int* __restrict__ counts) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    atomicAdd(&counts[bits[i] >> n_low], 1);
}

// exclusive scan of counts[0..n) into offs[0..n] (offs[n] = total) and
// cursor[0..n); one CTA of 1024 threads: warp w owns a contiguous span, read
// in coalesced 32-element chunks with shuffle scans (a per-thread sequential
// span made every load its own L2 round trip: 80 us for c3's 2^15 rows)
__global__ void __launch_bounds__(1024) bucket_scan_kernel(const int* __restrict__ counts, int* __restrict__ offs,
                                                           int* __restrict__ cursor, long long n) {
  __shared__ int wsum[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long span = (n + 31) / 32, b = w * span, e = min(n, b + span);
  int tot = 0;  // pass 1: this warp's total (8 chunks of loads in flight)
  for (long long c0 = b; c0 < e; c0 += 256) {
    int v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = c0 + 32 * k + lane < e ? counts[c0 + 32 * k + lane] : 0;
    int sum = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) sum += v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    tot += sum;
  }
  if (lane == 0) wsum[w] = tot;
  __syncthreads();
  if (w == 0) {  // exclusive scan of the 32 warp totals
    const int x = wsum[lane];
    int inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    wsum[lane] = inc - x;
    if (lane == 31) offs[n] = inc;
  }
  __syncthreads();
  int run = wsum[w];  // pass 2: scan each chunk, carry the running total
  for (long long c0 = b; c0 < e; c0 += 256) {
    int v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = c0 + 32 * k + lane < e ? counts[c0 + 32 * k + lane] : 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const long long c = c0 + 32 * k;
      const int x = v[k];
      int inc = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (c + lane < e) {
        offs[c + lane] = run + inc - x;
        cursor[c + lane] = run + inc - x;
      }
      run += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
}

__global__ void bucket_scatter_kernel(const unsigned long long* __restrict__ bits, long long n, int n_low,
                                      int* __restrict__ cursor, int* __restrict__ perm) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    perm[atomicAdd(&cursor[bits[i] >> n_low], 1)] = (int)i;
}

// one warp per A row r: the row (T float4 per lane, K = 64*T complex) stays in
// registers; the row's samples are taken two at a time (both B rows in flight)
template <int T>
__global__ void gather_grouped_c64_kernel(const float4* __restrict__ AT, const float4* __restrict__ BT,
                                          const unsigned long long* __restrict__ bits, const int* __restrict__ offs,
                                          const int* __restrict__ perm, float2* __restrict__ out, long long n_rows,
                                          int n_low, const TrailParams tw, const float2* __restrict__ trail,
                                          int accumulate) {
  constexpr int K2 = 32 * T;  // float4 per operand row
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const unsigned long long maskB = (1ull << n_low) - 1ull;
  for (long long r = warp; r < n_rows; r += nwarps) {
    const int beg = offs[r], end = offs[r + 1];
    if (beg == end) continue;
    float4 a[T];
#pragma unroll
    for (int t = 0; t < T; ++t) a[t] = __ldg(&AT[r * K2 + lane + 32 * t]);
    // the row's sample indices and bitstrings, up to 32 at a time, loaded by
    // the lanes in parallel and broadcast (no dependent perm -> bits -> B
    // chain per sample pair)
    for (int jb = beg; jb < end; jb += 32) {
    const int nb = end - jb < 32 ? end - jb : 32;
    int pl = 0;
    unsigned long long bl = 0;
    if (lane < nb) {
      pl = perm[jb + lane];
      bl = bits[pl];
    }
    // 4 samples per step: 4 B rows in flight per warp
    for (int jj = 0; jj < nb; jj += 4) {
      int ii[4];
      unsigned long long bb[4];
      float4 y[4][T];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int src = jj + u < nb ? jj + u : jj;  // warp-uniform
        ii[u] = __shfl_sync(0xffffffffu, pl, src);
        bb[u] = __shfl_sync(0xffffffffu, bl, src);
        const float4* q = BT + (long long)(bb[u] & maskB) * K2;
#pragma unroll
        for (int t = 0; t < T; ++t) y[u][t] = __ldg(&q[lane + 32 * t]);
      }
      float re[4], im[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        re[u] = 0.f;
        im[u] = 0.f;
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const float4 x = a[t];
          re[u] = fmaf(x.x, y[u][t].x, fmaf(-x.y, y[u][t].y, re[u]));
          im[u] = fmaf(x.x, y[u][t].y, fmaf(x.y, y[u][t].x, im[u]));
          re[u] = fmaf(x.z, y[u][t].z, fmaf(-x.w, y[u][t].w, re[u]));
          im[u] = fmaf(x.z, y[u][t].w, fmaf(x.w, y[u][t].z, im[u]));
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          re[u] += __shfl_xor_sync(0xffffffffu, re[u], o);
          im[u] += __shfl_xor_sync(0xffffffffu, im[u], o);
        }
      const int nv = nb - jj < 4 ? nb - jj : 4;
      if (lane < nv) {  // lane u writes sample jj + u
        int idx = ii[0];
        unsigned long long bs = bb[0];
        float2 v = make_float2(re[0], im[0]);
#pragma unroll
        for (int u = 1; u < 4; ++u)
          if (lane == u) {
            idx = ii[u];
            bs = bb[u];
            v = make_float2(re[u], im[u]);
          }
        float2 res = tw.n ? cmul(v, trail_weight(tw, trail, bs)) : v;
        if (accumulate) {
          res.x += out[idx].x;
          res.y += out[idx].y;
        }
        out[idx] = res;
      }
    }
    }
  }
}

// Swapped path-sum (prefix outputs): the GEMM wrote outT[j][i] (j < MB
// columns of half B, i < rows of half A); out[i][j] = outT[j][i] (+= out).
// 32 x 32 tiles through SMEM, coalesced on both sides.
__global__ void swap_transpose_kernel(const float2* __restrict__ outT, float2* __restrict__ out, long long rows,
                                      long long MB, long long ldT, int accumulate) {
  __shared__ float2 t[32][33];
  const long long j0 = (long long)blockIdx.x * 32, i0 = (long long)blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    const long long j = j0 + r, i = i0 + tx;
    t[r][tx] = (j < MB && i < rows) ? outT[j * ldT + i] : make_float2(0.f, 0.f);
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const long long i = i0 + r, j = j0 + tx;
    if (i < rows && j < MB) {
      float2 v = t[tx][r];
      if (accumulate) {
        const float2 o = out[i * MB + j];
        v.x += o.x;
        v.y += o.y;
      }
      out[i * MB + j] = v;
    }
  }
}

// ------------------------------------------------------------------ K5s
// out[(i - row0) * MB + j] = sum_p c_p A[p][i] B[p][j]  for i in [row0, row0+rows)
// A: [K][MA] node-major leaves, B: [K][MB].  64x64 output tile per CTA,
// 256 threads x (4x4) outputs, K staged in chunks of 16 through SMEM.
template <typename C, typename R>
__global__ void __launch_bounds__(256) simt_gemm_kernel(const C* __restrict__ A, const C* __restrict__ B,
                                                        const C* __restrict__ cp, C* __restrict__ out,
                                                        long long K, long long MA, long long MB, long long row0,
                                                        long long rows, int accumulate) {
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ C As[BK][BM];
  __shared__ C Bs[BK][BN];
  const int tid = threadIdx.x;
  const int tr = tid / 16, tc = tid % 16;  // 16 x 16 threads, each 4 x 4
  const long long i0 = row0 + (long long)blockIdx.y * BM;
  const long long j0 = (long long)blockIdx.x * BN;
  C acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      acc[a][b].x = 0;
      acc[a][b].y = 0;
    }
  for (long long k0 = 0; k0 < K; k0 += BK) {
    for (int e = tid; e < BK * BM; e += 256) {
      int kk = e / BM, ii = e % BM;
      long long k = k0 + kk, i = i0 + ii;
      C v;
      v.x = 0;
      v.y = 0;
      if (k < K && i < row0 + rows && i < MA) v = cmul(A[k * MA + i], cp[k]);
      As[kk][ii] = v;
    }
    for (int e = tid; e < BK * BN; e += 256) {
      int kk = e / BN, jj = e % BN;
      long long k = k0 + kk, j = j0 + jj;
      C v;
      v.x = 0;
      v.y = 0;
      if (k < K && j < MB) v = B[k * MB + j];
      Bs[kk][jj] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      C a[4], b[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) a[x] = As[kk][tr + 16 * x];
#pragma unroll
      for (int y = 0; y < 4; ++y) b[y] = Bs[kk][tc + 16 * y];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = cfma(a[x], b[y], acc[x][y]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    long long i = i0 + tr + 16 * x;
    if (i >= row0 + rows || i >= MA) continue;
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      long long j = j0 + tc + 16 * y;
      if (j < MB) {
        C r = acc[x][y];
        if (accumulate) {
          r.x += out[(i - row0) * MB + j].x;
          r.y += out[(i - row0) * MB + j].y;
        }
        out[(i - row0) * MB + j] = r;
      }
    }
  }
}

}  // namespace hsf
