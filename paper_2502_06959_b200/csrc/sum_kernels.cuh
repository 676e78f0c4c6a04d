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
// ldo: output row stride (>= K); columns [K, ldo) of rows < M are written as
// zeros when the grid spans them (gridDim.y = ldo / 32, the block gather's
// power-of-two padded rows).
__global__ void transpose_fold_c64_kernel(const float2* __restrict__ in, float2* __restrict__ out,
                                          const float2* __restrict__ cp, long long K, long long M, long long ldo) {
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
      if (k + 1 < ldo && (ldo & 1) == 0)
        *reinterpret_cast<float4*>(out + m * ldo + k) = v;
      else {
        if (k < ldo) out[m * ldo + k] = make_float2(v.x, v.y);
        if (k + 1 < ldo) out[m * ldo + k + 1] = make_float2(v.z, v.w);
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
    const int lo = __ffsll((long long)m) - 1;
    if ((((m >> lo) + 1ull) & (m >> lo)) == 0ull) {  // contiguous bits: one shift and mask
      idx = (uint32_t)((s >> lo) & (m >> lo));
    } else {
      for (int j = 0; m; ++j, m &= m - 1) idx |= (uint32_t)((s >> (__ffsll((long long)m) - 1)) & 1ull) << j;
    }
    w = cmul(w, __ldg(&tab[tw.off[u] + idx]));
  }
  return w;
}

// amp[s] = sum_p AT[s >> nB][p] * BT[s & maskB][p]   (AT already holds c_p)
template <typename C>
__global__ void gather_dot_kernel(const C* __restrict__ AT, const C* __restrict__ BT,
                                  const unsigned long long* __restrict__ bits, C* __restrict__ out,
                                  long long n_samples, long long K, int n_low, const TrailParams tw,
                                  const C* __restrict__ trail, int accumulate, unsigned long long maskA) {
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const unsigned long long maskB = (1ull << n_low) - 1ull;
  for (long long s = warp; s < n_samples; s += nwarps) {
    unsigned long long b = bits[s];
    const C* a = AT + (long long)((b >> n_low) & maskA) * K;
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
                                          const float2* __restrict__ trail, int accumulate,
                                          unsigned long long maskA) {
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const unsigned long long maskB = (1ull << n_low) - 1ull;
  const long long K2 = K >> 1;  // float4 per row
  for (long long s = warp; s < n_samples; s += nwarps) {
    unsigned long long b = bits[s];
    const float4* a = AT + (long long)((b >> n_low) & maskA) * K2;
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

// Samples with bits at or above n violate hsf_run's precondition: flag them
// (word in mapped host memory, read when the run synchronises).  Every gather
// masks its row indices, so such a sample never reads out of bounds.
__global__ void check_bits_kernel(const unsigned long long* __restrict__ bits, long long n, int n_qubits,
                                  unsigned int* __restrict__ flag) {
  unsigned long long acc = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    acc |= bits[i];
  if (n_qubits < 64 && __any_sync(0xffffffffu, (acc >> n_qubits) != 0ull) && (threadIdx.x & 31) == 0)
    atomicOr(flag, 1u);
}

// ------------------------------------------------------- K6b, block gather
// The bitstring path-sum amp[s] = sum_p A'[iA(s)][p] B[iB(s)][p] (a3
// folded into A') reads one side -- the "direct" half D, whose path tree
// finishes last -- straight from its node-major leaves [K][2^mD]: the samples
// are bucketed by the 32-row block of their D row (counting sort: count, one
// CTA scan, scatter of sample indices), one CTA per block stages the block's
// 32 x K amplitudes in shared memory (K-row segments of 256 B, coalesced),
// and each sample then reads only its row of the other half, transposed to
// [2^mT][Kp] (Kp = K padded to 2*G*NF with zeros).  D needs no transpose, so
// the kernel follows D's last simulator pass directly; traffic = D's leaves
// once + one Kp row of T per sample.
// Counting sort of the samples by block, aggregated per CTA: each CTA takes a
// contiguous chunk of the samples and histograms it in shared memory (shared
// atomics), then adds its non-zero bucket counts to the global counts -- one
// global atomic per (CTA, bucket) instead of one per sample (c3's 1024
// buckets hold ~1000 samples each: per-sample atomics serialised at L2).
__global__ void __launch_bounds__(1024) bucket_count_kernel(const unsigned long long* __restrict__ bits, long long n,
                                                            int shift, unsigned long long kmask, int nbk,
                                                            int* __restrict__ counts) {
  extern __shared__ int h[];
  for (int i = threadIdx.x; i < nbk; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const long long c0 = n * blockIdx.x / gridDim.x, c1 = n * (blockIdx.x + 1) / gridDim.x;
  for (long long i = c0 + threadIdx.x; i < c1; i += blockDim.x) atomicAdd(&h[(bits[i] >> shift) & kmask], 1);
  __syncthreads();
  for (int i = threadIdx.x; i < nbk; i += blockDim.x)
    if (h[i]) atomicAdd(&counts[i], h[i]);
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

// scatter of the samples into block order (same chunks as the count): each
// CTA reserves its range in every bucket it touches (one global atomic per
// (CTA, bucket)), then places its samples with shared atomics; sidx[pos] =
// sample index, sbits[pos] = its bitstring (the gather reads both coalesced,
// no dependent lookup).  Order within a bucket is unspecified.
__global__ void __launch_bounds__(1024) bucket_scatter_kernel(const unsigned long long* __restrict__ bits, long long n,
                                                              int shift, unsigned long long kmask, int nbk,
                                                              int* __restrict__ cursor, int* __restrict__ sidx,
                                                              unsigned long long* __restrict__ sbits) {
  extern __shared__ int h[];
  for (int i = threadIdx.x; i < nbk; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const long long c0 = n * blockIdx.x / gridDim.x, c1 = n * (blockIdx.x + 1) / gridDim.x;
  for (long long i = c0 + threadIdx.x; i < c1; i += blockDim.x) atomicAdd(&h[(bits[i] >> shift) & kmask], 1);
  __syncthreads();
  for (int i = threadIdx.x; i < nbk; i += blockDim.x)
    if (h[i]) h[i] = atomicAdd(&cursor[i], h[i]);
  __syncthreads();
  for (long long i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
    const unsigned long long b = bits[i];
    const int pos = atomicAdd(&h[(b >> shift) & kmask], 1);
    sidx[pos] = (int)i;
    sbits[pos] = b;
  }
}


struct BlockGatherParams {
  const float2* D;       // direct half's leaves [K][ldD]
  long long ldD;         // 2^mD
  long long K;           // paths (rows of D; columns of T below Kp are these)
  const float2* cpD;     // c_p of the direct half when it is A (else nullptr)
  const float4* T;       // other half, [2^mT][Kp] complex64 (Kp / 2 float4 per row)
  const int* offs;       // [n_blocks + 1] sample offsets per block
  const int* sidx;       // sample indices in block order
  const unsigned long long* sbits;  // their bitstrings
  float2* out;
  long long n_blocks;
  int n_low;             // n_B
  int direct_b;          // 1: D = half B (index bits & maskB), 0: D = half A (index bits >> n_B)
  unsigned long long maskA, maskB;
  int accumulate;
  int debug;             // tuning only: 1 skips the staging, 2 skips the samples
  // owner-sharded output (fused exchange, hsf_run_args.out_shards): sample s
  // is reduce-added (vector red.add) into shard[s / shard_len][s % shard_len]
  // -- device or peer (NVLink / CUDA IPC) memory; n_shards == 0: plain out
  float2* shard[8];
  long long shard_len;
  int n_shards;
  int multicast;  // shard[0] is an NVLS multicast address: multimem.red into every rank's copy
  int ldmode;     // T-row load flavour (ld_row)
  // the direct half's deferred final diagonal (DeferOut), applied per staged
  // row: factor(row) = prod_r dtab[doff[r] + ((row >> dlo[r]) & dmask[r])]
  const float2* dtab;
  int dnr;
  int dlo[4];
  unsigned dmask[4];
  long long doff[4];
};

// a T-row chunk: 0 = ld.global.nc (L1 allocate), 1 = ld.global.cg (L2 only),
// 2 = ld.global.nc.L1::no_allocate.L2::256B
__device__ __forceinline__ float4 ld_row(const float4* a, int mode) {
  float4 v;
  if (mode == 1) {
    v = __ldcg(a);
  } else if (mode == 2) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(a));
  } else {
    v = __ldg(a);
  }
  return v;
}

// Warp sums of U (re, im) pairs by recursive halving: each xor step sends half
// of the lane's remaining values and keeps the other half (2U - 1 shuffles
// instead of 10 U for U separate butterflies); lane L then holds the sum of
// value (L >> (5 - log2 2U)), values 0..U-1 = re, U..2U-1 = im.  Returns
// sample u_sel's (re, im) to every lane (two indexed shuffles).
template <int U>
__device__ __forceinline__ float2 warp_sum_pairs(const float (&re)[U], const float (&im)[U], int lane, int u_sel) {
  constexpr int V = 2 * U;
  constexpr int LV = V == 2 ? 1 : V == 4 ? 2 : V == 8 ? 3 : V == 16 ? 4 : 5;
  static_assert((1 << LV) == V, "U a power of two <= 16");
  float v[V];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    v[u] = re[u];
    v[U + u] = im[u];
  }
#pragma unroll
  for (int step = 0; step < LV; ++step) {
    const int o = 16 >> step, half = V >> (step + 1);
    const bool hi = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float send = hi ? v[i] : v[i + half];
      const float keep = hi ? v[i + half] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
#pragma unroll
  for (int o = 16 >> LV; o > 0; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
  constexpr int sh = 5 - LV;
  const float r = __shfl_sync(0xffffffffu, v[0], u_sel << sh);
  const float i = __shfl_sync(0xffffffffu, v[0], 16 + (u_sel << sh));
  return make_float2(r, i);
}

// the result of sample `sid`: stored (+= with accumulate) into out, or
// reduce-added into its owner's shard
__device__ __forceinline__ void put_amp(const BlockGatherParams& p, int sid, float2 v) {
  if (p.multicast) {  // in-switch reduction into all ranks' buffers (sm_90+ multimem)
    float2* a = p.shard[0] + sid;
    asm volatile("multimem.red.relaxed.sys.global.add.v2.f32 [%0], {%1, %2};" ::"l"(a), "f"(v.x), "f"(v.y)
                 : "memory");
    return;
  }
  if (p.n_shards) {
    const int o = (int)(sid / p.shard_len);
    atomicAdd(p.shard[o] + (sid - (long long)o * p.shard_len), v);
    return;
  }
  if (p.accumulate) {
    const float2 w = p.out[sid];
    v.x += w.x;
    v.y += w.y;
  }
  p.out[sid] = v;
}

// One warp per sample, NF float4 of the K-row per lane (Kp = 64 * NF), U
// samples in flight per warp, RB rows of the direct half per block, NT
// threads, MINB CTAs per SM.  Warp w takes the w-th contiguous share of the
// block's samples, 32 at a time: lane i loads sample i's metadata (the
// block-ordered arrays, coalesced), then the warp walks them U at a time,
// each round one dependent load of U rows of T (addresses by shuffle).
// Shared memory S[RB][F] float4 (F = Kp / 2), slot f of row r at
// f ^ (r & (F - 1)): the per-sample reads (one row, consecutive slots) run at
// the minimum wavefront count.
template <int NF, int U, int RB, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) gather_block_c64_kernel(const BlockGatherParams p, const TrailParams tw,
                                                                    const float2* __restrict__ trail) {
  constexpr int F = 32 * NF;  // float4 per row (Kp / 2)
  constexpr int NW = NT / 32;
  static_assert(RB == 16 || RB == 32, "block rows");
  extern __shared__ float4 S[];  // [RB][F]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (long long blk = blockIdx.x; blk < p.n_blocks; blk += gridDim.x) {
    const int beg = p.offs[blk], end = p.offs[blk + 1];
    if (beg == end) continue;
    __syncthreads();  // the previous block's readers are done with S
    // ---- fill: rows r0 .. r0+RB-1 of D; a warp load covers 32 / RB k rows
    const long long r0 = blk * RB;
    constexpr int KPW = 32 / RB;
    const int r = lane % RB, kq = lane / RB;
    float2 fr = make_float2(1.f, 0.f);  // this thread's staged row's deferred diagonal
    for (int u = 0; u < p.dnr; ++u)
      fr = cmul(fr, __ldg(&p.dtab[p.doff[u] + (long long)(((unsigned long long)(r0 + r) >> p.dlo[u]) & p.dmask[u])]));
    for (int k0 = KPW * warp; k0 < 2 * F && !(p.debug & 1); k0 += KPW * NW * 4) {
      float2 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const long long k = k0 + KPW * NW * q + kq;
        v[q] = (k < p.K) ? __ldg(&p.D[k * p.ldD + r0 + r]) : make_float2(0.f, 0.f);
        if (p.cpD && k < p.K) v[q] = cmul(v[q], __ldg(&p.cpD[k]));
        if (p.dnr) v[q] = cmul(v[q], fr);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = k0 + KPW * NW * q + kq;
        if (RB == 16) {  // lanes r and r + 16 hold k and k + 1 (k even)
          const float ox = __shfl_down_sync(0xffffffffu, v[q].x, 16), oy = __shfl_down_sync(0xffffffffu, v[q].y, 16);
          if (kq == 0 && k < 2 * F) S[r * F + ((k >> 1) ^ (r & (F - 1)))] = make_float4(v[q].x, v[q].y, ox, oy);
        } else {  // RB == 32: one k per warp load; pairs are written as halves
          if (k < 2 * F) reinterpret_cast<float2*>(S)[2 * (r * F + ((k >> 1) ^ (r & (F - 1)))) + (k & 1)] = v[q];
        }
      }
    }
    __syncthreads();
    if (p.debug & 2) continue;
    // ---- samples: warp w's share [s0, s1)
    const int cnt = end - beg;
    const int s0 = beg + (int)((long long)cnt * warp / NW), s1 = beg + (int)((long long)cnt * (warp + 1) / NW);
    for (int jb = s0; jb < s1; jb += 32) {
      const int nb = min(32, s1 - jb);
      int sid = 0;
      unsigned long long sbv = 0;
      if (lane < nb) {
        sid = p.sidx[jb + lane];
        sbv = p.sbits[jb + lane];
      }
      // the batch's per-sample weights (folded units, deferred diagonals),
      // all lanes at once: their table loads overlap the first round's rows
      float2 wgt = make_float2(1.f, 0.f);
      if (tw.n && lane < nb) wgt = trail_weight(tw, trail, sbv);
      for (int jj = 0; jj < nb; jj += U) {
        float4 x[U][NF];
        unsigned long long bw[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          bw[u] = __shfl_sync(0xffffffffu, sbv, min(jj + u, nb - 1));
          const unsigned long long iT = p.direct_b ? (bw[u] >> p.n_low) & p.maskA : bw[u] & p.maskB;
          const float4* q = p.T + (long long)iT * F;
#pragma unroll
          for (int t = 0; t < NF; ++t) x[u][t] = ld_row(q + lane + 32 * t, p.ldmode);
        }
        float re[U], im[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          re[u] = 0.f;
          im[u] = 0.f;
          const int rd = (int)((p.direct_b ? bw[u] & p.maskB : (bw[u] >> p.n_low) & p.maskA) & (RB - 1));
          const float4* srow = S + rd * F;
          const int sw = rd & (F - 1);
#pragma unroll
          for (int t = 0; t < NF; ++t) {
            const float4 y = srow[(lane + 32 * t) ^ sw];
            const float4 a = p.direct_b ? x[u][t] : y;  // a = A' (c_p folded), c = B
            const float4 c = p.direct_b ? y : x[u][t];
            re[u] = fmaf(a.x, c.x, fmaf(-a.y, c.y, re[u]));
            im[u] = fmaf(a.x, c.y, fmaf(a.y, c.x, im[u]));
            re[u] = fmaf(a.z, c.z, fmaf(-a.w, c.w, re[u]));
            im[u] = fmaf(a.z, c.w, fmaf(a.w, c.z, im[u]));
          }
        }
        // lane jj + u (the holder of sample jj + u's metadata) writes it
        const int us = lane - jj;
        float2 v = warp_sum_pairs<U>(re, im, lane, (us >= 0 && us < U) ? us : 0);
        if (lane >= jj && lane < jj + U && lane < nb) {
          if (tw.n) v = cmul(v, wgt);
          put_amp(p, sid, v);
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
