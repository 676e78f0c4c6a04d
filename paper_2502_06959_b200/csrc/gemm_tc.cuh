// gemm_tc.cuh — full-output Kronecker path-sum on the 5th-generation tensor
// cores (tcgen05 + TMEM + TMA), split-bf16 emulation of the complex64 product
//
//   psi[i][j] = sum_p (c_p A[p][i]) B[p][j]          (a3 folded in)
//
// as ONE real GEMM  D[i][2j+c] = sum_kk A''[i][kk] B''[2j+c][kk]  whose fp32
// row-major output IS the interleaved complex64 result:
//   A'' row i       = (re, im) of c_p A[p][i]          for p = 0..K-1
//   B'' row 2j      = (re, -im) of B[p][j]
//   B'' row 2j+1    = (im,  re) of B[p][j]
// Each operand x is split x = hi + lo with hi = bf16_rn(x), lo = bf16_rn(x-hi);
// per k-block the kernel loads A_hi, A_lo, B_hi, B_lo once and issues three
// MMAs into the same TMEM accumulator: A_hi*B_hi + A_hi*B_lo + A_lo*B_hi
// (HSF_PREC_BF16X3; BF16X1 issues only the first).
//
// K4 (split_a/split_b): node-major leaves -> K-major bf16 hi/lo operands.
// K5 (tc_gemm_kernel): persistent, warp-specialised, one CTA per SM:
//   warp 0  TMA producer (cp.async.bulk.tensor, SWIZZLE_128B, mbarrier tx)
//   warp 1  TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=256,
//           K=16 per instruction), tcgen05.commit -> smem/TMEM barriers
//   warps 2-9 epilogue (2 per TMEM lane quarter, alternating 32-column
//           chunks): tcgen05.ld 32x32b -> registers -> st.shared into a
//           128B-swizzled 32x32 fp32 box -> TMA store (cp.async.bulk.tensor,
//           bulk_group, L2 evict-first), so the output is written as full
//           128 B row segments by the TMA engine
//   2 SMEM stages x (16+16+32+32) KB, 2 TMEM accumulators x 256 columns.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <cstring>

#include "hsf_internal.h"

namespace hsf {
namespace tc {

constexpr int BM = 128, BN = 256, BK = 64;  // BK in bf16 elements = 128 B rows
constexpr int STAGES = 2;
constexpr int A_TILE = BM * BK * 2;  // 16 KB
constexpr int B_TILE = BN * BK * 2;  // 32 KB
constexpr int STAGE_BYTES = 2 * A_TILE + 2 * B_TILE;
constexpr int EPI_WARPS = 8;             // 2 per TMEM lane quarter, alternating 32-column chunks
constexpr int EPI_BYTES = EPI_WARPS * 4096;  // per epilogue warp: one 32 x 128 B staging box
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_BYTES + 1024;  // + alignment slack
constexpr int THREADS = 64 + 32 * EPI_WARPS;
constexpr int TMEM_COLS = 512;  // 2 accumulators x 256 fp32 columns

struct Params {
  int num_m, num_n, num_k;  // blocks
  int n_fastest;            // tile raster: 1 => consecutive tiles walk N
  int group_m;              // > 0 => grouped raster (group_m row blocks per column sweep)
  int a_evict_last;         // 1 => A operand loads carry an L2 evict-last hint
  int accumulate;           // 1 => out += D (TMA reduce-add) instead of out = D
  int mn;                   // 1 => both operands MN-major (A''^T [2*Kpad][rows_pad], B''^T [2*Kpad][nrows_b_pad];
                            //      split_a_mn_kernel / split_b_mn_kernel)

  int x3;
  int x6;                   // bf16x6: third operand plane (lo2), 6 products (pair kernel only)
  int bk;                   // 1 (pair kernel, with mn): B K-major [nrows_b_pad][Kpad] instead (swapped path-sum)
  int bn;                   // pair tile N (multiple of 32, <= BN; < BN only with bk)
  int n_maps;               // > 0: fused reduce-scatter -- output rows [o*rows_per_map, +rows_per_map)
  int rows_per_map;         //      are TMA-reduce-added into OutMaps::m[o] (row o*rows_per_map -> 0)
  float* out;               // D, row-major, ld = ldo floats
  long long ldo;
  long long rows, cols;     // valid D extent (rows of this call, 2*MB)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
#ifndef HSF_DEBUG_SYNC
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}
#else
// Debug build (libhsf_debug.so, -DHSF_DEBUG_SYNC; the substitute for
// compute-sanitizer, which this pool does not run): every mbarrier wait is
// bounded -- after ~2 s of SM clock without the phase flipping (a lost TMA
// transaction, a wrong expect_tx byte count, a missing arrive) the thread
// reports the barrier and traps, so a protocol bug ends the kernel with an
// error instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  const long long t0 = clock64();
  for (;;) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    if (ok) return;
    if (clock64() - t0 > 4000000000ll) {
      uint64_t st;
      asm volatile("ld.shared.b64 %0, [%1];" : "=l"(st) : "r"(addr));
      printf("hsf debug: mbarrier wait timed out: block (%d,%d) thread %d barrier smem 0x%x parity %u state 0x%llx\n",
             blockIdx.x, blockIdx.y, threadIdx.x, addr, parity, (unsigned long long)st);
      __trap();
    }
  }
}
#endif
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
// output tiles are written once and never re-read by this kernel: evict-first
// so the streaming stores do not push the re-used operand tiles out of L2
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1, uint64_t policy) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"(
                   map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "l"(policy)
               : "memory");
}
// accumulate mode: the TMA engine adds the box into global memory (fp32 add)
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, const void* src, int c0, int c1,
                                                  uint64_t policy) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"(
          map),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  // UMMA shared-memory descriptor, K-major, SWIZZLE_128B: start>>4, LBO=1 (unused),
  // SBO=1024 B between 8-row swizzle atoms, version 1 (sm_100), layout type 2.
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// MN-major operand, SWIZZLE_128B: 64-element (128 B) rows along M/N, one row
// per k; LBO = 8 KB between 64-wide MN atoms (TMA boxes of 64 x BK),
// SBO = 1024 B between 8-row k groups
__device__ __forceinline__ uint64_t sw128_desc_mn(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(8192 >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
constexpr uint32_t kMajorMN = (1u << 15) | (1u << 16);  // instruction descriptor: A and B MN-major
// kind::f16 instruction descriptor: D=F32, A=B=BF16, K-major both, N=BN, M=BM
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accum,
                                         uint32_t idesc = IDESC) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tile_coords(const Params& p, int tile, int& mb, int& nb) {
  if (p.group_m > 0) {  // groups of group_m row blocks, each swept column tile by column tile
    const int gsz = p.group_m * p.num_n, g = tile / gsz, first = g * p.group_m;
    const int gm = min(p.num_m - first, p.group_m), r = tile % gsz;
    mb = first + r % gm;
    nb = r / gm;
  } else if (p.n_fastest) {
    mb = tile / p.num_n;
    nb = tile % p.num_n;
  } else {
    mb = tile % p.num_m;
    nb = tile / p.num_m;
  }
}

__global__ void __launch_bounds__(THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap mA_hi, const __grid_constant__ CUtensorMap mA_lo,
                   const __grid_constant__ CUtensorMap mB_hi, const __grid_constant__ CUtensorMap mB_lo,
                   const __grid_constant__ CUtensorMap mOut, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int num_tiles = p.num_m * p.num_n;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 32 * EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mA_hi) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mB_hi) : "memory");
    if (p.x3) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mA_lo) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mB_lo) : "memory");
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_base = tmem_base_sh;

  const uint32_t stage_bytes = p.x3 ? (uint32_t)STAGE_BYTES : (uint32_t)(A_TILE + B_TILE);

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      // A row-block tiles are re-read once per N tile: keep them in L2 when the
      // whole A operand fits comfortably (c4); otherwise normal priority
      const uint64_t a_pol = p.a_evict_last ? policy_evict_last() : policy_evict_normal();
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int mb, nb;
        tile_coords(p, tile, mb, nb);
        for (int kb = 0; kb < p.num_k; ++kb) {
          mbar_wait(&empty_bar[s], ph ^ 1);
          uint8_t* st = smem + s * STAGE_BYTES;
          mbar_expect_tx(&full_bar[s], stage_bytes);
          if (p.mn) {  // 64(m|n) x BK(k) boxes: two per A operand, four per B operand
            for (int j = 0; j < BM / 64; ++j) {
              tma_load_2d_hint(st + j * 8192, &mA_hi, &full_bar[s], mb * BM + j * 64, kb * BK, a_pol);
              if (p.x3) tma_load_2d_hint(st + A_TILE + j * 8192, &mA_lo, &full_bar[s], mb * BM + j * 64, kb * BK, a_pol);
            }
            for (int j = 0; j < BN / 64; ++j) {
              tma_load_2d(st + 2 * A_TILE + j * 8192, &mB_hi, &full_bar[s], nb * BN + j * 64, kb * BK);
              if (p.x3) tma_load_2d(st + 2 * A_TILE + B_TILE + j * 8192, &mB_lo, &full_bar[s], nb * BN + j * 64, kb * BK);
            }
          } else {
            tma_load_2d_hint(st, &mA_hi, &full_bar[s], kb * BK, mb * BM, a_pol);
            if (p.x3) tma_load_2d_hint(st + A_TILE, &mA_lo, &full_bar[s], kb * BK, mb * BM, a_pol);
            tma_load_2d(st + 2 * A_TILE, &mB_hi, &full_bar[s], kb * BK, nb * BN);
            if (p.x3) tma_load_2d(st + 2 * A_TILE + B_TILE, &mB_lo, &full_bar[s], kb * BK, nb * BN);
          }
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        mbar_wait(&tempty_bar[acc], aph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t d = tmem_base + (uint32_t)(acc * BN);
        for (int kb = 0; kb < p.num_k; ++kb) {
          mbar_wait(&full_bar[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t st = smem_u32(smem + s * STAGE_BYTES);
          const uint32_t a_hi = st, a_lo = st + A_TILE, b_hi = st + 2 * A_TILE, b_lo = st + 2 * A_TILE + B_TILE;
          if (p.mn) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint32_t kr = k * 2048;  // 16 k rows of 128 B
              const uint32_t id = IDESC | kMajorMN;
              mma_bf16(d, sw128_desc_mn(a_hi + kr), sw128_desc_mn(b_hi + kr), (kb | k) ? 1u : 0u, id);
              if (p.x3) {
                mma_bf16(d, sw128_desc_mn(a_hi + kr), sw128_desc_mn(b_lo + kr), 1u, id);
                mma_bf16(d, sw128_desc_mn(a_lo + kr), sw128_desc_mn(b_hi + kr), 1u, id);
              }
            }
          } else {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint32_t ko = k * 32;  // 16 bf16 = 32 B inside the 128 B swizzle row
              mma_bf16(d, sw128_desc(a_hi + ko), sw128_desc(b_hi + ko), (kb | k) ? 1u : 0u);
              if (p.x3) {
                mma_bf16(d, sw128_desc(a_hi + ko), sw128_desc(b_lo + ko), 1u);
                mma_bf16(d, sw128_desc(a_lo + ko), sw128_desc(b_hi + ko), 1u);
              }
            }
          }
          mma_commit(&empty_bar[s]);  // frees the smem stage when these MMAs retire
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        mma_commit(&tfull_bar[acc]);  // accumulator ready for the epilogue
        if (++acc == 2) {
          acc = 0;
          aph ^= 1;
        }
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    const uint64_t st_pol = policy_evict_first();
    const int q = warp & 3;  // TMEM lane quarter this warp may access (rows 32q..32q+31)
    const int half = (warp - 2) / 4;  // which alternate chunks this warp drains
    uint8_t* stg = smem + STAGES * STAGE_BYTES + (warp - 2) * 4096;  // 1024-aligned 4 KB box
    int acc = 0;
    uint32_t aph = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      int mb, nb;
      tile_coords(p, tile, mb, nb);
      mbar_wait(&tfull_bar[acc], aph);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll 1
      for (int c = half; c < BN / 32; c += 2) {
        uint32_t v[32];
        const uint32_t taddr = tmem_base + (uint32_t)(acc * BN + c * 32) + ((uint32_t)(q * 32) << 16);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
              "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c >= BN / 32 - 2) {  // this warp's last chunk read: release its share of the accumulator
          asm volatile("tcgen05.fence::before_thread_sync;");
          mbar_arrive(&tempty_bar[acc]);
        }
        // the previous TMA store from this box must have finished reading it
        // (overlapped with the tcgen05.ld above)
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
        // row `lane` of the 32x32 box, 128B swizzle: 16 B chunk j at j ^ (row & 7)
        float4* dst = reinterpret_cast<float4*>(stg + lane * 128);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          dst[j ^ (lane & 7)] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                            __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> async proxy
        __syncwarp();
        if (lane == 0) {
          if (p.accumulate)
            tma_reduce_add_2d(&mOut, stg, nb * BN + c * 32, mb * BM + q * 32, st_pol);
          else
            tma_store_2d(&mOut, stg, nb * BN + c * 32, mb * BM + q * 32, st_pol);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      if (++acc == 2) {
        acc = 0;
        aph ^= 1;
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
}

// ------------------------------------------------- K5, CTA-pair (cta_group::2)
// Two CTAs of a cluster (one TPC) cooperate on a 256 x 256 output tile: each
// holds its own 128 A rows and HALF of the tile's B rows (128 of 256) in
// shared memory; the leader CTA (rank 0) issues tcgen05.mma.cta_group::2
// with M = 256, N = 256, which reads A from each CTA's SMEM and the B halves
// from both, and accumulates each CTA's 128 rows x 256 columns into that
// CTA's TMEM.  Per SM this halves the B operand traffic (TMA into SMEM and
// MMA reads out of it): single-CTA x3 needs ~160 B/clk of SMEM bandwidth per
// SM at full tensor rate (ncu: tensor pipe 77 % active), the pair ~104 B/clk.
// Protocol (CUTLASS sm100 2SM conventions): every CTA's TMA loads signal the
// LEADER's full barrier (shared::cluster address with the peer bit cleared,
// .cta_group::2); only the leader arms it with both CTAs' bytes; MMA commits
// multicast to both CTAs' empty / accumulator-full barriers; every epilogue
// thread of both CTAs arrives on the leader's accumulator-empty barrier.
constexpr int B2_TILE = (BN / 2) * BK * 2;               // 16 KB: this CTA's half of B
constexpr int STAGE2_BYTES = 2 * A_TILE + 2 * B2_TILE;   // 64 KB
constexpr int smem2_bytes(int nst, int ebuf, int npl = 2, int ew = EPI_WARPS) {
  return nst * npl * (A_TILE + B2_TILE) + ebuf * ew * 4096 + 1024;
}
constexpr uint32_t IDESC2 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)((2 * BM) >> 4) << 24);
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // shared::cluster address -> the pair's rank-0 CTA

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2sm(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                             uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar) & kPeerMask), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void mma2_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accum,
                                          uint32_t idesc = IDESC2) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
// kind::tf32: D=F32, A=B=TF32 (format 2), K = 8 per instruction (32 B, the
// same byte step as bf16's K = 16)
constexpr uint32_t IDESC2_TF32 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                 ((uint32_t)((2 * BM) >> 4) << 24);
__device__ __forceinline__ void mma2_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(IDESC2_TF32), "r"(accum));
}
__device__ __forceinline__ void mma2_commit_both(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .b16 m;\n"
      "mov.b16 m, 3;\n"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & kPeerMask)
               : "memory");
}

// p.num_m counts 256-row PAIR tiles here
// NST SMEM stages, EBUF staging boxes per epilogue warp: <3,1> for long K
// (c2: deep operand pipeline), <2,2> for short K (c4: num_k <= 2, the kernel
// is output-write-bound, so a second box keeps two TMA stores per warp in flight)
// TF32: kind::tf32 on fp32-storage operands (tf32x3; K-major only, boxes of
// 32 fp32 = the same 128 B rows)
// Destination shards of the fused reduce-scatter (tensor maps of device or
// peer-GPU memory: each owner's row shard)
constexpr int kMaxOutMaps = 8;
struct OutMaps {
  CUtensorMap m[kMaxOutMaps];
};

// EW epilogue warps (8, or 16 for the output-write-bound short-K shape: more
// 4 KB TMA stores in flight per SM)
template <int NST, int EBUF, bool TF32 = false, int EW = EPI_WARPS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64 + 32 * EW, 1)
    tc_gemm2_kernel(const __grid_constant__ CUtensorMap mA_hi, const __grid_constant__ CUtensorMap mA_lo,
                    const __grid_constant__ CUtensorMap mB_hi, const __grid_constant__ CUtensorMap mB_lo,
                    const __grid_constant__ CUtensorMap mA_l2, const __grid_constant__ CUtensorMap mB_l2,
                    const __grid_constant__ CUtensorMap mOut, const Params p, const __grid_constant__ OutMaps om) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[NST], empty_bar[NST], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int num_tiles = p.num_m * p.num_n;
  const uint32_t rank = cluster_rank();
  const int pair = blockIdx.x >> 1, num_pairs = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full_bar[s], 1);   // the leader's producer arms it (both CTAs' bytes)
      mbar_init(&empty_bar[s], 1);  // one multicast commit per stage use
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 2 * 32 * EW);  // epilogue threads of both CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mA_hi) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mB_hi) : "memory");
  }
  if (warp == 1) {  // same logical warp in both CTAs
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();  // peer barriers initialised before any remote arrive / complete_tx
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_base = tmem_base_sh;
  // stage layout: npl A plane slots, then npl B plane slots (hi, lo[, lo2])
  const int npl = p.x6 ? 3 : 2;
  // (narrow K-major B: a bn/2-row slot per plane, so more stages fit)
  const uint32_t BSL = p.bk ? (((uint32_t)(p.bn / 2) * 128u + 1023u) & ~1023u) : (uint32_t)B2_TILE;
  const uint32_t SS = (uint32_t)npl * (A_TILE + BSL);
  const uint32_t stage_bytes = (uint32_t)(p.x6 ? 3 : p.x3 ? 2 : 1) * (A_TILE + (p.bk ? (p.bn / 2) * 128 : B2_TILE));

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      const uint64_t a_pol = p.a_evict_last ? policy_evict_last() : policy_evict_normal();
      const uint64_t b_pol = policy_evict_normal();
      int s = 0;
      uint32_t ph = 0;
      for (int tile = pair; tile < num_tiles; tile += num_pairs) {
        int mb, nb;
        tile_coords(p, tile, mb, nb);
        const int arow = (2 * mb + (int)rank) * BM, brow = nb * p.bn + (int)rank * (p.bn / 2);
        for (int kb = 0; kb < p.num_k; ++kb) {
          mbar_wait(&empty_bar[s], ph ^ 1);
          uint8_t* st = smem + s * SS;
          uint8_t* sb = st + npl * A_TILE;
          if (rank == 0) mbar_expect_tx(&full_bar[s], 2 * stage_bytes);
          if (p.mn) {  // 64(m|n) x BK(k) boxes: two per A operand, two per B operand half
            for (int j = 0; j < BM / 64; ++j) {
              tma_load_2sm(st + j * 8192, &mA_hi, &full_bar[s], arow + j * 64, kb * BK, a_pol);
              if (p.x3) tma_load_2sm(st + A_TILE + j * 8192, &mA_lo, &full_bar[s], arow + j * 64, kb * BK, a_pol);
              if (p.x6) tma_load_2sm(st + 2 * A_TILE + j * 8192, &mA_l2, &full_bar[s], arow + j * 64, kb * BK, a_pol);
            }
            if (p.bk) {  // K-major B: one {BK, bn/2} box per plane
              tma_load_2sm(sb, &mB_hi, &full_bar[s], kb * BK, brow, b_pol);
              if (p.x3) tma_load_2sm(sb + BSL, &mB_lo, &full_bar[s], kb * BK, brow, b_pol);
              if (p.x6) tma_load_2sm(sb + 2 * BSL, &mB_l2, &full_bar[s], kb * BK, brow, b_pol);
            } else {
              for (int j = 0; j < BN / 128; ++j) {
                tma_load_2sm(sb + j * 8192, &mB_hi, &full_bar[s], brow + j * 64, kb * BK, b_pol);
                if (p.x3) tma_load_2sm(sb + B2_TILE + j * 8192, &mB_lo, &full_bar[s], brow + j * 64, kb * BK, b_pol);
                if (p.x6) tma_load_2sm(sb + 2 * B2_TILE + j * 8192, &mB_l2, &full_bar[s], brow + j * 64, kb * BK, b_pol);
              }
            }
          } else {
            const int kc = kb * (TF32 ? BK / 2 : BK);  // element coordinate of this 128 B k block
            tma_load_2sm(st, &mA_hi, &full_bar[s], kc, arow, a_pol);
            if (p.x3) tma_load_2sm(st + A_TILE, &mA_lo, &full_bar[s], kc, arow, a_pol);
            if (p.x6) tma_load_2sm(st + 2 * A_TILE, &mA_l2, &full_bar[s], kc, arow, a_pol);
            tma_load_2sm(sb, &mB_hi, &full_bar[s], kc, brow, b_pol);
            if (p.x3) tma_load_2sm(sb + B2_TILE, &mB_lo, &full_bar[s], kc, brow, b_pol);
            if (p.x6) tma_load_2sm(sb + 2 * B2_TILE, &mB_l2, &full_bar[s], kc, brow, b_pol);
          }
          if (++s == NST) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    if (lane == 0 && rank == 0) {
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      for (int tile = pair; tile < num_tiles; tile += num_pairs) {
        mbar_wait(&tempty_bar[acc], aph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t d = tmem_base + (uint32_t)(acc * BN);
        for (int kb = 0; kb < p.num_k; ++kb) {
          mbar_wait(&full_bar[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t st = smem_u32(smem + s * SS);
          const uint32_t a_hi = st, a_lo = st + A_TILE, a_l2 = st + 2 * A_TILE;
          const uint32_t b_hi = st + npl * A_TILE, b_lo = b_hi + BSL, b_l2 = b_hi + 2 * BSL;
          if (p.mn && p.bk) {  // A MN-major (k step 16 rows = 2 KB), B K-major (k step 32 B), N = bn
            const uint32_t id = (IDESC2 & ~(0x3Fu << 17)) | ((uint32_t)(p.bn >> 3) << 17) | (1u << 15);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint32_t kr = k * 2048, ko = k * 32;
              mma2_bf16(d, sw128_desc_mn(a_hi + kr), sw128_desc(b_hi + ko), (kb | k) ? 1u : 0u, id);
              if (p.x3) {
                mma2_bf16(d, sw128_desc_mn(a_hi + kr), sw128_desc(b_lo + ko), 1u, id);
                mma2_bf16(d, sw128_desc_mn(a_lo + kr), sw128_desc(b_hi + ko), 1u, id);
              }
              if (p.x6) {
                mma2_bf16(d, sw128_desc_mn(a_lo + kr), sw128_desc(b_lo + ko), 1u, id);
                mma2_bf16(d, sw128_desc_mn(a_hi + kr), sw128_desc(b_l2 + ko), 1u, id);
                mma2_bf16(d, sw128_desc_mn(a_l2 + kr), sw128_desc(b_hi + ko), 1u, id);
              }
            }
          } else if (p.mn) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint32_t kr = k * 2048;
              const uint32_t id = IDESC2 | kMajorMN;
              mma2_bf16(d, sw128_desc_mn(a_hi + kr), sw128_desc_mn(b_hi + kr), (kb | k) ? 1u : 0u, id);
              if (p.x3) {
                mma2_bf16(d, sw128_desc_mn(a_hi + kr), sw128_desc_mn(b_lo + kr), 1u, id);
                mma2_bf16(d, sw128_desc_mn(a_lo + kr), sw128_desc_mn(b_hi + kr), 1u, id);
              }
              if (p.x6) {  // bf16x6: + lo*lo + hi*lo2 + lo2*hi
                mma2_bf16(d, sw128_desc_mn(a_lo + kr), sw128_desc_mn(b_lo + kr), 1u, id);
                mma2_bf16(d, sw128_desc_mn(a_hi + kr), sw128_desc_mn(b_l2 + kr), 1u, id);
                mma2_bf16(d, sw128_desc_mn(a_l2 + kr), sw128_desc_mn(b_hi + kr), 1u, id);
              }
            }
          } else {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint32_t ko = k * 32;
              if constexpr (TF32) {
                mma2_tf32(d, sw128_desc(a_hi + ko), sw128_desc(b_hi + ko), (kb | k) ? 1u : 0u);
                mma2_tf32(d, sw128_desc(a_hi + ko), sw128_desc(b_lo + ko), 1u);
                mma2_tf32(d, sw128_desc(a_lo + ko), sw128_desc(b_hi + ko), 1u);
                continue;
              }
              mma2_bf16(d, sw128_desc(a_hi + ko), sw128_desc(b_hi + ko), (kb | k) ? 1u : 0u);
              if (p.x3) {
                mma2_bf16(d, sw128_desc(a_hi + ko), sw128_desc(b_lo + ko), 1u);
                mma2_bf16(d, sw128_desc(a_lo + ko), sw128_desc(b_hi + ko), 1u);
              }
              if (p.x6) {
                mma2_bf16(d, sw128_desc(a_lo + ko), sw128_desc(b_lo + ko), 1u);
                mma2_bf16(d, sw128_desc(a_hi + ko), sw128_desc(b_l2 + ko), 1u);
                mma2_bf16(d, sw128_desc(a_l2 + ko), sw128_desc(b_hi + ko), 1u);
              }
            }
          }
          mma2_commit_both(&empty_bar[s]);  // both CTAs' stage s free once these retire
          if (++s == NST) {
            s = 0;
            ph ^= 1;
          }
        }
        mma2_commit_both(&tfull_bar[acc]);  // both CTAs' accumulators ready
        if (++acc == 2) {
          acc = 0;
          aph ^= 1;
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const uint64_t st_pol = policy_evict_first();
    const int q = warp & 3;
    constexpr int G = EW / 4;  // warps per TMEM lane quarter, interleaving 32-column chunks
    const int half = (warp - 2) / 4;
    uint8_t* stg0 = smem + NST * SS + (warp - 2) * 4096 * EBUF;
    int buf = 0;
    int acc = 0;
    uint32_t aph = 0;
    for (int tile = pair; tile < num_tiles; tile += num_pairs) {
      int mb, nb;
      tile_coords(p, tile, mb, nb);
      const int row0 = (2 * mb + (int)rank) * BM;
      const int nc = p.bn / 32;  // 32-column chunks of the tile
      mbar_wait(&tfull_bar[acc], aph);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (half >= nc) {  // narrow tile: no chunk for this warp
        asm volatile("tcgen05.fence::before_thread_sync;");
        mbar_arrive_leader(&tempty_bar[acc]);
      }
#pragma unroll 1
      for (int c = half; c < nc; c += G) {
        uint32_t v[32];
        const uint32_t taddr = tmem_base + (uint32_t)(acc * BN + c * 32) + ((uint32_t)(q * 32) << 16);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
              "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c >= nc - G) {
          asm volatile("tcgen05.fence::before_thread_sync;");
          mbar_arrive_leader(&tempty_bar[acc]);
        }
        // the TMA store issued EBUF chunks ago from this box must have read it
        if (lane == 0) {
          if (EBUF == 1)
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          else
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        }
        __syncwarp();
        uint8_t* stg = stg0 + buf * 4096;
        buf = (buf + 1) % EBUF;
        float4* dst = reinterpret_cast<float4*>(stg + lane * 128);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          dst[j ^ (lane & 7)] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                            __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          if (p.n_maps) {  // fused reduce-scatter: this CTA's 128 rows belong to one owner shard
            const int o = row0 / p.rows_per_map;
            tma_reduce_add_2d(&om.m[o], stg, nb * p.bn + c * 32, row0 - o * p.rows_per_map + q * 32, st_pol);
          } else if (p.accumulate) {
            tma_reduce_add_2d(&mOut, stg, nb * p.bn + c * 32, row0 + q * 32, st_pol);
          } else {
            tma_store_2d(&mOut, stg, nb * p.bn + c * 32, row0 + q * 32, st_pol);
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      if (++acc == 2) {
        acc = 0;
        aph ^= 1;
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();  // the peer is done with the leader's barriers and the MMAs with both SMEMs
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
}

// ----------------------------------------------------------------------- K4
__device__ __forceinline__ float2 cmul_f(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// tf32 (fp32 storage, low 13 mantissa bits zero; RNA as cvt.rna.tf32.f32)
__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// pair splitters of the K-major kernels: (re|im) pair -> hi, lo, lo2 pairs
__device__ __forceinline__ void split3(float x, __nv_bfloat16& hi, __nv_bfloat16& lo, __nv_bfloat16& lo2);
__device__ __forceinline__ void split_pair(float a, float b, __nv_bfloat162& h, __nv_bfloat162& l, __nv_bfloat162& m) {
  split3(a, h.x, l.x, m.x);
  split3(b, h.y, l.y, m.y);
}
__device__ __forceinline__ void split_pair(float a, float b, float2& h, float2& l, float2& m) {  // tf32x3
  h = make_float2(to_tf32(a), to_tf32(b));
  l = make_float2(to_tf32(a - h.x), to_tf32(b - h.y));
  m = make_float2(0.f, 0.f);
}

// three-way split for bf16x6: x ~ hi + lo + lo2
__device__ __forceinline__ void split3(float x, __nv_bfloat16& hi, __nv_bfloat16& lo, __nv_bfloat16& lo2) {
  hi = __float2bfloat16_rn(x);
  const float r = x - __bfloat162float(hi);
  lo = __float2bfloat16_rn(r);
  lo2 = __float2bfloat16_rn(r - __bfloat162float(lo));
}

__device__ __forceinline__ void split_bf16(float x, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(x);
  lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}

// Half-sided folds (plan.cpp, Plan::Tail): the leaf of path p is the tree leaf
// ((p / T) mod Tt) times prod_u F_{u,d_u}[i's bits on mask_u], the tail units
// [u0, U) being the fastest digits of p; head-scalar units [0, v0) are not in
// the tree (their scalars are in c_p).
struct TailParams {
  int n;
  int radix[kMaxTail];
  unsigned mask[kMaxTail];     // half-local support bits of unit u0 + j
  long long off[kMaxTail];     // digit-0 diagonal of unit u0 + j in the tail table
  long long stride[kMaxTail];  // digit d_j = (p / stride[j]) % radix[j]
  int mapped;                  // 1 => half variant active: leaf = ((p / T) mod Tt) - node0 (else leaf = p)
  long long T;                 // prod of the folded radices
  long long Tt;                // tree paths
  long long node0;             // first materialised leaf
  long long p0;                // global path of operand column 0
  const float2* W;             // optional [T][2^m] table of the tail weights (tail_weights_kernel)
  long long wld;               // its row length 2^m
};

// Per 32-path x 32-amplitude tile: the leaf row of each path and, per folded
// unit, each path's diagonal (table offset) and each amplitude's index in it
struct TailTile {
  long long node[32];
  int base[kMaxTail][32];
  int idx[kMaxTail][32];
};

__device__ __forceinline__ void tail_tile_setup(TailTile& tt, const TailParams& tp, long long pb, long long ib) {
  const int tid = threadIdx.y * 32 + threadIdx.x;  // 256 threads
  if (tid < 32) tt.node[tid] = ((tp.p0 + pb + tid) / tp.T) % tp.Tt - tp.node0;
  for (int e = tid; e < tp.n * 32; e += 256) {
    const int u = e >> 5, r = e & 31;
    const long long p = tp.p0 + pb + r;
    const int d = (int)((p / tp.stride[u]) % tp.radix[u]);
    tt.base[u][r] = (int)(tp.off[u] + ((long long)d << __popc(tp.mask[u])));
    const unsigned i = (unsigned)(ib + r);
    unsigned mk = tp.mask[u], x = 0;
    for (int j = 0; mk; ++j, mk &= mk - 1) x |= ((i >> (__ffs(mk) - 1)) & 1u) << j;
    tt.idx[u][r] = (int)x;
  }
  __syncthreads();
}

__device__ __forceinline__ float2 tail_weight(const TailTile& tt, int n, const float2* __restrict__ tab, int r, int c) {
  float2 w = __ldg(&tab[tt.base[0][r] + tt.idx[0][c]]);
  for (int u = 1; u < n; ++u) {
    const float2 f = __ldg(&tab[tt.base[u][r] + tt.idx[u][c]]);
    w = make_float2(w.x * f.x - w.y * f.y, w.x * f.y + w.y * f.x);
  }
  return w;
}

// A'' rows [0, rows_pad): row i <- (re, im) of c_p * A[p][r0 + i]; zero padding.
// T2 = __nv_bfloat162 (bf16 splits) or float2 (tf32x3)
template <typename T2>
__global__ void split_a_kernel(const float2* __restrict__ leaves, const float2* __restrict__ cp,
                               T2* __restrict__ hi, T2* __restrict__ lo, long long K,
                               long long Kpad, long long MA, long long r0, long long rows, const TailParams tp,
                               const float2* __restrict__ ttab, T2* __restrict__ lo2) {
  __shared__ float2 t[32][33];
  __shared__ TailTile tt;
  const long long i0 = (long long)blockIdx.x * 32, p0 = (long long)blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  if (tp.mapped) tail_tile_setup(tt, tp, p0, r0 + i0);
  for (int r = ty; r < 32; r += 8) {
    long long p = p0 + r, i = i0 + tx;
    float2 v = make_float2(0.f, 0.f);
    if (p < K && i < rows) {
      float2 c = cp[p];
      const float2 a = leaves[(tp.mapped ? tt.node[r] : p) * MA + r0 + i];
      if (tp.W) c = cmul_f(c, tp.W[((tp.p0 + p) % tp.T) * tp.wld + r0 + i]);
      else if (tp.n) c = cmul_f(c, tail_weight(tt, tp.n, ttab, r, tx));
      v = make_float2(a.x * c.x - a.y * c.y, a.x * c.y + a.y * c.x);
    }
    t[r][tx] = v;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    long long i = i0 + r, p = p0 + tx;
    float2 v = t[tx][r];
    T2 h, l, l2;
    split_pair(v.x, v.y, h, l, l2);
    hi[i * Kpad + p] = h;
    if (lo) lo[i * Kpad + p] = l;
    if (lo2) lo2[i * Kpad + p] = l2;
  }
}

// B'' rows [0, 2*MB_pad): row 2j <- (re, -im), row 2j+1 <- (im, re) of B[p][j]
// (swapped path-sum: the leaves are half A's, columns col0.. of rows of
// length MS, times c_p when cp is given)
template <typename T2>
__global__ void split_b_kernel(const float2* __restrict__ leaves, T2* __restrict__ hi,
                               T2* __restrict__ lo, long long K, long long Kpad, long long MB,
                               const TailParams tp, const float2* __restrict__ ttab,
                               T2* __restrict__ lo2, const float2* __restrict__ cp, long long col0, long long MS) {
  __shared__ float2 t[32][33];
  const long long j0 = (long long)blockIdx.x * 32, p0 = (long long)blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  __shared__ TailTile tt;
  if (tp.mapped) tail_tile_setup(tt, tp, p0, col0 + j0);
  for (int r = ty; r < 32; r += 8) {
    long long p = p0 + r, j = j0 + tx;
    float2 v = make_float2(0.f, 0.f);
    if (p < K && j < MB) {
      v = leaves[(tp.mapped ? tt.node[r] : p) * MS + col0 + j];
      if (tp.W) v = cmul_f(v, tp.W[((tp.p0 + p) % tp.T) * tp.wld + col0 + j]);
      else if (tp.n) v = cmul_f(v, tail_weight(tt, tp.n, ttab, r, tx));
      if (cp) v = cmul_f(v, cp[p]);
    }
    t[r][tx] = v;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    long long j = j0 + r, p = p0 + tx;
    float2 v = t[tx][r];
    T2 h0, l0, h1, l1, m0, m1;
    split_pair(v.x, -v.y, h0, l0, m0);
    split_pair(v.y, v.x, h1, l1, m1);
    if (lo2) {
      lo2[(2 * j) * Kpad + p] = m0;
      lo2[(2 * j + 1) * Kpad + p] = m1;
    }
    hi[(2 * j) * Kpad + p] = h0;
    hi[(2 * j + 1) * Kpad + p] = h1;
    if (lo) {
      lo[(2 * j) * Kpad + p] = l0;
      lo[(2 * j + 1) * Kpad + p] = l1;
    }
  }
}

// W[t][i] = prod_u F_{u,d_u(t)}[i's bits on mask_u] for the tail digit
// combinations t in [0, T) (the folded units' digits of p mod T): the split
// kernels then take one table load per element instead of the per-unit loop
__global__ void tail_weights_kernel(float2* __restrict__ W, long long wld, const TailParams tp,
                                    const float2* __restrict__ ttab) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= tp.T * wld) return;
  const long long t = e / wld;
  const unsigned i = (unsigned)(e % wld);
  float2 w = make_float2(1.f, 0.f);
  for (int u = 0; u < tp.n; ++u) {
    const int d = (int)((t / tp.stride[u]) % tp.radix[u]);
    unsigned mk = tp.mask[u], x = 0;
    for (int q = 0; mk; ++q, mk &= mk - 1) x |= ((i >> (__ffs(mk) - 1)) & 1u) << q;
    w = cmul_f(w, ttab[tp.off[u] + ((long long)d << __popc(tp.mask[u])) + x]);
  }
  W[e] = w;
}

// MN-major A'' (p.mn): row 2p <- Re, row 2p+1 <- Im of c_p * A[p][r0 + i] over
// i in [0, rows_pad) (zero past `rows`): split_a_kernel's operand transposed,
// written elementwise.  One CTA per (path, 2048 rows), 8 rows per thread
// (16 B stores per plane row).
__global__ void split_a_mn_kernel(const float2* __restrict__ leaves, const float2* __restrict__ cp,
                                  __nv_bfloat16* __restrict__ hi, __nv_bfloat16* __restrict__ lo, long long K,
                                  long long lda, long long MA, long long r0, long long rows, const TailParams tp,
                                  const float2* __restrict__ ttab, __nv_bfloat16* __restrict__ lo2) {
  // 4 rounds per thread of 2 consecutive rows: each warp load / store
  // instruction covers 512 B / 128 B contiguous (coalesced; 8 consecutive rows
  // per thread left half of every L1 sector unused)
  __shared__ int base[kMaxTail];
  __shared__ unsigned smask[kMaxTail];
  __shared__ long long node;
  const long long p = blockIdx.y;
  if (tp.mapped) {
    if (threadIdx.x < tp.n) {
      const int u = threadIdx.x;
      const int d = (int)(((tp.p0 + p) / tp.stride[u]) % tp.radix[u]);
      base[u] = (int)(tp.off[u] + ((long long)d << __popc(tp.mask[u])));
      smask[u] = tp.mask[u];
    }
    if (threadIdx.x == 0) node = ((tp.p0 + p) / tp.T) % tp.Tt - tp.node0;
    __syncthreads();
  }
  const float2 c = p < K ? (cp ? cp[p] : make_float2(1.f, 0.f)) : make_float2(0.f, 0.f);  // cp null => 1
  const long long row = tp.mapped ? node : p;
  const float2* __restrict__ wrow = tp.W ? tp.W + ((tp.p0 + p) % tp.T) * tp.wld : nullptr;
  const float2* __restrict__ src = leaves + row * MA + r0;
  const bool vec = ((r0 & 1) == 0);
#pragma unroll
  for (int rd = 0; rd < 4; ++rd) {
    const long long i = (long long)blockIdx.x * 2048 + rd * 512 + 2 * threadIdx.x;
    if (i >= lda) break;
    float2 v[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    if (p < K && i + 2 <= rows && vec) {
      const float4 a4 = *reinterpret_cast<const float4*>(src + i);
      v[0] = cmul_f(make_float2(a4.x, a4.y), c);
      v[1] = cmul_f(make_float2(a4.z, a4.w), c);
      if (tp.W) {
        const float4 w4 = *reinterpret_cast<const float4*>(wrow + r0 + i);
        v[0] = cmul_f(v[0], make_float2(w4.x, w4.y));
        v[1] = cmul_f(v[1], make_float2(w4.z, w4.w));
      }
    } else {
      for (int e = 0; e < 2; ++e)
        if (p < K && i + e < rows) {
          v[e] = cmul_f(src[i + e], c);
          if (tp.W) v[e] = cmul_f(v[e], wrow[r0 + i + e]);
        }
    }
    if (!tp.W && tp.n && p < K) {  // tail weights without the table: per-unit loop
      for (int e = 0; e < 2; ++e) {
        if (i + e >= rows) continue;
        const unsigned ii = (unsigned)(r0 + i + e);
        for (int u = 0; u < tp.n; ++u) {
          unsigned mk = smask[u], x = 0;
          for (int q = 0; mk; ++q, mk &= mk - 1) x |= ((ii >> (__ffs(mk) - 1)) & 1u) << q;
          v[e] = cmul_f(v[e], __ldg(&ttab[base[u] + x]));
        }
      }
    }
    __nv_bfloat162 h_re, h_im, l_re, l_im, m_re, m_im;
    split3(v[0].x, h_re.x, l_re.x, m_re.x);
    split3(v[1].x, h_re.y, l_re.y, m_re.y);
    split3(v[0].y, h_im.x, l_im.x, m_im.x);
    split3(v[1].y, h_im.y, l_im.y, m_im.y);
    const long long o0 = (2 * p) * lda + i, o1 = o0 + lda;
    *reinterpret_cast<__nv_bfloat162*>(hi + o0) = h_re;
    *reinterpret_cast<__nv_bfloat162*>(hi + o1) = h_im;
    if (lo) {
      *reinterpret_cast<__nv_bfloat162*>(lo + o0) = l_re;
      *reinterpret_cast<__nv_bfloat162*>(lo + o1) = l_im;
    }
    if (lo2) {
      *reinterpret_cast<__nv_bfloat162*>(lo2 + o0) = m_re;
      *reinterpret_cast<__nv_bfloat162*>(lo2 + o1) = m_im;
    }
  }
}

// MN-major B'' (p.mn): row 2p <- (re, im) of B[p][j] at columns (2j, 2j+1),
// row 2p+1 <- (-im, re): the same operand as split_b_kernel's, transposed, so
// each row is one leaf, written elementwise.  One CTA per (path, 512 amplitudes).
// (swapped path-sum: the leaves are half A's, columns col0.. of rows of
// length MS, times c_p when cp is given)
__global__ void split_b_mn_kernel(const float2* __restrict__ leaves, __nv_bfloat16* __restrict__ hi,
                                  __nv_bfloat16* __restrict__ lo, long long K, long long ldb, long long MB,
                                  const TailParams tp, const float2* __restrict__ ttab,
                                  __nv_bfloat16* __restrict__ lo2, const float2* __restrict__ cp, long long col0,
                                  long long MS) {
  __shared__ int base[kMaxTail];
  __shared__ unsigned smask[kMaxTail];
  __shared__ long long node;
  const long long p = blockIdx.y;
  const long long j = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 4;  // 4 amplitudes per thread
  if (tp.mapped) {
    if (threadIdx.x < tp.n) {
      const int u = threadIdx.x;
      const int d = (int)(((tp.p0 + p) / tp.stride[u]) % tp.radix[u]);
      base[u] = (int)(tp.off[u] + ((long long)d << __popc(tp.mask[u])));
      smask[u] = tp.mask[u];
    }
    if (threadIdx.x == 0) node = ((tp.p0 + p) / tp.T) % tp.Tt - tp.node0;
    __syncthreads();
  }
  if (2 * j >= ldb) return;
  float2 v[4];
  const long long row = tp.mapped ? node : p;
  const float2* __restrict__ wrow = tp.W ? tp.W + ((tp.p0 + p) % tp.T) * tp.wld + col0 : nullptr;
  const float2 cpv = cp && p < K ? cp[p] : make_float2(1.f, 0.f);
  if (p < K && j + 4 <= MB && (tp.W || !tp.n) && ((col0 & 1) == 0)) {
    const float2* __restrict__ src = leaves + row * MS + col0 + j;
    float2 w[4];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const float4 a4 = *reinterpret_cast<const float4*>(src + 2 * e);
      v[2 * e] = make_float2(a4.x, a4.y);
      v[2 * e + 1] = make_float2(a4.z, a4.w);
      if (tp.W) {
        const float4 w4 = *reinterpret_cast<const float4*>(wrow + j + 2 * e);
        w[2 * e] = make_float2(w4.x, w4.y);
        w[2 * e + 1] = make_float2(w4.z, w4.w);
      } else {
        w[2 * e] = w[2 * e + 1] = make_float2(1.f, 0.f);
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = cmul_f(v[e], w[e]);
  } else
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    v[e] = make_float2(0.f, 0.f);
    if (p < K && j + e < MB) {
      v[e] = leaves[row * MS + col0 + j + e];
      if (tp.W) {
        v[e] = cmul_f(v[e], wrow[j + e]);
      } else if (tp.n) {
        const unsigned ii = (unsigned)(col0 + j + e);
        for (int u = 0; u < tp.n; ++u) {
          unsigned mk = smask[u], x = 0;
          for (int q = 0; mk; ++q, mk &= mk - 1) x |= ((ii >> (__ffs(mk) - 1)) & 1u) << q;
          v[e] = cmul_f(v[e], __ldg(&ttab[base[u] + x]));
        }
      }
    }
  }
  if (cp) {
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = cmul_f(v[e], cpv);
  }
  __align__(16) __nv_bfloat16 h[16], l[16], m[16];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    split3(v[e].x, h[2 * e], l[2 * e], m[2 * e]);
    split3(v[e].y, h[2 * e + 1], l[2 * e + 1], m[2 * e + 1]);
    split3(-v[e].y, h[8 + 2 * e], l[8 + 2 * e], m[8 + 2 * e]);
    split3(v[e].x, h[8 + 2 * e + 1], l[8 + 2 * e + 1], m[8 + 2 * e + 1]);
  }
  const long long o0 = (2 * p) * ldb + 2 * j, o1 = o0 + ldb;
  *reinterpret_cast<uint4*>(hi + o0) = *reinterpret_cast<const uint4*>(h);
  *reinterpret_cast<uint4*>(hi + o1) = *reinterpret_cast<const uint4*>(h + 8);
  if (lo) {
    *reinterpret_cast<uint4*>(lo + o0) = *reinterpret_cast<const uint4*>(l);
    *reinterpret_cast<uint4*>(lo + o1) = *reinterpret_cast<const uint4*>(l + 8);
  }
  if (lo2) {
    *reinterpret_cast<uint4*>(lo2 + o0) = *reinterpret_cast<const uint4*>(m);
    *reinterpret_cast<uint4*>(lo2 + o1) = *reinterpret_cast<const uint4*>(m + 8);
  }
}

}  // namespace tc

// ------------------------------------------------------------------ host side
struct TcDims {
  long long Kpad, rows_pad, nrows_b_pad;  // Kpad in complex; operand rows
  size_t a_bytes, b_bytes;
};

// esz: operand element bytes (2 bf16, 4 tf32)
inline TcDims tc_dims(long long K, long long rows, long long MB, int esz = 2) {
  TcDims d;
  d.Kpad = (K + 31) / 32 * 32;  // 32 complex = 64 elements = one 128 B bf16 row (two tf32 rows)
  d.rows_pad = (rows + tc::BM - 1) / tc::BM * tc::BM;
  d.nrows_b_pad = (2 * MB + tc::BN - 1) / tc::BN * tc::BN;
  d.a_bytes = (size_t)d.rows_pad * d.Kpad * 2 * esz;  // Kpad complex = 2*Kpad elements
  d.b_bytes = (size_t)d.nrows_b_pad * d.Kpad * 2 * esz;
  return d;
}

// planes: 1 (bf16x1), 2 (bf16x3: hi, lo), 3 (bf16x6: hi, lo, lo2)
// planes 4 = tf32x3 (hi, lo in fp32 storage)
inline size_t tc_workspace_bytes(long long K, long long rows, long long MB, int planes) {
  TcDims d = tc_dims(K, rows, MB, planes == 4 ? 4 : 2);
  if (planes == 4) planes = 2;
  return (size_t)planes * (((d.a_bytes + 1023) & ~(size_t)1023) + ((d.b_bytes + 1023) & ~(size_t)1023));
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      fail(HSF_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    fn = (PFN_encodeTiled)p;
  }
  return fn;
}

// bf16 [rows][cols_bf16] with row stride ld_bf16 (>= cols; boxes past the
// extent read zeros), boxes of BK x box_rows, 128B swizzle
// (tf32: fp32 elements, boxes of 32 = the same 128 B rows)
inline CUtensorMap make_map(void* base, long long rows, long long cols_bf16, int box_rows, long long ld_bf16 = 0,
                            bool tf32 = false) {
  CUtensorMap m;
  const int esz = tf32 ? 4 : 2;
  cuuint64_t dims[2] = {(cuuint64_t)cols_bf16, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld_bf16 ? ld_bf16 : cols_bf16) * esz};
  cuuint32_t box[2] = {(cuuint32_t)(128 / esz), (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(&m, tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base,
                            dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(HSF_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

// fp32 output [rows][cols] (row-major, cols = 2*MB), 32x32 boxes, 128B swizzle
inline CUtensorMap make_out_map(float* base, long long rows, long long cols) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(HSF_ERR_CUDA, "cuTensorMapEncodeTiled (output) failed (" + std::to_string((int)r) + ")");
  return m;
}

inline int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

struct TcBuffers {
  TcDims d;
  __nv_bfloat162 *a_hi, *a_lo, *b_hi, *b_lo;
  __nv_bfloat162 *a_l2 = nullptr, *b_l2 = nullptr;  // bf16x6 third planes
  int planes = 2;
  bool tf32 = false;  // tf32x3: fp32-storage K-major operands, kind::tf32
  bool mn = false;    // operands MN-major: A''^T [2*Kpad][rows_pad], B''^T [2*Kpad][nrows_b_pad] bf16
  bool bk = false;    // with mn: B K-major instead, pair tiles bn columns wide (tc_swap_buffers)
  int bn = tc::BN;
  long long K = 0;    // paths (operand k extent before padding)
};

// Operand layout: MN-major (elementwise prep, B's fusable into half B's last
// pass) for long K; K-major when the GEMM has <= 2 k-blocks (c4: write-bound,
// measured 37.2 vs 40.0 ms with an MN-major B).  HSF_TC_BMN=0/1 forces either.
inline bool tc_mn(long long K) {
  const char* e = std::getenv("HSF_TC_BMN");
  if (e && (e[0] == '0' || e[0] == '1')) return e[0] == '1';
  return 2 * ((K + 31) / 32 * 32) > 2 * tc::BK;
}

inline TcBuffers tc_buffers(long long K, long long rows, long long MB, int planes, void* ws, size_t ws_bytes) {
  TcBuffers t;
  t.d = tc_dims(K, rows, MB, planes == 4 ? 4 : 2);
  if (tc_workspace_bytes(K, rows, MB, planes) > ws_bytes) fail(HSF_ERR_INVALID_ARG, "tc workspace too small");
  t.tf32 = planes == 4;
  if (t.tf32) planes = 2;
  t.planes = planes;
  const bool x3 = planes >= 2;
  char* w = (char*)ws;
  auto take = [&](size_t b) {
    char* r = w;
    w += (b + 1023) & ~(size_t)1023;
    return r;
  };
  t.a_hi = (__nv_bfloat162*)take(t.d.a_bytes);
  t.b_hi = (__nv_bfloat162*)take(t.d.b_bytes);
  t.a_lo = x3 ? (__nv_bfloat162*)take(t.d.a_bytes) : nullptr;
  t.b_lo = x3 ? (__nv_bfloat162*)take(t.d.b_bytes) : nullptr;
  t.a_l2 = planes >= 3 ? (__nv_bfloat162*)take(t.d.a_bytes) : nullptr;
  t.b_l2 = planes >= 3 ? (__nv_bfloat162*)take(t.d.b_bytes) : nullptr;
  t.mn = !t.tf32 && tc_mn(K);
  t.K = K;
  return t;
}

// swapped path-sum (few output rows): A'' = half B's leaves MN-major (2^nB
// GEMM rows), B'' = the MB output rows of half A (c_p, rotation) K-major, one
// pair tile of bn = 32 * ceil(2 MB / 32) columns -- the big operand is read
// once and the narrow one stays in L2
inline TcBuffers tc_swap_buffers(long long K, long long rows, long long MB, int planes, void* ws, size_t ws_bytes) {
  TcBuffers t = tc_buffers(K, rows, MB, planes, ws, ws_bytes);
  if (!t.mn || t.tf32) fail(HSF_ERR_UNSUPPORTED, "swapped path-sum needs MN-major bf16 operands");
  t.bk = true;
  t.bn = (int)((2 * MB + 31) / 32 * 32);
  return t;
}

// K4 for half A (c_p folded) — may run on its own stream
inline void tc_prep_a(const TcBuffers& t, const float2* leavesA, const float2* cp, long long K, long long MA,
                      long long r0, long long rows, const tc::TailParams& tp, const float2* ttab, cudaStream_t st) {
  if (t.mn) {
    const long long lda = t.d.rows_pad;
    tc::split_a_mn_kernel<<<dim3((unsigned)((lda + 2047) / 2048), (unsigned)t.d.Kpad), 256, 0, st>>>(
        leavesA, cp, (__nv_bfloat16*)t.a_hi, (__nv_bfloat16*)t.a_lo, K, lda, MA, r0, rows, tp, ttab,
        (__nv_bfloat16*)t.a_l2);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(HSF_ERR_CUDA, std::string("split_a_mn: ") + cudaGetErrorString(e));
    return;
  }
  const dim3 ga((unsigned)(t.d.rows_pad / 32), (unsigned)(t.d.Kpad / 32));
  if (t.tf32)
    tc::split_a_kernel<float2><<<ga, dim3(32, 8), 0, st>>>(leavesA, cp, (float2*)t.a_hi, (float2*)t.a_lo, K, t.d.Kpad,
                                                           MA, r0, rows, tp, ttab, nullptr);
  else
    tc::split_a_kernel<__nv_bfloat162><<<ga, dim3(32, 8), 0, st>>>(leavesA, cp, t.a_hi, t.a_lo, K, t.d.Kpad, MA, r0,
                                                                   rows, tp, ttab, t.a_l2);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(HSF_ERR_CUDA, std::string("split_a: ") + cudaGetErrorString(e));
}

// K4 for half B — may run on its own stream
// (swapped path-sum: leavesB are half A's leaves, columns col0.. of rows of
// length MS, with c_p; MN-major layout only)
inline void tc_prep_b(const TcBuffers& t, const float2* leavesB, long long K, long long MB,
                      const tc::TailParams& tp, const float2* ttab, cudaStream_t st, const float2* cp = nullptr,
                      long long col0 = 0, long long MS = 0) {
  if (t.mn && !t.bk) {
    const long long ldb = t.d.nrows_b_pad;
    tc::split_b_mn_kernel<<<dim3((unsigned)((ldb / 8 + 255) / 256), (unsigned)t.d.Kpad), 256, 0, st>>>(
        leavesB, (__nv_bfloat16*)t.b_hi, (__nv_bfloat16*)t.b_lo, K, ldb, MB, tp, ttab, (__nv_bfloat16*)t.b_l2, cp,
        col0, MS ? MS : MB);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(HSF_ERR_CUDA, std::string("split_b_mn: ") + cudaGetErrorString(e));
    return;
  }
  const dim3 gb((unsigned)(t.d.nrows_b_pad / 64), (unsigned)(t.d.Kpad / 32));
  if (t.tf32)
    tc::split_b_kernel<float2><<<gb, dim3(32, 8), 0, st>>>(leavesB, (float2*)t.b_hi, (float2*)t.b_lo, K, t.d.Kpad, MB,
                                                           tp, ttab, nullptr, cp, col0, MS ? MS : MB);
  else
    tc::split_b_kernel<__nv_bfloat162><<<gb, dim3(32, 8), 0, st>>>(leavesB, t.b_hi, t.b_lo, K, t.d.Kpad, MB, tp, ttab,
                                                                   t.b_l2, cp, col0, MS ? MS : MB);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(HSF_ERR_CUDA, std::string("split_b: ") + cudaGetErrorString(e));
}

// K5: the persistent tcgen05 GEMM over operand rows [row0, row0 + rows)
// (row0 a multiple of BM) into out[rows][2*MB] fp32
// shards (fused reduce-scatter): n_shards device pointers (local or peer-GPU
// memory), shard o receiving rows [o*shard_rows, (o+1)*shard_rows) of this
// call by TMA reduce-add; `out` unused then
inline void tc_gemm(const TcBuffers& t, float2* out, long long MB, long long row0, long long rows,
                    cudaStream_t st, bool accumulate = false, void* const* shards = nullptr, int n_shards = 0,
                    long long shard_rows = 0) {
  const bool x3 = t.planes >= 2, x6 = t.planes >= 3, tf = t.tf32;
  const long long kcols = 2 * t.d.Kpad;  // elements per K-major operand row
  if (row0 % tc::BM) fail(HSF_ERR_INVALID_ARG, "tc_gemm row offset not tile aligned");
  const long long rpad = (rows + tc::BM - 1) / tc::BM * tc::BM;
  if (row0 + rpad > t.d.rows_pad) fail(HSF_ERR_INVALID_ARG, "tc_gemm rows out of range");
  // K-major A rows from row0 (bf16 pairs 4 B, tf32 pairs 8 B per complex)
  auto ka = [&](void* base) { return (void*)((char*)base + (size_t)row0 * t.d.Kpad * (tf ? 8 : 4)); };
  // MN-major A: columns [row0, row0 + rows) of [2K][rows_pad], 64 x BK boxes
  __nv_bfloat16* a_hi_mn = (__nv_bfloat16*)t.a_hi + row0;
  __nv_bfloat16* a_lo_mn = x3 ? (__nv_bfloat16*)t.a_lo + row0 : nullptr;
  CUtensorMap mAh = t.mn ? make_map(a_hi_mn, 2 * t.K, rows, tc::BK, t.d.rows_pad)
                         : make_map(ka(t.a_hi), rpad, kcols, tc::BM, 0, tf);
  // MN-major B: [2K][2MB] valid of [kcols][nrows_b_pad] storage, 64 x BK
  // boxes; the padding rows / columns are read as zeros (TMA OOB fill), so
  // producers need not write them (operand-store passes do not)
  const bool bk = t.mn && t.bk;  // K-major B of the swapped path-sum, {BK, bn/2} boxes
  if (bk && (t.bn % 32 || t.bn > tc::BN || 2 * MB > t.bn)) fail(HSF_ERR_INVALID_ARG, "narrow tile too small");
  CUtensorMap mBh = bk ? make_map(t.b_hi, t.d.nrows_b_pad, kcols, t.bn / 2)
                  : t.mn ? make_map(t.b_hi, 2 * t.K, 2 * MB, tc::BK, t.d.nrows_b_pad)
                           : make_map(t.b_hi, t.d.nrows_b_pad, kcols, tc::BN, 0, tf);
  CUtensorMap mAl = !x3 ? mAh
                   : t.mn ? make_map(a_lo_mn, 2 * t.K, rows, tc::BK, t.d.rows_pad)
                          : make_map(ka(t.a_lo), rpad, kcols, tc::BM, 0, tf);
  CUtensorMap mBl = !x3 ? mBh
                   : bk ? make_map(t.b_lo, t.d.nrows_b_pad, kcols, t.bn / 2)
                   : t.mn ? make_map(t.b_lo, 2 * t.K, 2 * MB, tc::BK, t.d.nrows_b_pad)
                            : make_map(t.b_lo, t.d.nrows_b_pad, kcols, tc::BN, 0, tf);
  // bf16x6 third planes (pair kernel only)
  CUtensorMap mA2 = mAh, mB2 = mBh;
  if (x6) {
    mA2 = t.mn ? make_map((__nv_bfloat16*)t.a_l2 + row0, 2 * t.K, rows, tc::BK, t.d.rows_pad)
               : make_map(t.a_l2 + row0 * t.d.Kpad, rpad, kcols, tc::BM);
    mB2 = bk ? make_map(t.b_l2, t.d.nrows_b_pad, kcols, t.bn / 2)
        : t.mn ? make_map(t.b_l2, 2 * t.K, 2 * MB, tc::BK, t.d.nrows_b_pad)
               : make_map(t.b_l2, t.d.nrows_b_pad, kcols, tc::BN / 2);
  }
  tc::Params p;
  p.num_m = (int)(rpad / tc::BM);
  p.bk = bk ? 1 : 0;
  p.bn = bk ? t.bn : tc::BN;
  p.num_n = bk ? (int)((2 * MB + t.bn - 1) / t.bn) : (int)(t.d.nrows_b_pad / tc::BN);
  p.num_k = (int)(kcols / (tf ? tc::BK / 2 : tc::BK));
  p.x3 = x3 ? 1 : 0;
  p.x6 = x6 ? 1 : 0;
  p.n_maps = 0;
  p.rows_per_map = 0;
  tc::OutMaps om;
  std::memset(&om, 0, sizeof(om));
  if (n_shards > 0) {
    if (n_shards > tc::kMaxOutMaps || shard_rows % (2 * tc::BM) || shard_rows * n_shards != rows)
      fail(HSF_ERR_INVALID_ARG, "fused reduce-scatter: 1..8 shards of a multiple of 256 rows covering all rows");
    for (int o = 0; o < n_shards; ++o) om.m[o] = make_out_map((float*)shards[o], shard_rows, 2 * MB);
    p.n_maps = n_shards;
    p.rows_per_map = (int)shard_rows;
  }
  p.accumulate = accumulate ? 1 : 0;
  p.mn = t.mn ? 1 : 0;
  // M-fastest raster: the ~148 concurrent tiles share one B tile (read once
  // from DRAM) and sweep A; A stays L2-resident (evict-last) when it is small
  // (c4: 64 MiB for hi+lo), while the streaming output stores are evict-first.
  // (N-fastest re-reads all of B per row block: 7 GB of DRAM reads per 1/16
  // of c4, ncu profiles/r01.)
  p.n_fastest = 0;
  // short K (c4: output-write-bound): grouped raster, 16 row blocks per
  // column sweep -- concurrent tiles write longer contiguous row segments
  // (c4 36.8 -> 35.0 ms; B re-read once per group, 4 GB)
  // long K (c2): groups of 8 pair row blocks, so concurrent tiles share fewer
  // A rows and B columns in L2 (c2 GEMM 0.816 -> 0.809 ms against M-fastest)
  p.group_m = p.num_k <= 2 ? 16 : 8;
  if (const char* g = std::getenv("HSF_TC_GROUP_M")) p.group_m = std::atoi(g);

  p.a_evict_last = ((long long)t.planes * rpad * kcols * (tf ? 4 : 2) <= (64ll << 20)) ? 1 : 0;
  p.out = (float*)out;
  p.ldo = 2 * MB;
  p.rows = rows;
  p.cols = 2 * MB;
  static bool attr = false;
  cudaError_t e;
  if (!attr) {
    e = cudaFuncSetAttribute(tc::tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM_BYTES);
    if (e != cudaSuccess) fail(HSF_ERR_CUDA, std::string("tc smem attr: ") + cudaGetErrorString(e));
    attr = true;
  }
  CUtensorMap mO = n_shards > 0 ? om.m[0] : make_out_map((float*)out, rows, 2 * MB);
  const char* pair_env = std::getenv("HSF_TC_PAIR");
  // (bf16x6: the pair kernel only -- three planes do not fit two single-CTA stages)
  const bool pair = bk || x6 || tf || n_shards > 0 || (rows > tc::BM && !(pair_env && pair_env[0] == '0'));
  if (pair) {
    // CTA pairs: 256-row M tiles, each CTA loads half of every B tile
    static bool attr2 = false;
    if (!attr2) {
      e = cudaFuncSetAttribute(tc::tc_gemm2_kernel<3, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               tc::smem2_bytes(3, 1));
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(tc::tc_gemm2_kernel<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 tc::smem2_bytes(2, 2));
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(tc::tc_gemm2_kernel<2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 tc::smem2_bytes(2, 1, 3));
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(tc::tc_gemm2_kernel<3, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 tc::smem2_bytes(3, 1));
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(tc::tc_gemm2_kernel<2, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 tc::smem2_bytes(2, 2));
      if (e != cudaSuccess) fail(HSF_ERR_CUDA, std::string("tc2 smem attr: ") + cudaGetErrorString(e));
      attr2 = true;
    }
    CUtensorMap mBh2 = t.mn ? mBh : make_map(t.b_hi, t.d.nrows_b_pad, kcols, tc::BN / 2, 0, tf);
    CUtensorMap mBl2 = t.mn ? mBl : x3 ? make_map(t.b_lo, t.d.nrows_b_pad, kcols, tc::BN / 2, 0, tf) : mBh2;
    p.num_m = (int)((rows + 2 * tc::BM - 1) / (2 * tc::BM));
    const long long tiles = (long long)p.num_m * p.num_n;
    const int grid = 2 * (int)std::min<long long>(tiles, num_sms() / 2);
    if (bk) {  // narrow B slots: as many stages of the M operand in flight as fit (5 for bn <= 128 at x3)
      const int bsl = (t.bn / 2 * 128 + 1023) / 1024 * 1024, npl = x6 ? 3 : 2;
      // (227 KB opt-in limit less the kernel's static barriers)
      const int budget = 232448 - 1024 - tc::EPI_WARPS * 4096 - 1024;
      const int fit = budget / (npl * (tc::A_TILE + bsl));
      const int nst = fit >= 5 ? 5 : fit >= 3 ? 3 : 2;
      const int smem = nst * npl * (tc::A_TILE + bsl) + tc::EPI_WARPS * 4096 + 1024;
      static int attr5 = 0, attr3 = 0, attr2n = 0;
      int& cur = nst == 5 ? attr5 : nst == 3 ? attr3 : attr2n;
      if (smem > cur) {
        e = cudaFuncSetAttribute(nst == 5 ? (const void*)tc::tc_gemm2_kernel<5, 1>
                                 : nst == 3 ? (const void*)tc::tc_gemm2_kernel<3, 1>
                                            : (const void*)tc::tc_gemm2_kernel<2, 1>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) fail(HSF_ERR_CUDA, std::string("tc2 narrow smem attr: ") + cudaGetErrorString(e));
        cur = smem;
      }
      const CUtensorMap& a2 = x6 ? mA2 : mAh;
      const CUtensorMap& b2 = x6 ? mB2 : mBh2;
      if (nst == 5)
        tc::tc_gemm2_kernel<5, 1><<<grid, tc::THREADS, smem, st>>>(mAh, mAl, mBh2, mBl2, a2, b2, mO, p, om);
      else if (nst == 3)
        tc::tc_gemm2_kernel<3, 1><<<grid, tc::THREADS, smem, st>>>(mAh, mAl, mBh2, mBl2, a2, b2, mO, p, om);
      else
        tc::tc_gemm2_kernel<2, 1><<<grid, tc::THREADS, smem, st>>>(mAh, mAl, mBh2, mBl2, a2, b2, mO, p, om);
    } else if (tf && p.num_k <= 2)
      tc::tc_gemm2_kernel<2, 2, true><<<grid, tc::THREADS, tc::smem2_bytes(2, 2), st>>>(mAh, mAl, mBh2, mBl2, mAh, mBh2,
                                                                                        mO, p, om);
    else if (tf)
      tc::tc_gemm2_kernel<3, 1, true><<<grid, tc::THREADS, tc::smem2_bytes(3, 1), st>>>(mAh, mAl, mBh2, mBl2, mAh, mBh2,
                                                                                        mO, p, om);
    else if (x6)  // 2 stages x 96 KB + one staging box per epilogue warp
      tc::tc_gemm2_kernel<2, 1><<<grid, tc::THREADS, tc::smem2_bytes(2, 1, 3), st>>>(mAh, mAl, mBh2, mBl2, mA2, mB2,
                                                                                     mO, p, om);
    else if (p.num_k <= 2)
      tc::tc_gemm2_kernel<2, 2><<<grid, tc::THREADS, tc::smem2_bytes(2, 2), st>>>(mAh, mAl, mBh2, mBl2, mAh, mBh2,
                                                                                  mO, p, om);
    else
      tc::tc_gemm2_kernel<3, 1><<<grid, tc::THREADS, tc::smem2_bytes(3, 1), st>>>(mAh, mAl, mBh2, mBl2, mAh, mBh2,
                                                                                  mO, p, om);
  } else {
    const long long tiles = (long long)p.num_m * p.num_n;
    const int grid = (int)std::min<long long>(tiles, num_sms());
    tc::tc_gemm_kernel<<<grid, tc::THREADS, tc::SMEM_BYTES, st>>>(mAh, mAl, mBh, mBl, mO, p);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) fail(HSF_ERR_CUDA, std::string("tc_gemm: ") + cudaGetErrorString(e));
}

}  // namespace hsf
