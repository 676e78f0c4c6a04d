// jit_prelude.cuh — device helpers shared by every run-time specialised
// simulator pass (jit.cpp generates one kernel per tile pass and compiles it
// with NVRTC for sm_100a).  Self-contained: NVRTC sees only this text plus
// the generated kernel, no system headers.
//
// Semantics are those of hsf_pass_kernel (sim_kernels.cuh): one CTA owns one
// (path-tree node, tile) pair, the tile lives in shared memory with the
// padded layout sw(e) = e + e/16 + e/256 + e/4096 (additive over disjoint bits), and the pass's ops are
// applied in order.  In the generated kernels every qubit position, table
// offset, digit divisor and loop bound is a compile-time constant.
typedef unsigned int u32;
typedef unsigned long long u64;

struct JitArgs {
  const void* src;       // parent level buffer, nullptr => |0...0>
  void* dst;             // output level buffer (node-major)
  const void* coef;      // complex table in the run dtype
  long long node_first;  // global index (output level) of blockIdx.y == 0
  long long node_local0; // local output-node index of blockIdx.y == 0
  long long src_first;   // global index of the first node of the input level
  long long src_div;     // parent = node_global / src_div
  unsigned tile0;        // tile index of blockIdx.x == 0 (row-restricted leaf passes)
  void* dst_lo;          // operand-store passes: lo plane of the split-bf16 B operand (nullptr => hi only)
  long long ldw;         //   and its row stride in 32-bit words (bf16 pairs)
  unsigned tile_free;    // ~0u: tile = tile0 + blockIdx; else deposit(blockIdx into its set bits) | tile0
};
__device__ __forceinline__ u32 restricted_tile(u32 id, u32 tile0, u32 free_mask) {
  if (free_mask == 0xFFFFFFFFu) return id + tile0;
  u32 t = tile0;
  for (u32 m = free_mask; m; m &= m - 1, id >>= 1) t |= (id & 1u) ? (m & (0u - m)) : 0u;
  return t;
}

__device__ __forceinline__ int sw(int e) { return e + (e >> 4) + (e >> 8) + (e >> 12); }

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cfma(float2 a, float2 b, float2 acc) {
  acc.x = fmaf(a.x, b.x, fmaf(-a.y, b.y, acc.x));
  acc.y = fmaf(a.x, b.y, fmaf(a.y, b.x, acc.y));
  return acc;
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
  return acc;
}
// packed FP32 (sm_100 FFMA2 / FMUL2): both components of a complex64 in one
// instruction; a scalar factor broadcast to both lanes is an immediate
__device__ __forceinline__ unsigned long long pk2(float2 a) { return *reinterpret_cast<unsigned long long*>(&a); }
__device__ __forceinline__ float2 up2(unsigned long long a) { return *reinterpret_cast<float2*>(&a); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)), "l"(pk2(c)));
  return up2(d);
}
// a + s b (s a literal): the scaled rotation's update, one FFMA2 with a broadcast immediate
__device__ __forceinline__ float2 axpy2(float s, float2 b, float2 a) { return fma2(b, make_float2(s, s), a); }
template <typename C>
__device__ __forceinline__ C czero();
template <>
__device__ __forceinline__ float2 czero<float2>() { return make_float2(0.f, 0.f); }
template <>
__device__ __forceinline__ double2 czero<double2>() { return make_double2(0.0, 0.0); }

// two consecutive amplitudes from / to global memory (16 B for complex64)
// HSF_LD_MODE / HSF_ST_MODE (env HSF_JIT_LDST = 10 * ld + st, measurement
// only): cache operators of the passes' 16 B state loads / stores -- 0 default,
// 1 .cg (L2 only), 2 .cs (streaming, evict first), 3 store .wt
#ifndef HSF_LD_MODE
#define HSF_LD_MODE 0
#endif
#ifndef HSF_ST_MODE
#define HSF_ST_MODE 0
#endif
__device__ __forceinline__ void ld2(const float2* p, float2& a, float2& b) {
#if HSF_LD_MODE == 1
  const float4 x = __ldcg(reinterpret_cast<const float4*>(p));
#elif HSF_LD_MODE == 2
  const float4 x = __ldcs(reinterpret_cast<const float4*>(p));
#else
  const float4 x = *reinterpret_cast<const float4*>(p);
#endif
  a = make_float2(x.x, x.y);
  b = make_float2(x.z, x.w);
}
__device__ __forceinline__ void ld2(const double2* p, double2& a, double2& b) {
  a = p[0];
  b = p[1];
}
__device__ __forceinline__ void st2(float2* p, float2 a, float2 b) {
#if HSF_ST_MODE == 1
  __stcg(reinterpret_cast<float4*>(p), make_float4(a.x, a.y, b.x, b.y));
#elif HSF_ST_MODE == 2
  __stcs(reinterpret_cast<float4*>(p), make_float4(a.x, a.y, b.x, b.y));
#elif HSF_ST_MODE == 3
  __stwt(reinterpret_cast<float4*>(p), make_float4(a.x, a.y, b.x, b.y));
#else
  *reinterpret_cast<float4*>(p) = make_float4(a.x, a.y, b.x, b.y);
#endif
}
__device__ __forceinline__ void st2(double2* p, double2 a, double2 b) {
  p[0] = a;
  p[1] = b;
}

// Operand-store passes (half B's last pass of a full-output tensor-core run):
// instead of the leaf, write rows 2k and 2k+1 of the MN-major split-bf16 B
// operand -- (re, im) and (-im, re) of each amplitude at word G -- hi plane
// and, if present, the lo plane (x - bf16(x)), RNE conversions (cvt.rn)
__device__ __forceinline__ u32 bf2(float lo_half, float hi_half) {
  u32 d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi_half), "f"(lo_half));
  return d;
}
__device__ __forceinline__ float bf_lo(u32 d) { return __uint_as_float(d << 16); }
__device__ __forceinline__ float bf_hi(u32 d) { return __uint_as_float(d & 0xFFFF0000u); }
__device__ __forceinline__ void st_bop(const JitArgs& a, long long k, u32 g, float2 x, float2 y) {
  u32* hi = reinterpret_cast<u32*>(a.dst);
  const long long o0 = 2 * k * a.ldw + g, o1 = o0 + a.ldw;
  const u32 h0 = bf2(x.x, x.y), h1 = bf2(y.x, y.y), r0 = bf2(-x.y, x.x), r1 = bf2(-y.y, y.x);
  *reinterpret_cast<uint2*>(hi + o0) = make_uint2(h0, h1);
  *reinterpret_cast<uint2*>(hi + o1) = make_uint2(r0, r1);
  if (a.dst_lo) {
    u32* lo = reinterpret_cast<u32*>(a.dst_lo);
    *reinterpret_cast<uint2*>(lo + o0) =
        make_uint2(bf2(x.x - bf_lo(h0), x.y - bf_hi(h0)), bf2(y.x - bf_lo(h1), y.y - bf_hi(h1)));
    *reinterpret_cast<uint2*>(lo + o1) =
        make_uint2(bf2(-x.y - bf_lo(r0), x.x - bf_hi(r0)), bf2(-y.y - bf_lo(r1), y.x - bf_hi(r1)));
  }
}
__device__ __forceinline__ void st_bop(const JitArgs&, long long, u32, double2, double2) {}
// swapped path-sum: rows 2k (Re) and 2k+1 (Im) of the MN-major split-bf16 M
// operand (tc_swap_buffers' A''), amplitudes G and G+1 as one bf16 pair per
// row; a.ldw = the row length in 4 B words
__device__ __forceinline__ void st_aop(const JitArgs& a, long long k, u32 g, float2 x, float2 y) {
  u32* hi = reinterpret_cast<u32*>(a.dst);
  const long long o0 = 2 * k * a.ldw + (g >> 1), o1 = o0 + a.ldw;
  const u32 hr = bf2(x.x, y.x), hm = bf2(x.y, y.y);
  hi[o0] = hr;
  hi[o1] = hm;
  if (a.dst_lo) {
    u32* lo = reinterpret_cast<u32*>(a.dst_lo);
    lo[o0] = bf2(x.x - bf_lo(hr), y.x - bf_hi(hr));
    lo[o1] = bf2(x.y - bf_lo(hm), y.y - bf_hi(hm));
  }
}
__device__ __forceinline__ void st_aop(const JitArgs&, long long, u32, double2, double2) {}

// 1-qubit gate on register slot J of 16 amplitudes held by one thread
template <int J, typename C>
__device__ __forceinline__ void r1(C (&v)[16], const C* __restrict__ M) {
  const C m00 = __ldg(&M[0]), m01 = __ldg(&M[1]), m10 = __ldg(&M[2]), m11 = __ldg(&M[3]);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (i & (1 << J)) continue;
    const C a = v[i], b = v[i | (1 << J)];
    v[i] = cfma(m01, b, cmul(m00, a));
    v[i | (1 << J)] = cfma(m11, b, cmul(m10, a));
  }
}

// cluster tier helpers: rank in the cluster, generic pointer to the same
// shared-memory variable in CTA `r` of the cluster (DSMEM), cluster barrier
__device__ __forceinline__ u32 cluster_rank() {
  u32 r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
template <typename T>
__device__ __forceinline__ T* map_rank(T* p, u32 r) {
  u64 out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(reinterpret_cast<u64>(p)), "r"(r));
  return reinterpret_cast<T*>(out);
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// same with the matrix entries as compile-time literals (fixed gates)
template <int J, typename C>
__device__ __forceinline__ void r1c(C (&v)[16], const C m00, const C m01, const C m10, const C m11) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (i & (1 << J)) continue;
    const C a = v[i], b = v[i | (1 << J)];
    v[i] = cfma(m01, b, cmul(m00, a));
    v[i | (1 << J)] = cfma(m11, b, cmul(m10, a));
  }
}

// insert a zero bit at position P (ascending use: smallest position first)
template <int P>
__device__ __forceinline__ u32 ins0(u32 b) {
  return ((b >> P) << (P + 1)) | (b & ((1u << P) - 1u));
}
