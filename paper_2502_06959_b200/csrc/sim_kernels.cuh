// sim_kernels.cuh — batched half-state simulator (K1 SMEM-resident tier and
// K2 HBM/L2-streamed tile-pass tier in one kernel).
//
// One CTA owns one (path-tree node, tile) pair: it loads 2^t amplitudes of
// that node's half-state into shared memory, applies every op of the pass
// (fixed local gates and the node's Schmidt factors X_{u,d}/Y_{u,d})
// and writes the tile back.  t == m is the SMEM-resident tier (whole half-state
// on chip, one pass per tree level).  t < m is the streamed tier: tile qubits T
// always include qubits 0..4 so every global access is a 256 B (c64) row;
// diagonal ops are applied to any qubit (their non-tile bits are fixed per
// tile); dense ops only touch tile qubits (the host pass planner guarantees it).
//
// Thread mapping: element e of the tile is owned by thread e % blockDim for
// load, diagonal sweeps and store, so only dense ops need __syncthreads().
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "hsf_internal.h"

namespace hsf {

template <typename R>
struct cplx;
template <>
struct cplx<float> {
  using T = float2;
};
template <>
struct cplx<double> {
  using T = double2;
};

template <typename C>
__device__ __forceinline__ C cmul(C a, C b) {
  C r;
  r.x = a.x * b.x - a.y * b.y;
  r.y = a.x * b.y + a.y * b.x;
  return r;
}
template <typename C>
__device__ __forceinline__ C cfma(C a, C b, C acc) {  // acc + a*b
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
  return acc;
}

// two consecutive amplitudes (16 B for complex64: one LDG.128 / STG.128)
__device__ __forceinline__ void ld2(const float2* p, float2& a, float2& b) {
  const float4 x = *reinterpret_cast<const float4*>(p);
  a = make_float2(x.x, x.y);
  b = make_float2(x.z, x.w);
}
__device__ __forceinline__ void ld2(const double2* p, double2& a, double2& b) {
  a = p[0];
  b = p[1];
}
__device__ __forceinline__ void st2(float2* p, float2 a, float2 b) {
  *reinterpret_cast<float4*>(p) = make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ void st2(double2* p, double2 a, double2 b) {
  p[0] = a;
  p[1] = b;
}

// SMEM layout of a tile: element e lives at sw(e) = e ^ ((e >> 4) & 15).  The
// XOR folds index bits 4..7 into the bank bits 0..3, so the register passes
// (a thread owns the 16 amplitudes spanned by 4 tile qubits, often qubits
// 0..3) and the 1/2-qubit sweeps hit 16 distinct 8-byte bank slots per
// half-warp instead of one.  sw is an involution (bits 4..7 are unchanged).
__device__ __forceinline__ int sw(int e) { return e ^ ((e >> 4) & 15); }

// in-place layout conversion linear <-> swizzled (bulk-copied whole states)
template <typename C, int NT>
__device__ __forceinline__ void swizzle_inplace(C* s, int nel) {
  for (int e = threadIdx.x; e < nel; e += NT) {
    const int f = sw(e);
    if (f > e) {
      const C a = s[e], b = s[f];
      s[e] = b;
      s[f] = a;
    }
  }
}

constexpr int kSimThreads = 256;      // default CTA (3 CTAs/SM at <= 85 regs)
constexpr int kSimThreadsWide = 512;  // narrow tree levels: one wide CTA per node
constexpr int kMaxNonTile = 32;

struct PassParams {
  const void* src;         // parent level buffer, nullptr => |0...0>
  void* dst;               // output level buffer (node-major [nodes][2^m])
  const DevOp* ops;
  const void* coef;        // complex table in the run dtype
  int n_ops;
  int m, t;
  int n_hi;                // t - 5 when t < m
  int T_hi[8];             // half qubits at tile positions 5..t-1
  int n_nt;                // m - t
  int nonT[kMaxNonTile];   // half qubits outside the tile, ascending
  long long state_elems;   // 2^m
  long long node_first;    // global index (at the output level) of blockIdx.y == 0
  unsigned tile0;          // tile index of blockIdx.x == 0 (row-restricted leaf passes)
  long long node_local0;   // local output-node index of blockIdx.y == 0
  long long src_first;     // global index of the first node of the input level
  long long src_div;       // parent = node_global / src_div
  int tbl_elems;           // SMEM diagonal-table area (complex elements)
  unsigned tile_free;      // ~0u: tiles tile0 + blockIdx.x; else tile = deposit(blockIdx.x into
                           // the set bits of tile_free) | tile0 (row light-cone of earlier passes)
};

// the blockIdx.x-th tile of a row-restricted pass (see tile_free)
__device__ __forceinline__ uint32_t restricted_tile(uint32_t id, uint32_t tile0, uint32_t free_mask) {
  if (free_mask == 0xFFFFFFFFu) return id + tile0;
  uint32_t t = tile0;
  for (uint32_t m = free_mask; m; m &= m - 1, id >>= 1) t |= (id & 1u) ? (m & (0u - m)) : 0u;
  return t;
}

template <int K, typename C>
__device__ __forceinline__ void apply_dense_k(C* s, int t, const DevOp& op, const C* __restrict__ M) {
  constexpr int D = 1 << K;
  int ps[K];
#pragma unroll
  for (int j = 0; j < K; ++j) ps[j] = op.q[j];
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int b = a + 1; b < K; ++b)
      if (ps[b] < ps[a]) {
        int tmp = ps[a];
        ps[a] = ps[b];
        ps[b] = tmp;
      }
  const int ngroups = 1 << (t - K);
  if (K == 1) {
    int off[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      int o = 0;
#pragma unroll
      for (int j = 0; j < K; ++j) o |= ((i >> j) & 1) << op.q[j];
      off[i] = o;
    }
    C mat[D * D];
#pragma unroll
    for (int i = 0; i < D * D; ++i) mat[i] = M[i];
    for (int g = threadIdx.x; g < ngroups; g += blockDim.x) {
      int b = g;
#pragma unroll
      for (int j = 0; j < K; ++j) b = ((b >> ps[j]) << (ps[j] + 1)) | (b & ((1 << ps[j]) - 1));
      C v[D];
#pragma unroll
      for (int i = 0; i < D; ++i) v[i] = s[sw(b + off[i])];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        C acc;
        acc.x = 0;
        acc.y = 0;
#pragma unroll
        for (int j = 0; j < D; ++j) acc = cfma(mat[i * D + j], v[j], acc);
        s[sw(b + off[i])] = acc;
      }
    }
  } else {
    for (int g = threadIdx.x; g < ngroups; g += blockDim.x) {
      int b = g;
#pragma unroll
      for (int j = 0; j < K; ++j) b = ((b >> ps[j]) << (ps[j] + 1)) | (b & ((1 << ps[j]) - 1));
      C v[D];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        int o = 0;
#pragma unroll
        for (int j = 0; j < K; ++j) o |= ((i >> j) & 1) << op.q[j];
        v[i] = s[sw(b + o)];
      }
#pragma unroll 1
      for (int i = 0; i < D; ++i) {
        C acc;
        acc.x = 0;
        acc.y = 0;
#pragma unroll
        for (int j = 0; j < D; ++j) acc = cfma(__ldg(&M[i * D + j]), v[j], acc);
        int o = 0;
        for (int j = 0; j < K; ++j) o |= ((i >> j) & 1) << op.q[j];
        s[sw(b + o)] = acc;
      }
    }
  }
}

// Wide dense ops (4, 5 qubits): one group of 2^K amplitudes per 2^K lanes;
// each lane holds one input amplitude and computes one output row, the
// other inputs arrive by warp shuffles (all reads precede the write).
template <int K, typename C>
__device__ __forceinline__ void apply_dense_shfl(C* s, int t, const DevOp& op, const C* __restrict__ M) {
  constexpr int GS = 1 << K, GPW = 32 / GS;
  int ps[K];
#pragma unroll
  for (int j = 0; j < K; ++j) ps[j] = op.q[j];
#pragma unroll
  for (int a = 0; a < K; ++a)
#pragma unroll
    for (int b = a + 1; b < K; ++b)
      if (ps[b] < ps[a]) {
        int tmp = ps[a];
        ps[a] = ps[b];
        ps[b] = tmp;
      }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int sub = lane / GS, r = lane % GS;
  int off = 0;
#pragma unroll
  for (int j = 0; j < K; ++j) off |= ((r >> j) & 1) << op.q[j];
  const int ngroups = 1 << (t - K);
  for (int g0 = wid * GPW; g0 < ngroups; g0 += nw * GPW) {
    const int g = g0 + sub;
    const bool ok = g < ngroups;
    int b = ok ? g : 0;
#pragma unroll
    for (int j = 0; j < K; ++j) b = ((b >> ps[j]) << (ps[j] + 1)) | (b & ((1 << ps[j]) - 1));
    C v = s[sw(b + off)];
    C acc;
    acc.x = 0;
    acc.y = 0;
#pragma unroll 4
    for (int j = 0; j < GS; ++j) {
      C vj;
      vj.x = __shfl_sync(0xffffffffu, v.x, sub * GS + j);
      vj.y = __shfl_sync(0xffffffffu, v.y, sub * GS + j);
      acc = cfma(__ldg(&M[r * GS + j]), vj, acc);
    }
    if (ok) s[sw(b + off)] = acc;
  }
}

template <typename C>
__device__ __forceinline__ void apply_dense(C* s, int t, const DevOp& op, const C* M) {
  switch (op.k) {
    case 1: apply_dense_k<1>(s, t, op, M); break;
    case 2: apply_dense_k<2>(s, t, op, M); break;
    case 3: apply_dense_k<3>(s, t, op, M); break;
    case 4: apply_dense_shfl<4>(s, t, op, M); break;
    case 5: apply_dense_shfl<5>(s, t, op, M); break;
    default: break;
  }
}

// table index of a diagonal op: bit j <- state bit q[j]; fast path for up to
// three contiguous runs of qubits
__device__ __forceinline__ uint32_t diag_idx(const DevOp& d, uint32_t g) {
  if (d.nruns == 0) {
    uint32_t idx = 0;
    for (int j = 0; j < d.k; ++j) idx |= ((g >> d.q[j]) & 1u) << j;
    return idx;
  }
  uint32_t idx = (g >> d.rshift[0]) & ((1u << d.rlen[0]) - 1u);
  if (d.nruns > 1) idx |= ((g >> d.rshift[1]) & ((1u << d.rlen[1]) - 1u)) << d.roff[1];
  if (d.nruns > 2) idx |= ((g >> d.rshift[2]) & ((1u << d.rlen[2]) - 1u)) << d.roff[2];
  return idx;
}

// Branch-free two-run index in registers (runs beyond the second use the
// generic path).
struct DiagIdx {
  uint32_t s0, m0, s1, m1, o1;
  bool slow;
  __device__ __forceinline__ void load(const DevOp& d) {
    slow = d.nruns == 0 || d.nruns > 2;
    s0 = d.rshift[0];
    m0 = (1u << d.rlen[0]) - 1u;
    s1 = d.nruns > 1 ? d.rshift[1] : 0u;
    m1 = d.nruns > 1 ? (1u << d.rlen[1]) - 1u : 0u;
    o1 = d.nruns > 1 ? d.roff[1] : 0u;
  }
  __device__ __forceinline__ uint32_t operator()(const DevOp& d, uint32_t g) const {
    if (slow) return diag_idx(d, g);
    return ((g >> s0) & m0) | (((g >> s1) & m1) << o1);
  }
};

template <int J, typename C>
__device__ __forceinline__ void reg_apply1(C (&v)[16], const C m00, const C m01, const C m10, const C m11) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (i & (1 << J)) continue;
    const C a = v[i], b = v[i | (1 << J)];
    C x, y;
    x.x = 0;
    x.y = 0;
    y = x;
    x = cfma(m00, a, x);
    x = cfma(m01, b, x);
    y = cfma(m10, a, y);
    y = cfma(m11, b, y);
    v[i] = x;
    v[i | (1 << J)] = y;
  }
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Whole-state tier: the node state is one contiguous block, moved by the TMA
// bulk-copy engine (cp.async.bulk) with an mbarrier transaction count.
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  const uint32_t b = smem_addr(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  for (uint32_t off = 0; off < bytes; off += 65536u) {
    const uint32_t n = min(65536u, bytes - off);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr((const char*)sdst + off)),
                 "l"((const char*)gsrc + off), "r"(n), "r"(b)
                 : "memory");
  }
}
__device__ __forceinline__ void mbar_wait0(uint64_t* bar) {
  const uint32_t b = smem_addr(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "W_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
      "@!P1 bra W_%=;\n"
      "}\n" ::"r"(b)
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
  for (uint32_t off = 0; off < bytes; off += 65536u) {
    const uint32_t n = min(65536u, bytes - off);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"((char*)gdst + off),
                 "r"(smem_addr((const char*)ssrc + off)), "r"(n)
                 : "memory");
  }
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem may be released
}

// HEAVY = register passes and 3..5-qubit dense ops compiled in (128 regs,
// 2 CTAs/SM); light passes (diagonals + 1/2-qubit SMEM sweeps) run a lean
// variant at 4 CTAs/SM.  The host picks the variant per pass.
template <typename R, int NT, bool HEAVY>
__global__ void __launch_bounds__(NT, (NT == 256 ? (HEAVY ? 2 : 4) : 1)) hsf_pass_kernel(const PassParams p) {
  using C = typename cplx<R>::T;
  constexpr int CH = (NT == 256 && HEAVY) ? 8 : 4;  // elements per thread in registers for diagonal sweeps
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t load_bar;
  C* s = reinterpret_cast<C*>(smem_raw);
  size_t off = sizeof(C) << p.t;
  uint32_t* hi_off = reinterpret_cast<uint32_t*>(smem_raw + off);
  off += (p.t < p.m) ? (sizeof(uint32_t) << (p.t - 5)) : 0;
  off = (off + 15) & ~(size_t)15;
  DevOp* sops = reinterpret_cast<DevOp*>(smem_raw + off);
  off += sizeof(DevOp) * p.n_ops;
  const C** sM = reinterpret_cast<const C**>(smem_raw + off);  // per-op matrix for this node's digit
  off += sizeof(void*) * p.n_ops;
  off = (off + 15) & ~(size_t)15;
  C* stab = reinterpret_cast<C*>(smem_raw + off);  // staged diagonal tables

  const uint32_t tile = restricted_tile(blockIdx.x, p.tile0, p.tile_free);
  const long long node_local = p.node_local0 + blockIdx.y;
  const long long node_g = p.node_first + blockIdx.y;
  const int nel = 1 << p.t;
  const bool whole = (p.t == p.m);
  const C* coef = reinterpret_cast<const C*>(p.coef);

  const C* src = nullptr;
  if (p.src) {
    const long long parent = node_g / p.src_div - p.src_first;
    src = reinterpret_cast<const C*>(p.src) + parent * p.state_elems;
  }
  C* dst = reinterpret_cast<C*>(p.dst) + node_local * p.state_elems;
  const bool bulk = whole && src != nullptr;
  // kick off the state load first so it overlaps the op staging below
  if (bulk && threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&load_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    bulk_load(s, src, (uint32_t)(sizeof(C) << p.t), &load_bar);
  }

  uint32_t base = 0;
  if (!whole) {
    for (int j = 0; j < p.n_nt; ++j) base |= ((tile >> j) & 1u) << p.nonT[j];
    const int nh = 1 << p.n_hi;
    for (int j = threadIdx.x; j < nh; j += NT) {
      uint32_t o = 0;
      for (int b = 0; b < p.n_hi; ++b) o |= (uint32_t)((j >> b) & 1) << p.T_hi[b];
      hi_off[j] = o;
    }
  }
  for (int i = threadIdx.x; i < p.n_ops; i += NT) {
    const DevOp d = p.ops[i];
    sops[i] = d;
    const long long digit = (d.radix > 1) ? (node_g / d.div) % d.radix : 0;
    sM[i] = (d.kind == OP_DIAG && d.soff >= 0) ? stab + d.soff : coef + d.table + digit * d.stride;
  }
  __syncthreads();
  if (p.tbl_elems > 0) {
    // stage this node's digit-resolved small diagonal tables (one warp per op)
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x >> 5; i < p.n_ops; i += NT / 32) {
      const DevOp& d = sops[i];
      if (d.kind != OP_DIAG || d.soff < 0) continue;
      const long long digit = (d.radix > 1) ? (node_g / d.div) % d.radix : 0;
      const C* g = coef + d.table + digit * d.stride;
      for (int e = lane; e < (1 << d.k); e += 32) stab[d.soff + e] = __ldg(&g[e]);
    }
  }
  auto gidx_of = [&](int e) -> uint32_t { return whole ? (uint32_t)e : (base | (e & 31) | hi_off[e >> 5]); };

  if (bulk) {
    mbar_wait0(&load_bar);
    __syncthreads();
    swizzle_inplace<C, NT>(s, nel);
  } else if (src) {
    // tiled tier: pairs (e, e+1) are contiguous in global memory (tile
    // position 0 is qubit 0); LB 16-byte requests in flight per thread
    constexpr int LB = 4;
    for (int e0 = 2 * threadIdx.x; e0 < nel; e0 += 2 * NT * LB) {
      C a[LB], b[LB];
#pragma unroll
      for (int u = 0; u < LB; ++u) {
        const int e = e0 + 2 * NT * u;
        if (e < nel) ld2(src + gidx_of(e), a[u], b[u]);
      }
#pragma unroll
      for (int u = 0; u < LB; ++u) {
        const int e = e0 + 2 * NT * u;
        if (e < nel) {
          s[sw(e)] = a[u];
          s[sw(e + 1)] = b[u];
        }
      }
    }
  } else {
    for (int e = threadIdx.x; e < nel; e += NT) {
      C v;
      v.x = (gidx_of(e) == 0) ? R(1) : R(0);
      v.y = R(0);
      s[sw(e)] = v;
    }
  }
  __syncthreads();  // state and staged tables visible to every mapping below

  // mapping discipline: standalone diagonal sweeps use the element-owner
  // mapping (e % NT); dense sweeps and register passes use group mappings and
  // are bracketed by barriers
  int i = 0;
  while (i < p.n_ops) {
    const int kind = sops[i].kind;
    if (kind == OP_DENSE) {
      __syncthreads();
      if (HEAVY) {
        apply_dense<C>(s, p.t, sops[i], sM[i]);
      } else {
        if (sops[i].k == 1)
          apply_dense_k<1>(s, p.t, sops[i], sM[i]);
        else
          apply_dense_k<2>(s, p.t, sops[i], sM[i]);
      }
      __syncthreads();
      ++i;
    } else if (HEAVY && kind == OP_RPASS) {
      const DevOp& h = sops[i];
      const int n = h.k;
      int ps[kRegQ];
      uint32_t ebit[kRegQ], gbit[kRegQ];  // tile-index and state-index bit of each register qubit
#pragma unroll
      for (int j = 0; j < kRegQ; ++j) {
        const int pos = h.q[j];
        ps[j] = pos;
        ebit[j] = 1u << pos;
        gbit[j] = 1u << (whole || pos < 5 ? pos : p.T_hi[pos - 5]);
      }
#pragma unroll
      for (int a = 0; a < kRegQ; ++a)
#pragma unroll
        for (int b = a + 1; b < kRegQ; ++b)
          if (ps[b] < ps[a]) {
            int tmp = ps[a];
            ps[a] = ps[b];
            ps[b] = tmp;
          }
      __syncthreads();
      const int ngr = 1 << (p.t - kRegQ);
      for (int gi = threadIdx.x; gi < ngr; gi += NT) {
        int b = gi;
#pragma unroll
        for (int j = 0; j < kRegQ; ++j) b = ((b >> ps[j]) << (ps[j] + 1)) | (b & ((1 << ps[j]) - 1));
        const uint32_t gb = gidx_of(b);
        C v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          uint32_t e = (uint32_t)b;
#pragma unroll
          for (int j = 0; j < kRegQ; ++j)
            if ((k >> j) & 1) e |= ebit[j];
          v[k] = s[sw(e)];
        }
        for (int r = i + 1; r <= i + n; ++r) {
          const DevOp& d = sops[r];
          const C* M = sM[r];
          if (d.kind == OP_R1) {
            const C m00 = M[0], m01 = M[1], m10 = M[2], m11 = M[3];
            switch (d.q[0]) {
              case 0: reg_apply1<0>(v, m00, m01, m10, m11); break;
              case 1: reg_apply1<1>(v, m00, m01, m10, m11); break;
              case 2: reg_apply1<2>(v, m00, m01, m10, m11); break;
              default: reg_apply1<3>(v, m00, m01, m10, m11); break;
            }
          } else {
            // the table index is a bitwise gather, so
            // idx(gb | gbit[j] | ...) = idx(gb) | ibit[j] | ...
            DiagIdx di;
            di.load(d);
            const uint32_t i0 = di(d, gb);
            uint32_t ib[kRegQ];
#pragma unroll
            for (int j = 0; j < kRegQ; ++j) ib[j] = di(d, gbit[j]);
            const C* T = (d.soff >= 0) ? stab + d.soff : M;
            const bool sh = d.soff >= 0;
#pragma unroll
            for (int hk = 0; hk < 16; hk += 8) {
              C tv[8];
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                uint32_t x = i0;
#pragma unroll
                for (int j = 0; j < kRegQ; ++j)
                  if (((hk + k) >> j) & 1) x |= ib[j];
                tv[k] = sh ? T[x] : __ldg(&T[x]);
              }
#pragma unroll
              for (int k = 0; k < 8; ++k) v[hk + k] = cmul(v[hk + k], tv[k]);
            }
          }
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          uint32_t e = (uint32_t)b;
#pragma unroll
          for (int j = 0; j < kRegQ; ++j)
            if ((k >> j) & 1) e |= ebit[j];
          s[sw(e)] = v[k];
        }
      }
      __syncthreads();
      i += n + 1;
    } else {
      // standalone run of diagonal ops, element-owner mapping, CH elements
      // per thread in registers (CH independent table loads per op)
      int j = i;
      while (j < p.n_ops && sops[j].kind == OP_DIAG) ++j;
      for (int e0 = threadIdx.x; e0 < nel; e0 += CH * NT) {
        C v[CH];
        uint32_t g[CH];
#pragma unroll
        for (int u = 0; u < CH; ++u) {
          const int e = e0 + u * NT;
          if (e < nel) {
            v[u] = s[sw(e)];
            g[u] = gidx_of(e);
          }
        }
        for (int r = i; r < j; ++r) {
          const DevOp& d = sops[r];
          DiagIdx di;
          di.load(d);
          C tv[CH];
          if (d.soff >= 0) {
            const C* T = stab + d.soff;
#pragma unroll
            for (int u = 0; u < CH; ++u) tv[u] = T[(e0 + u * NT < nel) ? di(d, g[u]) : 0];
          } else {
            const C* T = sM[r];
#pragma unroll
            for (int u = 0; u < CH; ++u) tv[u] = __ldg(&T[(e0 + u * NT < nel) ? di(d, g[u]) : 0]);
          }
#pragma unroll
          for (int u = 0; u < CH; ++u) v[u] = cmul(v[u], tv[u]);
        }
#pragma unroll
        for (int u = 0; u < CH; ++u) {
          const int e = e0 + u * NT;
          if (e < nel) s[sw(e)] = v[u];
        }
      }
      i = j;
    }
  }
  __syncthreads();
  if (whole) {
    swizzle_inplace<C, NT>(s, nel);
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
      bulk_store(dst, s, (uint32_t)(sizeof(C) << p.t));
    }
  } else {
    for (int e = 2 * threadIdx.x; e < nel; e += 2 * NT) st2(dst + gidx_of(e), s[sw(e)], s[sw(e + 1)]);
  }
}

}  // namespace hsf
