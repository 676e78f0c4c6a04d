// jit.cpp — run-time specialisation of the simulator tile passes.
//
// For every tile pass of a plan (both halves, both tree variants) the host
// generates one CUDA kernel in which every qubit position, tile map, table
// offset, digit divisor and loop bound of the pass's op list is a
// compile-time constant, compiles it with NVRTC for sm_100a (once per
// distinct source per process and device, in parallel host threads) and
// launches it through the driver API.  The generated kernels compute exactly
// what the generic interpreter kernel hsf_pass_kernel (sim_kernels.cuh)
// computes for the same pass -- same CTA/tile/node mapping, same swizzled
// shared-memory layout, same op order -- without its per-op dispatch and
// variable-shift index arithmetic (ncu on the interpreter: FFMA was 20 % of
// the issued instructions, profiles/r01).
#include <cctype>
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "hsf_internal.h"
#include "jit.h"

namespace hsf {

static const char* kPrelude =
#include "jit_prelude.inc"
    ;

// ------------------------------------------------------------ code generation
namespace {

std::string u(uint64_t v) {
  char b[32];
  std::snprintf(b, sizeof b, "%lluu", (unsigned long long)v);
  return b;
}

// expression gathering bits: sum_j ((x >> from[j]) & 1) << to[j], merged into runs
std::string gather_expr(const std::string& x, const std::vector<int>& from, const std::vector<int>& to) {
  std::vector<std::string> terms;
  size_t j = 0;
  while (j < from.size()) {
    size_t e = j + 1;
    while (e < from.size() && from[e] == from[e - 1] + 1 && to[e] == to[e - 1] + 1) ++e;
    const int len = (int)(e - j);
    const uint64_t mask = (len >= 32) ? 0xffffffffull : ((1ull << len) - 1);
    std::string t = "((" + x + " >> " + std::to_string(from[j]) + ") & " + u(mask) + ")";
    if (to[j]) t = "(" + t + " << " + std::to_string(to[j]) + ")";
    terms.push_back(t);
    j = e;
  }
  if (terms.empty()) return "0u";
  std::string s = terms[0];
  for (size_t i = 1; i < terms.size(); ++i) s += " | " + terms[i];
  return "(" + s + ")";
}

// shared-memory tile layout (8 B / 16 B elements), same as the prelude's
// sw(): a padded index e + e/16 + e/256 + e/4096.  Every 4-bit group of the
// index adds onto the bank bits, so any 4 register positions leave lane
// positions of every residue mod 4 (distinct banks per half-warp, see rpass);
// and the map is additive over disjoint bits (no carry out of a group), so a
// register access is base + constant: an immediate LDS / STS offset instead
// of an XOR per access (c5 B leaf pass: ~96 LOP3 per thread)
static uint32_t swz(uint32_t e) { return e + (e >> 4) + (e >> 8) + (e >> 12); }
// padded tile size in elements
static uint32_t padded(int t) { return swz((1u << t) - 1u) + 1u; }

// T-leaf group stride: tile + tables, then padded to 16 mod 64 bytes.  In the
// transposed store a half-warp reads 4 consecutive rows e (8 contiguous
// words after the swizzle) of the column groups c2 = 0, 2, 4, 6: strides of
// 4 mod 16 words put them at word offsets 0, 8, 16, 24 (t1: 4, 12, 20, 28), so
// each half-warp covers the 32 banks once (ncu: the 32 mod 64 B stride
// left 2-way conflicts, 4 wavefronts per load instead of 2)
static size_t tleaf_group_bytes(int t, long long tbl_elems, size_t elem) {
  return ((((elem * padded(t)) + (size_t)tbl_elems * elem) + 63) & ~(size_t)63) + 16;
}

struct Gen {
  std::ostringstream o;
  const Half& H;
  const Pass& ps;
  bool c64;
  int t, m;
  bool whole;
  std::vector<DevOp> ops;
  std::vector<int> pos2q;  // tile position -> half qubit

  const std::vector<cd>* coef = nullptr;  // plan master table (fp64): fixed-gate literals

  Gen(const Half& h, const Pass& p, bool c, const std::vector<cd>* cf) : H(h), ps(p), c64(c), coef(cf) {
    t = p.t;
    m = h.m;
    whole = (t == m);
    ops.assign(h.dev_ops.begin() + p.op_begin, h.dev_ops.begin() + p.op_end);
    pos2q.resize(t);
    for (int i = 0; i < t; ++i) pos2q[i] = whole ? i : p.T[i];
    if (const char* e = std::getenv("HSF_JIT_GIVENS")) givens = std::atoi(e) != 0;
    if (const char* e = std::getenv("HSF_JIT_TPAD")) tpad = std::atoi(e) != 0;
    packed = c64;
    if (const char* e = std::getenv("HSF_JIT_PACKED")) packed = c64 && std::atoi(e) != 0;
  }

  std::string table(int i) const { return "M" + std::to_string(i); }

  // direct register passes: the pass's first register pass loads its 16
  // amplitudes straight from the parent state and its last one stores them
  // straight to the node state (no tile copy through shared memory on either
  // side: two shared-memory round trips and two barriers fewer per tile; the
  // B leaf pass of c5 is bound by the L1 / shared-memory pipe)
  bool direct_ld = false, direct_st = false;
  bool tpad = true;  // staged tables at the padded index (HSF_JIT_TPAD=0: plain)
  std::string TP() const { return tpad ? "e + (e >> 4)" : "e"; }
  // G(e) without the tile's base: G is bit-linear, G(b | e) = G(b) | fmap(e)
  uint32_t fmap(uint32_t e) const {
    if (whole) return e;
    uint32_t g = 0;
    for (int i = 0; i < t; ++i)
      if ((e >> i) & 1u) g |= 1u << pos2q[i];
    return g;
  }
  bool any_staged() const {
    for (auto& d : ops)
      if (staged(d)) return true;
    return false;
  }
  // T-leaf: one group's shared memory (its tile + staged tables; 16 B more so
  // consecutive groups' tiles start on different banks)
  size_t group_bytes() const { return tleaf_group_bytes(t, ps.tbl_elems, c64 ? 8 : 16); }
  // fixed (non-factor) gate entries become literals in the generated code: no
  // dependent table loads on the gate chain (exact: %a of the run-dtype value)
  bool literal(const DevOp& d) const { return coef && d.radix <= 1 && (d.kind == OP_R1 || d.kind == OP_DENSE); }
  std::string lit(int64_t idx) const {
    const cd v = (*coef)[(size_t)idx];
    char b[128];
    if (c64)
      std::snprintf(b, sizeof b, "make_float2(%af, %af)", (double)(float)v.real(), (double)(float)v.imag());
    else
      std::snprintf(b, sizeof b, "make_double2(%a, %a)", v.real(), v.imag());
    return b;
  }
  // one real literal of the run dtype
  std::string rl(double x) const {
    char b[64];
    if (c64)
      std::snprintf(b, sizeof b, "%af", (double)(float)x);
    else
      std::snprintf(b, sizeof b, "%a", x);
    return b;
  }
  // 1-qubit literal gate on register slot J of the 16 register amplitudes,
  // written out per pair with the terms of exactly-zero matrix parts dropped:
  // RX (real diagonal, imaginary off-diagonal) and H (real) cost 4 real
  // multiply-adds per amplitude instead of 8 (the QAOA mixers of c4 / q*)
  void r1_literal(int J, const DevOp& d) {
    cd m[4];
    for (int e = 0; e < 4; ++e) {
      const cd v = (*coef)[(size_t)(d.table + e)];
      m[e] = c64 ? cd((float)v.real(), (float)v.imag()) : v;
    }
    // out.re = sum_j (m_j.re x_j.re - m_j.im x_j.im); out.im = sum_j (m_j.re x_j.im + m_j.im x_j.re)
    auto expr = [&](const cd& m0, const cd& m1, bool im) {
      struct T {
        double c;
        std::string x;
      };
      std::vector<T> ts;
      auto add = [&](double c, const std::string& x) {
        if (c != 0.0) ts.push_back({c, x});
      };
      if (!im) {
        add(m0.real(), "a.x");
        add(-m0.imag(), "a.y");
        add(m1.real(), "b.x");
        add(-m1.imag(), "b.y");
      } else {
        add(m0.real(), "a.y");
        add(m0.imag(), "a.x");
        add(m1.real(), "b.y");
        add(m1.imag(), "b.x");
      }
      if (ts.empty()) return rl(0.0);
      std::string e = ts[0].x + " * " + rl(ts[0].c);
      for (size_t k = 1; k < ts.size(); ++k) e = std::string(c64 ? "fmaf(" : "fma(") + ts[k].x + ", " + rl(ts[k].c) + ", " + e + ")";
      return e;
    };
    const char* mk = c64 ? "make_float2" : "make_double2";
    for (int i = 0; i < 16; ++i) {
      if (i & (1 << J)) continue;
      const int j = i | (1 << J);
      o << "    { const C a = v[" << i << "], b = v[" << j << "]; v[" << i << "] = " << mk << "(" << expr(m[0], m[1], false)
        << ", " << expr(m[0], m[1], true) << "); v[" << j << "] = " << mk << "(" << expr(m[2], m[3], false) << ", "
        << expr(m[2], m[3], true) << "); }\n";
    }
  }
  std::string mat(const DevOp& d, int i, int e) const {
    return literal(d) ? lit(d.table + e) : "__ldg(&" + table(i) + "[" + std::to_string(e) + "])";
  }
  std::string didx(const DevOp& d, const std::string& g) const {
    std::vector<int> from(d.q, d.q + d.k), to(d.k);
    for (int j = 0; j < d.k; ++j) to[j] = j;
    // order by destination bit j (already), merge runs where both advance by 1
    return gather_expr(g, from, to);
  }
  bool staged(const DevOp& d) const { return d.kind == OP_DIAG && d.soff >= 0; }
  // staged tables sit at the padded index x + x/16 (entries x and x + 16 on
  // different banks: the lanes of a register pass differ in high index bits,
  // 2-way conflicts on c5's B leaf pass, ncu r02f); additive over disjoint bits
  std::string tload(const DevOp& d, int i, const std::string& idx) const {
    if (!staged(d)) return "__ldg(&" + table(i) + "[" + idx + "])";
    return tpad ? table(i) + "[(" + idx + ") + ((" + idx + ") >> 4)]" : table(i) + "[" + idx + "]";
  }

  int multi = 0;  // T-leaf variant: leaves per CTA (0 = one node per CTA)
  // T-leaf: the first op is a register pass, which loads straight from the
  // (swizzled) parent tile instead of a per-group copy of it
  bool pb_first = false;
  // T-leaf: one 64-thread group per leaf (its own tile and tables, named
  // barrier 1 + group); elsewhere the whole CTA
  std::string TIDs = "threadIdx.x", SYNCs = "__syncthreads()";

  // tile -> state index map G(e) (uses TILE_ID)
  void emit_G() {
    // tile -> state index map
    if (whole) {
      o << "  auto G = [&](u32 e) -> u32 { return e; };\n";
    } else {
      std::vector<int> nonT;
      for (int q = 0; q < m; ++q)
        if (std::find(ps.T.begin(), ps.T.end(), q) == ps.T.end()) nonT.push_back(q);
      std::vector<int> from(nonT.size()), to = nonT;
      for (size_t j = 0; j < nonT.size(); ++j) from[j] = (int)j;
      o << "  const u32 tile = restricted_tile(TILE_ID >> CB, a.tile0, a.tile_free);\n";
      o << "  const u32 base = " << gather_expr("tile", from, to) << ";\n";
      std::vector<int> pf, pt;
      for (int i = 0; i < t; ++i) {
        pf.push_back(i);
        pt.push_back(pos2q[i]);
      }
      o << "  auto G = [&](u32 e) -> u32 { return base | " << gather_expr("e", pf, pt) << "; };\n";
    }
  }


  // T-leaf: index of the first staged table op (-1: none)
  int first_staged() const {
    for (size_t i = 0; i < ops.size(); ++i)
      if (ops[i].kind != OP_RPASS && staged(ops[i])) return (int)i;
    return -1;
  }
  bool cp_in_table() const { return multi && first_staged() >= 0; }

  // T-leaf kernel head: persistent CTAs over (tile, parent) items; the next
  // item's parent tile is prefetched by cp.async into a double buffer while the
  // groups (one 64-thread group per leaf) evaluate the current one
  void header_multi(const std::string& name, int minb) {
    const size_t elem = c64 ? 8 : 16;
    o << "extern \"C\" __global__ void __launch_bounds__(" << nt << ", " << minb << ") " << name
      << "(const JitArgs a) {\n";
    o << "  typedef " << (c64 ? "float2" : "double2") << " C;\n";
    o << "  constexpr u32 NT = 64u, NEL = 1u << " << t << ";\n";
    o << "  constexpr u32 CB = 0u, LB = " << t << "u, LNEL = 1u << LB;\n  (void)CB; (void)NEL;\n";
    o << "  constexpr u32 RANK = 0u;\n";
    o << "  extern __shared__ __align__(128) unsigned char smem_raw[];\n";
    o << "  const u32 GRP = threadIdx.x >> 6, TID = threadIdx.x & 63u;\n";
    o << "  unsigned char* gbase = smem_raw + GRP * " << group_bytes() << "u;\n";
    o << "  C* s = reinterpret_cast<C*>(gbase);\n";
    o << "  C* stab = reinterpret_cast<C*>(gbase + sizeof(C) * " << padded(t) << "u);\n  (void)stab;\n";
    o << "  constexpr u32 PADL = " << padded(t) << "u;\n";
    o << "  C* pbuf = reinterpret_cast<C*>(smem_raw + " << (size_t)multi * group_bytes() << "u);\n";
    o << "  const C* coef = reinterpret_cast<const C*>(a.coef);\n";
    o << "  const C* srcb = reinterpret_cast<const C*>(a.src);\n";
    o << "  constexpr long long NTILES = " << (1ll << (m - t)) << "ll;\n";
    // items = (tile, parent) with the parent fastest: the CTAs in flight
    // write all K columns of the same rows close together in time, so L2
    // merges whole 1 KiB operand rows before they reach DRAM
    o << "  const u32 NPAR = a.tile_free;  // tile_free = parents\n";
    o << "  const u32 n_items = (u32)NTILES * NPAR;\n";
    // item -> (tile, parent) in 32-bit arithmetic (shift / mask when the
    // parent count is a power of two); parent p's tile sits at src index
    // pb0 + p (node_first is a multiple of src_div == leaves per parent)
    o << "  const bool npow = (NPAR & (NPAR - 1u)) == 0u;\n";
    o << "  const u32 nsh = npow ? (u32)(__ffs(NPAR) - 1) : 0u;\n";
    o << "  auto par_of = [&](u32 it) -> u32 { return npow ? (it & (NPAR - 1u)) : (it % NPAR); };\n";
    o << "  auto til_of = [&](u32 it) -> u32 { return npow ? (it >> nsh) : (it / NPAR); };\n";
    o << "  const long long pb0 = a.node_first / a.src_div - a.src_first;\n";
    // tile map of an item's tile
    std::vector<int> nonT;
    for (int q = 0; q < m; ++q)
      if (std::find(ps.T.begin(), ps.T.end(), q) == ps.T.end()) nonT.push_back(q);
    std::vector<int> from(nonT.size()), to = nonT;
    for (size_t j = 0; j < nonT.size(); ++j) from[j] = (int)j;
    std::vector<int> pf, pt;
    for (int i = 0; i < t; ++i) {
      pf.push_back(i);
      pt.push_back(pos2q[i]);
    }
    o << "  auto base_of = [&](u32 tile) -> u32 { return " << gather_expr("tile", from, to) << "; };\n";
    o << "  auto GE = [&](u32 e) -> u32 { return " << gather_expr("e", pf, pt) << "; };\n";
    o << "  auto prefetch = [&](u32 it, u32 buf) {\n";
    o << "    const u32 parent = par_of(it); const u32 pb = base_of(til_of(it));\n";
    o << "    const C* p_ = srcb + (pb0 + (long long)parent) * " << (1ll << m) << "ll;\n";
    o << "    C* d_ = pbuf + buf * PADL;\n";
    if (pb_first) {
      // swizzled like the group tiles (8 B copies: the swizzle may swap a
      // pair's halves), so the first register pass reads it in place
      o << "    const u32 e0 = threadIdx.x, g0 = pb | GE(e0), s0 = (u32)sw((int)e0);\n";
      o << "    const unsigned sa0 = (unsigned)__cvta_generic_to_shared(d_);\n";
      o << "#pragma unroll\n";
      o << "    for (u32 j = 0; j < LNEL / " << nt << "u; ++j) {\n";
      o << "      const u32 ej = j * " << nt << "u;\n";
      o << "      asm volatile(\"cp.async.ca.shared.global [%0], [%1], 8;\" :: \"r\"(sa0 + 8u * (s0 + (u32)sw((int)ej))), "
           "\"l\"(p_ + (g0 | GE(ej))) : \"memory\");\n";
      o << "    }\n";
    } else {
      o << "    for (u32 e = 2u * threadIdx.x; e < LNEL; e += " << 2 * nt << "u) {\n";
      o << "      const unsigned sa = (unsigned)__cvta_generic_to_shared(d_ + e);\n";
      o << "      asm volatile(\"cp.async.cg.shared.global [%0], [%1], 16;\" :: \"r\"(sa), \"l\"(p_ + (pb | GE(e))) : \"memory\");\n";
      o << "    }\n";
    }
    o << "    asm volatile(\"cp.async.commit_group;\" ::: \"memory\");\n  };\n";
    o << "  u32 it = blockIdx.x;\n  u32 buf = 0u;\n";
    // one CTA barrier at the end of an item covers both the group tiles'
    // reuse and the next parent tile's arrival (its copies were issued at the
    // item's start into the buffer the previous item had finished reading)
    o << "  if (it < n_items) prefetch(it, 0u); else asm volatile(\"cp.async.commit_group;\" ::: \"memory\");\n";
    o << "  asm volatile(\"cp.async.wait_group 0;\" ::: \"memory\");\n  __syncthreads();\n";
    o << "  const C* cpt = reinterpret_cast<const C*>(a.dst_lo);\n";
    o << "  const u32 c2 = 2u * (threadIdx.x % " << multi / 2 << "u);\n";
    o << "  for (; it < n_items; it += gridDim.x, buf ^= 1u) {\n";
    o << "  if (it + gridDim.x < n_items) prefetch(it + gridDim.x, buf ^ 1u);\n";
    o << "  else asm volatile(\"cp.async.commit_group;\" ::: \"memory\");\n";
    o << "  const long long parent = par_of(it);\n";
    o << "  const u32 base = base_of(til_of(it));\n";
    o << "  const long long k0 = a.node_local0 + parent * " << multi << "ll;\n";
    // c_p of each group's leaf rides on its first staged table (every
    // amplitude is multiplied by one of its entries); without such a table
    // the store applies the two c_p columns, requested before the evaluation
    o << "  C w0 = czero<C>(), w1 = czero<C>();\n";
    if (!cp_in_table()) o << "  if (cpt) { w0 = cpt[k0 + c2]; w1 = cpt[k0 + c2 + 1u]; }\n";
    else o << "  (void)w0; (void)w1;\n";
    o << "  auto G = [&](u32 e) -> u32 { return base | GE(e); };\n";
    o << "  {\n  const long long node_g = a.node_first + parent * " << multi << "ll + GRP;\n";
    // per-op table pointers (digit-resolved)
    for (size_t i = 0; i < ops.size(); ++i) {
      const DevOp& d = ops[i];
      if (d.kind == OP_RPASS) continue;
      std::string ptr = "coef + " + std::to_string(d.table) + "ll";
      if (d.radix > 1)
        ptr += " + ((node_g / " + std::to_string(d.div) + "ll) % " + std::to_string(d.radix) + "ll) * " +
               std::to_string(d.stride) + "ll";
      if (staged(d)) {
        o << "  C* " << table(i) << " = stab + " << d.soff << ";\n";
        if (cp_in_table() && (int)i == first_staged())
          o << "  { const C* g_ = " << ptr << "; const C cpl = cpt ? cpt[k0 + GRP] : make_" << (c64 ? "float2" : "double2")
            << "(1, 0); for (u32 e = TID; e < " << (1u << d.k) << "u; e += NT) " << table(i)
            << "[" << TP() << "] = cmul(__ldg(&g_[e]), cpl); }\n";
        else
          o << "  { const C* g_ = " << ptr << "; for (u32 e = TID; e < " << (1u << d.k) << "u; e += NT) " << table(i)
            << "[" << TP() << "] = __ldg(&g_[e]); }\n";
      } else {
        o << "  const C* __restrict__ " << table(i) << " = " << ptr << ";\n";
      }
    }
    if (pb_first) {
      o << "  const C* pb_ = pbuf + buf * PADL;\n";
    } else {
      o << "  { const C* pp = pbuf + buf * PADL; for (u32 e = TID; e < LNEL; e += NT) s[sw(e)] = pp[e]; }\n";
      o << "  " << SYNCs << ";\n";
    }
    (void)elem;
  }

  void header(const std::string& name, int minb) {
    if (multi) {
      header_multi(name, minb);
      return;
    }
    o << "extern \"C\" __global__ void __launch_bounds__(" << nt << ", " << minb << ") " << name
      << "(const JitArgs a) {\n";
    o << "  typedef " << (c64 ? "float2" : "double2") << " C;\n";
    o << "  constexpr u32 NT = " << (multi ? 64 : nt) << "u, NEL = 1u << " << t << ";\n";
    // cluster tier (cb > 0): the tile is split over 2^cb CTAs of a cluster by
    // its top cb tile positions; CTA `RANK` holds elements [RANK << LB, +LNEL)
    o << "  constexpr u32 CB = " << cb << "u, LB = " << (t - cb) << "u, LNEL = 1u << LB;\n";
    o << "  (void)CB;\n";
    o << "  extern __shared__ __align__(128) unsigned char smem_raw[];\n";
    if (multi) {
      o << "  const u32 GRP = threadIdx.x >> 6, TID = threadIdx.x & 63u;\n";
      o << "  unsigned char* gbase = smem_raw + GRP * " << group_bytes() << "u;\n";
      o << "  C* s = reinterpret_cast<C*>(gbase);\n";
      o << "  C* stab = reinterpret_cast<C*>(gbase + sizeof(C) * " << padded(t) << "u);\n";
    } else {
      o << "  C* s = reinterpret_cast<C*>(smem_raw);\n";
      o << "  C* stab = reinterpret_cast<C*>(smem_raw + sizeof(C) * " << padded(t - cb) << "u);\n";
    }
    if (cb) {
      o << "  const u32 RANK = cluster_rank();\n";
      o << "  C* sr[" << (1 << cb) << "];\n";
      o << "#pragma unroll\n  for (u32 r = 0; r < " << (1 << cb) << "u; ++r) sr[r] = map_rank(s, r);\n";
      o << "  auto P = [&](u32 e) -> C& { return sr[e >> LB][sw(e & (LNEL - 1u))]; };\n";
    } else {
      o << "  constexpr u32 RANK = 0u;\n";
    }
    o << "  (void)stab;\n";
    // grid: x = tile, y = node (T-leaf: y = parent, its `multi` leaves looped over)
    o << "  const u32 TILE_ID = blockIdx.x;\n";
    o << "  (void)TILE_ID;\n";
    o << "  const C* coef = reinterpret_cast<const C*>(a.coef);\n";
    if (multi) {
      emit_G();
      o << "  {\n  const u32 NODE_ID = blockIdx.y * " << multi << "u + GRP;\n";
    } else {
      o << "  const u32 NODE_ID = blockIdx.y;\n";
    }
    o << "  const long long node_g = a.node_first + NODE_ID;\n";
    o << "  C* dst = reinterpret_cast<C*>(a.dst) + (a.node_local0 + NODE_ID) * " << (1ll << m) << "ll;\n";
    o << "  (void)dst;\n";
    // (a 32-bit division for the parent index whenever the node index fits,
    // as it does below the default path budget of 2^26: ~5x fewer
    // instructions per thread than the 64-bit one)
    o << "  const long long par_g = ((node_g | a.src_div) >> 32) == 0 ? (long long)((unsigned)node_g / (unsigned)a.src_div) : node_g / a.src_div;\n";
    o << "  const C* src = a.src ? reinterpret_cast<const C*>(a.src) + (par_g - a.src_first) * "
      << (1ll << m) << "ll : nullptr;\n";
    if (!multi) emit_G();
    // per-op table pointers (digit-resolved for Schmidt factors)
    for (size_t i = 0; i < ops.size(); ++i) {
      const DevOp& d = ops[i];
      if (d.kind == OP_RPASS) continue;
      std::string ptr = "coef + " + std::to_string(d.table) + "ll";
      if (d.radix > 1)
        ptr += " + ((node_g / " + std::to_string(d.div) + "ll) % " + std::to_string(d.radix) + "ll) * " +
               std::to_string(d.stride) + "ll";
      if (staged(d)) {
        o << "  C* " << table(i) << " = stab + " << d.soff << ";\n";
        o << "  { const C* g_ = " << ptr << "; for (u32 e = " << TIDs << "; e < " << (1u << d.k)
          << "u; e += NT) " << table(i) << "[" << TP() << "] = __ldg(&g_[e]); }\n";
      } else {
        o << "  const C* __restrict__ " << table(i) << " = " << ptr << ";\n";
      }
    }
    // load (or |0...0>).  Unrolled with the thread's element split off: the
    // tile map G and the swizzle are bit-linear over disjoint bits, so
    // G(e0 | ej) = G(e0) | G(ej) and sw(e0 | ej) = sw(e0) ^ sw(ej) with ej a
    // constant per unrolled step (the generic loop spent ~20 integer
    // instructions per pair on them)
    // (direct first register pass: it reads the parent state itself; the tile
    // load stays for the HSF_NO_DIRECT build, see nvrtc_compile)
    if (direct_ld) o << "#ifdef HSF_NO_DIRECT\n";
    o << "  if (src) {\n";
    if (!cb && (1 << t) >= 2 * nt) {
      o << "    const u32 e0 = 2u * " << TIDs << ", g0 = G(e0), s0 = (u32)sw((int)e0);\n";
      o << "#pragma unroll\n";
      o << "    for (u32 j = 0; j < LNEL / (2u * NT); ++j) { const u32 ej = j * 2u * NT; C x_, y_; "
           "ld2(src + (g0 | G(ej)), x_, y_); const u32 sj = s0 + (u32)sw((int)ej); s[sj] = x_; s[sj + 1u] = y_; }\n";
    } else {
      o << "#pragma unroll 4\n";
      o << "    for (u32 e = 2u * " << TIDs << "; e < LNEL; e += 2u * NT) { C x_, y_; ld2(src + G((RANK << LB) | e), x_, y_); "
           "s[sw(e)] = x_; s[sw(e + 1)] = y_; }\n";
    }
    o << "  } else {\n";
    o << "    for (u32 e = " << TIDs << "; e < LNEL; e += NT) { C v_ = czero<C>(); if (G((RANK << LB) | e) == 0u) v_.x = 1; "
         "s[sw(e)] = v_; }\n";
    o << "  }\n";
    o << (cb ? "  cluster_sync();\n" : "  " + SYNCs + ";\n");
    if (direct_ld) o << "#endif\n";
  }

  bool cross(const int* pos, int k) const {
    for (int j = 0; j < k; ++j)
      if (pos[j] >= t - cb) return true;
    return false;
  }
  // element access: local op -> this CTA's SMEM, cross op -> any CTA's (DSMEM)
  std::string el(bool x, const std::string& e) const { return x ? "P(" + e + ")" : "s[sw(" + e + ")]"; }
  void sync_pre(bool x) { o << (x ? std::string("  cluster_sync();\n") : "  " + SYNCs + ";\n"); }
  // loop over groups: local ops walk this CTA's groups, cross ops the whole tile's
  void group_loop(bool x, const std::string& var, int shift) {
    if (x)
      o << "  for (u32 " << var << " = RANK * NT + threadIdx.x; " << var << " < (NEL >> " << shift << "); " << var
        << " += (NT << CB)) {\n";
    else
      o << "  for (u32 " << var << " = " << TIDs << "; " << var << " < (LNEL >> " << shift << "); " << var
        << " += NT) {\n";
  }

  void dense(const DevOp& d, int i) {
    const int K = d.k, D = 1 << K;
    const bool x = cross(d.q, K);
    std::vector<int> sorted(d.q, d.q + K);
    std::sort(sorted.begin(), sorted.end());
    sync_pre(x);
    group_loop(x, "g", K);
    o << "    u32 b = g;";
    for (int p : sorted) o << " b = ins0<" << p << ">(b);";
    o << "\n    C v[" << D << "];\n";
    std::vector<uint32_t> off(D);
    for (int r = 0; r < D; ++r) {
      uint32_t xo = 0;
      for (int j = 0; j < K; ++j)
        if ((r >> j) & 1) xo |= 1u << d.q[j];
      off[r] = xo;
      o << "    v[" << r << "] = " << el(x, "b + " + std::to_string(xo) + "u") << ";\n";
    }
    if (K <= 3) {
      for (int r = 0; r < D; ++r) {
        o << "    { C acc = czero<C>();";
        for (int c = 0; c < D; ++c) o << " acc = cfma(" << mat(d, i, r * D + c) << ", v[" << c << "], acc);";
        o << " " << el(x, "b + " + std::to_string(off[r]) + "u") << " = acc; }\n";
      }
    } else {
      o << "    const u32 offs[" << D << "] = {";
      for (int r = 0; r < D; ++r) o << (r ? ", " : "") << off[r] << "u";
      o << "};\n";
      o << "#pragma unroll 1\n    for (int r = 0; r < " << D << "; ++r) { C acc = czero<C>();\n";
      o << "#pragma unroll\n      for (int c = 0; c < " << D << "; ++c) acc = cfma(__ldg(&" << table(i) << "[r * " << D
        << " + c]), v[c], acc);\n";
      o << "      " << el(x, "b + offs[r]") << " = acc; }\n";
    }
    o << "  }\n";
    sync_pre(x);
  }

  // ---- Euler / fast-Givens form of a register pass's literal 1-qubit gates.
  // A (scaled) unitary 2x2 literal is M = diag(p0, p1) . [[c, -s], [s, c]] .
  // diag(1, q1) (ZYZ Euler form with the phases as diagonals).  Diagonals
  // commute with each other and with gates on other register slots, so the
  // pass's right / left diagonals are carried at code-generation time as
  // separable per-slot factors and applied together, once per round of
  // rotations (a 16-entry product table: <= 15 complex multiplies per 16
  // amplitudes), and each rotation is applied in the scaled form
  // c . [[1, -t], [t, 1]] (t = s / c <= 1; else s . [[u, -1], [1, u]]), one
  // real FMA per component, with the scale folded into the carried constant.
  // A Haar SU(2) then costs 2 FP32 ops per amplitude plus its share of the
  // diagonal flushes instead of 8 (the B leaf / T-leaf passes of c5 are
  // FP32-issue bound).  Table-driven ops (Schmidt factors indexed
  // per node) are emitted as before, scheduled by the same commutation rules.
  bool givens = true;
  // deferral of the pass's final diagonals (see DeferOut): the pending
  // per-qubit phases carried from one register pass to the next and left
  // unapplied at the end
  bool defer = false;
  std::map<int, cd> carry;  // half-local qubit -> phase of |1> (|0> normalised to 1)
  cd carry_scalar = 1.0;
  // c64 rotations as packed FFMA2 with a broadcast immediate (SASS count of
  // c5's B leaf pass 1584 -> 1400; literal complex products stay scalar: their
  // FMUL2 / FFMA2 form needs the constant pairs in registers, 1400 -> 1672)
  bool packed = false;
  struct SOp {
    int kind;        // 0 const diag (slot J), 1 rotation, 2 table diag, 3 table R1, 4 general literal R1
    int J = 0;       // slot (kinds 0, 1, 3, 4)
    unsigned mask;   // slots touched
    cd d0, d1;       // kind 0
    int mode = 0;    // kind 1: 0 t-form, 1 u-form, 2 swap
    double x = 0;    // kind 1: t or u
    double scale = 1;
    size_t r = 0;    // op index (kinds 2, 3, 4)
  };
  static bool is_diag_kind(int k) { return k == 0 || k == 2; }
  std::string cl(const cd& v) const {
    char b[160];
    if (c64)
      std::snprintf(b, sizeof b, "make_float2(%af, %af)", (double)(float)v.real(), (double)(float)v.imag());
    else
      std::snprintf(b, sizeof b, "make_double2(%a, %a)", v.real(), v.imag());
    return b;
  }
  // decompose a literal 1-qubit op on slot J; false => not a scaled unitary
  bool euler(const DevOp& d, std::vector<SOp>& out) {
    const int J = d.q[0];
    cd m[4];
    for (int e = 0; e < 4; ++e) m[e] = (*coef)[(size_t)(d.table + e)];
    const double n0 = std::norm(m[0]) + std::norm(m[1]), n1 = std::norm(m[2]) + std::norm(m[3]);
    if (!(n0 > 0) || !(n1 > 0)) return false;
    const double tol = 1e-12 * (n0 + n1);
    if (std::abs(n0 - n1) > tol || std::abs(m[0] * std::conj(m[2]) + m[1] * std::conj(m[3])) > tol ||
        std::abs(std::norm(m[0]) - std::norm(m[3])) > tol)
      return false;
    SOp a{};
    a.J = J;
    a.mask = 1u << J;
    if (m[1] == cd(0) && m[2] == cd(0)) {  // diagonal
      a.kind = 0;
      a.d0 = m[0];
      a.d1 = m[3];
      out.push_back(a);
      return true;
    }
    if (m[0] == cd(0) && m[3] == cd(0)) {  // anti-diagonal: swap, then diag(m01, m10)
      a.kind = 1;
      a.mode = 2;
      out.push_back(a);
      a.kind = 0;
      a.d0 = m[1];
      a.d1 = m[2];
      out.push_back(a);
      return true;
    }
    const double lam = std::sqrt(n0);
    const double c = std::abs(m[0]) / lam, s = std::abs(m[1]) / lam;
    const cd p0 = m[0] / c, p1 = m[2] / s, q1 = -m[1] / (s * p0);
    a.kind = 0;
    a.d0 = 1.0;
    a.d1 = q1;
    out.push_back(a);
    SOp rt{};
    rt.kind = 1;
    rt.J = J;
    rt.mask = 1u << J;
    if (c >= s) {
      rt.mode = 0;
      rt.x = s / c;
      rt.scale = c;
    } else {
      rt.mode = 1;
      rt.x = c / s;
      rt.scale = s;
    }
    out.push_back(rt);
    a.d0 = p0;
    a.d1 = p1;
    out.push_back(a);
    return true;
  }
  template <typename TD>
  void givens_schedule(size_t i, int n, const int* qreg, TD&& emit_tdiag) {
    std::vector<SOp> sl;
    for (size_t r = i + 1; r <= i + (size_t)n; ++r) {
      const DevOp& d = ops[r];
      if (d.kind == OP_R1) {
        if (literal(d) && euler(d, sl)) continue;
        SOp g{};
        g.kind = literal(d) ? 4 : 3;
        g.J = d.q[0];
        g.mask = 1u << d.q[0];
        g.r = r;
        sl.push_back(g);
      } else {
        SOp g{};
        g.kind = 2;
        g.r = r;
        g.mask = 0;
        for (int j = 0; j < 4; ++j)
          for (int jj = 0; jj < d.k; ++jj)
            if (d.q[jj] == qreg[j]) g.mask |= 1u << j;
        sl.push_back(g);
      }
    }
    // carried constants: per-slot diag(1, pd[J]) and a global scalar gs
    // (deferral: seeded from what earlier register passes left pending)
    cd pd[4] = {1.0, 1.0, 1.0, 1.0};
    cd gs = 1.0;
    if (defer) {
      gs = carry_scalar;
      carry_scalar = 1.0;
      for (int j = 0; j < 4; ++j) {
        auto it = carry.find(qreg[j]);
        if (it != carry.end()) {
          pd[j] = it->second;
          carry.erase(it);
        }
      }
    }
    const char* fm = c64 ? "fmaf" : "fma";
    const char* mk = c64 ? "make_float2" : "make_double2";
    auto flush = [&](unsigned S, bool with_scalar) {
      for (int k = 0; k < 16; ++k) {
        cd f = with_scalar ? gs : cd(1.0);
        for (int j = 0; j < 4; ++j)
          if (((S >> j) & 1) && ((k >> j) & 1)) f *= pd[j];
        if (f == cd(1.0)) continue;
        const std::string v = "v[" + std::to_string(k) + "]";
        const double fr = c64 ? (double)(float)f.real() : f.real(), fi = c64 ? (double)(float)f.imag() : f.imag();
        if (fi == 0.0)
          o << "    " << v << " = " << mk << "(" << v << ".x * " << rl(fr) << ", " << v << ".y * " << rl(fr) << ");\n";
        else if (fr == 0.0)
          o << "    " << v << " = " << mk << "(" << v << ".y * " << rl(-fi) << ", " << v << ".x * " << rl(fi) << ");\n";
        else
          o << "    " << v << " = cmul(" << v << ", " << cl(f) << ");\n";
      }
      for (int j = 0; j < 4; ++j)
        if ((S >> j) & 1) pd[j] = 1.0;
      if (with_scalar) gs = 1.0;
    };
    auto emit_rot = [&](const SOp& s) {
      for (int a = 0; a < 16; ++a) {
        if (a & (1 << s.J)) continue;
        const int b = a | (1 << s.J);
        const std::string va = "v[" + std::to_string(a) + "]", vb = "v[" + std::to_string(b) + "]";
        if (s.mode == 2) {
          o << "    { const C t_ = " << va << "; " << va << " = " << vb << "; " << vb << " = t_; }\n";
        } else if (packed && s.mode == 0) {  // FFMA2 with the broadcast literal
          o << "    { const C a = " << va << ", b = " << vb << "; " << va << " = axpy2(" << rl(-s.x) << ", b, a); " << vb
            << " = axpy2(" << rl(s.x) << ", a, b); }\n";
        } else if (packed) {
          o << "    { const C a = " << va << ", b = " << vb << "; " << va << " = fma2(a, make_float2(" << rl(s.x) << ", "
            << rl(s.x) << "), make_float2(-b.x, -b.y)); " << vb << " = axpy2(" << rl(s.x) << ", b, a); }\n";
        } else if (s.mode == 0) {  // a' = a - t b, b' = b + t a
          const std::string mt = rl(-s.x), pt = rl(s.x);
          o << "    { const C a = " << va << ", b = " << vb << "; " << va << " = " << mk << "(" << fm << "(b.x, " << mt
            << ", a.x), " << fm << "(b.y, " << mt << ", a.y)); " << vb << " = " << mk << "(" << fm << "(a.x, " << pt
            << ", b.x), " << fm << "(a.y, " << pt << ", b.y)); }\n";
        } else {  // a' = u a - b, b' = u b + a
          const std::string u = rl(s.x);
          o << "    { const C a = " << va << ", b = " << vb << "; " << va << " = " << mk << "(" << fm << "(a.x, " << u
            << ", -b.x), " << fm << "(a.y, " << u << ", -b.y)); " << vb << " = " << mk << "(" << fm << "(b.x, " << u
            << ", a.x), " << fm << "(b.y, " << u << ", a.y)); }\n";
        }
      }
    };
    std::vector<char> done(sl.size(), 0);
    auto ready = [&](size_t x) {
      for (size_t y = 0; y < x; ++y)
        if (!done[y] && (sl[y].mask & sl[x].mask) && !(is_diag_kind(sl[x].kind) && is_diag_kind(sl[y].kind)))
          return false;
      return true;
    };
    for (;;) {
      bool any = false;
      for (bool ch = true; ch;) {  // every ready diagonal: carried (constants) or applied now (tables)
        ch = false;
        for (size_t x = 0; x < sl.size(); ++x) {
          if (done[x] || !is_diag_kind(sl[x].kind) || !ready(x)) continue;
          if (sl[x].kind == 0) {
            const SOp& s = sl[x];
            gs *= s.d0;
            pd[s.J] *= s.d1 / s.d0;
          } else {
            emit_tdiag(sl[x].r);
          }
          done[x] = 1;
          ch = any = true;
        }
      }
      std::vector<size_t> round;
      unsigned S = 0;
      for (size_t x = 0; x < sl.size(); ++x)
        if (!done[x] && !is_diag_kind(sl[x].kind) && ready(x)) {
          round.push_back(x);
          if (pd[sl[x].J] != cd(1.0)) S |= 1u << sl[x].J;
        }
      if (round.empty()) {
        if (!any) break;
        continue;
      }
      // (every op is linear, so the global scalar rides to the pass's end)
      if (S) flush(S, false);
      for (size_t x : round) {
        const SOp& s = sl[x];
        if (s.kind == 1) {
          emit_rot(s);
          gs *= s.scale;
        } else if (s.kind == 3) {
          o << "    r1<" << s.J << ">(v, " << table((int)s.r) << ");\n";
        } else {
          r1_literal(s.J, ops[s.r]);
        }
        done[x] = 1;
      }
    }
    if (defer) {  // left pending: later register passes or the gather apply them
      carry_scalar = gs;
      for (int j = 0; j < 4; ++j)
        if (pd[j] != cd(1.0)) carry[qreg[j]] = pd[j];
    } else {
      flush(0xFu, true);
    }
  }

  // register pass: header at ops[i], then ops[i+1 .. i+n]
  void rpass(size_t i) {
    const DevOp& h = ops[i];
    const int n = h.k;
    int pos[4], qreg[4];
    for (int j = 0; j < 4; ++j) {
      pos[j] = h.q[j];
      qreg[j] = pos2q[pos[j]];
    }
    std::vector<int> sorted(pos, pos + 4);
    std::sort(sorted.begin(), sorted.end());
    const bool x = cross(pos, 4);
    const bool dl = direct_ld && i == 0, ds = direct_st && i + (size_t)n + 1 == ops.size();
    if (!dl || any_staged()) sync_pre(x);  // (direct first pass: only staged tables to wait for; HSF_NO_DIRECT: the load's barrier)
    // direct passes unrolled over the thread's groups (as a loop, the global
    // addresses kept live across iterations spill at the 64-register cap: c3)
    if ((dl || ds) && !x) o << "#pragma unroll\n";
    group_loop(x, "gi", 4);
    if (!x && cb == 0 && t > 4) {
      // lane bits -> non-register tile positions, ordered so that the first
      // lanes' swizzled bank indices are linearly independent: sw(e) puts
      // e[0..3] ^ e[4..7] ^ e[8..11] ^ e[12..15] on the bank bits, so each position contributes a
      // GF(2) vector; a half-warp (c64, 8 B) / quarter-warp (c128, 16 B) then
      // touches distinct banks (c5's leaf pass: 2-way conflicts on the
      // register passes with low register positions, ncu profiles/r02c)
      const int bank_bits = c64 ? 4 : 3;
      std::vector<int> ns, order;
      for (int p = 0; p < t; ++p)
        if (std::find(pos, pos + 4, p) == pos + 4) ns.push_back(p);
      auto vec = [&](int p) -> unsigned { return (p < 16 ? 1u << (p & 3) : 0u) & ((1u << bank_bits) - 1); };
      std::vector<unsigned> basis;  // reduced row echelon by leading bit
      auto add_if_indep = [&](unsigned v) {
        for (unsigned bv : basis)
          if ((v ^ bv) < v) v ^= bv;
        if (!v) return false;
        basis.push_back(v);
        std::sort(basis.begin(), basis.end(), [](unsigned a, unsigned b) { return a > b; });
        return true;
      };
      std::vector<char> used(ns.size(), 0);
      for (size_t j = 0; j < ns.size() && (int)order.size() < bank_bits; ++j)
        if (add_if_indep(vec(ns[j]))) {
          order.push_back(ns[j]);
          used[j] = 1;
        }
      for (size_t j = 0; j < ns.size(); ++j)
        if (!used[j]) order.push_back(ns[j]);
      std::vector<int> from(order.size());
      for (size_t j = 0; j < order.size(); ++j) from[j] = (int)j;
      // gather_expr merges runs only when both sides advance by one, so pass
      // the pairs sorted by source bit (they already are)
      o << "    const u32 b = " << gather_expr("gi", from, order) << ";";
    } else {
      o << "    u32 b = gi;";
      for (int p : sorted) o << " b = ins0<" << p << ">(b);";
    }
    o << "\n    const u32 gb = G(" << (x ? "b" : "(RANK << LB) | b") << "); (void)gb;\n    C v[16];\n";
    // the swizzle is GF(2)-linear and b, e have disjoint bits: sw(b | e) =
    // sw(b) ^ sw(e), one XOR with a constant per access (c5 leaf pass: ~2 ALU
    // instructions fewer per shared-memory access)
    if (!x) o << "    const u32 sb = (u32)sw((int)b);\n";  // sw(b | e) = sw(b) + sw(e)
    auto elk = [&](uint32_t e) {
      if (x) return el(x, "(b | " + std::to_string(e) + "u)");
      const uint32_t swe = swz(e);
      return std::string("s[sb + ") + std::to_string(swe) + "u]";
    };
    const bool from_pb = pb_first && i == 0;
    auto elk_ld = [&](uint32_t e) {
      if (!from_pb) return elk(e);
      const uint32_t swe = swz(e);
      return std::string("pb_[sb + ") + std::to_string(swe) + "u]";
    };
    uint32_t ek[16];
    for (int k = 0; k < 16; ++k) {
      uint32_t e = 0;
      for (int j = 0; j < 4; ++j)
        if ((k >> j) & 1) e |= 1u << pos[j];
      ek[k] = e;
    }
    // direct access: register slot j0 on the tile position that G puts on
    // state bit 0 pairs slots k, k | 2^j0 into one 16 B (c64) access
    int j0 = -1;
    for (int j = 0; j < 4; ++j)
      if (fmap(1u << pos[j]) == 1u) j0 = j;
    auto direct = [&](bool load) {
      for (int k = 0; k < 16; ++k) {
        const std::string g = u(fmap(ek[k]));  // gb | g = gb + g (disjoint bits): an immediate offset
        if (j0 >= 0 && ((k >> j0) & 1)) continue;
        const int k1 = j0 >= 0 ? (k | (1 << j0)) : -1;
        if (load) {
          if (k1 >= 0)
            o << "      ld2(sp + " << g << ", v[" << k << "], v[" << k1 << "]);\n";
          else
            o << "      v[" << k << "] = sp[" << g << "];\n";
        } else {
          if (k1 >= 0)
            o << "    st2(dp + " << g << ", v[" << k << "], v[" << k1 << "]);\n";
          else
            o << "    dp[" << g << "] = v[" << k << "];\n";
        }
      }
    };
    if (dl) {
      o << "#ifndef HSF_NO_DIRECT\n";
      o << "    if (src) {\n      const C* sp = src + gb;\n";
      direct(true);
      o << "    } else {\n";
      for (int k = 0; k < 16; ++k)
        o << "      v[" << k << "] = czero<C>(); if ((gb | " << u(fmap(ek[k])) << ") == 0u) v[" << k << "].x = 1;\n";
      o << "    }\n#else\n";
    }
    for (int k = 0; k < 16; ++k) o << "    v[" << k << "] = " << elk_ld(ek[k]) << ";\n";
    if (dl) o << "#endif\n";
    auto emit_tdiag = [&](size_t r) {  // diagonal: index of element k = i0 | IK[k]
      const DevOp& d = ops[r];
      o << "    { const u32 i0 = " << didx(d, "gb") << ";\n";
      const bool st = staged(d) && tpad;
      if (st) o << "      const u32 p0 = i0 + (i0 >> 4);\n";  // padded(i0 | ik) = padded(i0) + padded(ik)
      for (int k = 0; k < 16; ++k) {
        uint32_t ik = 0;
        for (int j = 0; j < 4; ++j)
          if ((k >> j) & 1)
            for (int jj = 0; jj < d.k; ++jj)
              if (d.q[jj] == qreg[j]) ik |= 1u << jj;
        const std::string ld = st ? table((int)r) + "[p0 + " + std::to_string(ik + (ik >> 4)) + "u]"
                                  : tload(d, (int)r, "i0 | " + std::to_string(ik) + "u");
        o << "      v[" << k << "] = cmul(v[" << k << "], " << ld << ");\n";
      }
      o << "    }\n";
    };
    if (givens && coef) {
      givens_schedule(i, n, qreg, emit_tdiag);
    } else {
      for (size_t r = i + 1; r <= i + (size_t)n; ++r) {
        const DevOp& d = ops[r];
        if (d.kind == OP_R1) {
          if (literal(d))
            r1_literal(d.q[0], d);
          else
            o << "    r1<" << d.q[0] << ">(v, " << table((int)r) << ");\n";
        } else {
          emit_tdiag(r);
        }
      }
    }
    if (ds) {
      o << "#ifndef HSF_NO_DIRECT\n    C* dp = dst + gb;\n";
      direct(false);
      o << "#else\n";
    }
    for (int k = 0; k < 16; ++k) o << "    " << elk(ek[k]) << " = v[" << k << "];\n";
    if (ds) o << "#endif\n";
    o << "  }\n";
    if (ds) o << "#ifdef HSF_NO_DIRECT\n";
    sync_pre(x);
    if (ds) o << "#endif\n";
  }

  // run of standalone diagonal ops [i, j): element-owner mapping, 4 per thread
  void diag_run(size_t i, size_t j) {
    o << "  for (u32 e0 = " << TIDs << "; e0 < LNEL; e0 += 4u * NT) {\n";
    o << "#pragma unroll\n    for (u32 w = 0; w < 4u; ++w) { const u32 e = e0 + w * NT;";
    o << " if (e < LNEL) { const u32 g = G((RANK << LB) | e); C v = s[sw(e)];\n";
    for (size_t r = i; r < j; ++r)
      o << "      v = cmul(v, " << tload(ops[r], (int)r, didx(ops[r], "g")) << ");\n";
    o << "      s[sw(e)] = v; } }\n  }\n";
  }

  int nt = 256;  // threads per CTA (512 for narrow tree levels)
  int cb = 0;    // cluster tier: log2 CTAs per tile (0 = one CTA per tile)

  // store_mode: 0 leaf (node-major), 1 MN-major split-bf16 B operand,
  // 3 MN-major split-bf16 A operand of the swapped path-sum (st_aop)
  std::string build(const std::string& name, int threads, int cluster_bits, int store_mode = 0) {
    const bool operand_store = store_mode == 1 || store_mode == 3;
    nt = threads;
    cb = whole ? 0 : cluster_bits;
    bool heavy = false;
    for (auto& d : ops) heavy = heavy || d.kind == OP_RPASS || (d.kind == OP_DENSE && d.k > 2);
    // __launch_bounds__ min CTAs per SM (256 threads): 4 for heavy passes
    // (register passes, dense k > 2; <= 64 registers) -- measured against 2 / 3
    // / 5: q33-3 6.19 / 5.67 / 5.32 / 5.43 ms, q32-1 1.85 / 1.69 / 1.54 / 1.58,
    // c5 4.10 / 3.95 / 3.88 / 4.02 (latency-bound at 25 % occupancy with 86
    // registers); light passes insensitive 3 .. 5
    for (auto& d : ops) defer = defer && d.kind != OP_DENSE;  // a dense sweep would need the pending applied
    if (cb || !givens || !coef) defer = false;
    int heavy_minb = 4, light_minb = 3;
    if (const char* e = std::getenv("HSF_JIT_HEAVY_MINB")) heavy_minb = std::atoi(e);
    if (const char* e = std::getenv("HSF_JIT_LIGHT_MINB")) light_minb = std::atoi(e);
    {
      const char* e = std::getenv("HSF_JIT_DIRECT");
      const int dm = e ? std::atoi(e) : 3;  // bit 0: direct first register pass, bit 1: direct last
      const bool elig = !multi && !pb_first && cb == 0 && t > 4 && !ops.empty();
      direct_ld = elig && (dm & 1) && ops[0].kind == OP_RPASS;
      size_t r = 0, last = (size_t)-1;
      while (r < ops.size()) {
        if (ops[r].kind == OP_RPASS) {
          last = r;
          r += (size_t)ops[r].k + 1;
        } else {
          ++r;
        }
      }
      direct_st = elig && (dm & 2) && store_mode == 0 && last != (size_t)-1 && last + (size_t)ops[last].k + 1 == ops.size();
    }
    header(name, multi ? 2 : nt > 256 ? 1 : (heavy ? heavy_minb : light_minb));
    size_t i = 0;
    while (i < ops.size()) {
      const DevOp& d = ops[i];
      if (d.kind == OP_DENSE) {
        dense(d, (int)i);
        ++i;
      } else if (d.kind == OP_RPASS) {
        rpass(i);
        i += (size_t)d.k + 1;
      } else {
        size_t j = i;
        while (j < ops.size() && ops[j].kind == OP_DIAG) ++j;
        diag_run(i, j);
        o << "  " << SYNCs << ";\n";  // element-owner mapping differs from the store mapping
        i = j;
      }
    }
    // (direct last register pass: it stored the node state itself; the tile
    // store stays for the HSF_NO_DIRECT build)
    if (direct_st) o << "#ifdef HSF_NO_DIRECT\n";
    if (!multi) o << "  " << SYNCs << ";\n";  // (T-leaf: the CTA barrier before the store covers it)
    if (multi) {
      o << "  }\n  __syncthreads();\n";
      // transposed store of the item's `multi` leaves (group g's tile = leaf g):
      // row G(e) of the gather operand gets columns k0 .. k0 + multi - 1
      // (x c_p for half A), two columns (16 B) per thread, a row's multi / 2
      // threads adjacent
      const int hp = multi / 2;
      // (a thread's two columns are loop-invariant: their c_p loaded once)
      o << "  { C* T = reinterpret_cast<C*>(a.dst);\n";
      o << "    const C* t0 = reinterpret_cast<const C*>(smem_raw + c2 * " << group_bytes() << "u);\n";
      o << "    const C* t1 = reinterpret_cast<const C*>(smem_raw + (c2 + 1u) * " << group_bytes() << "u);\n";
      o << "    const bool hc = " << (cp_in_table() ? "false" : "cpt != nullptr") << ";\n";
      // unrolled: e = e0 + j * (rows per sweep), split off as in the load
      o << "    const u32 e0 = threadIdx.x / " << hp << "u, g0 = G(e0), s0 = (u32)sw((int)e0);\n";
      o << "#pragma unroll\n";
      o << "    for (u32 j = 0; j < LNEL * " << hp << "u / " << multi * 64 << "u; ++j) {\n";
      o << "      const u32 ej = j * " << multi * 64 / hp << "u, se = s0 + (u32)sw((int)ej);\n";
      o << "      C v0 = t0[se], v1 = t1[se];\n";
      o << "      if (hc) { v0 = cmul(v0, w0); v1 = cmul(v1, w1); }\n";
      o << "      st2(T + (long long)(g0 | G(ej)) * a.ldw + k0 + c2, v0, v1);\n";
      o << "    }\n  }\n";
      o << "  asm volatile(\"cp.async.wait_group 0;\" ::: \"memory\");\n";
      o << "  __syncthreads();\n  }\n";
    } else if (operand_store) {
      o << "#pragma unroll 4\n";
      o << "  for (u32 e = 2u * threadIdx.x; e < LNEL; e += 2u * NT) " << (store_mode == 3 ? "st_aop" : "st_bop")
        << "(a, a.node_local0 + NODE_ID, G((RANK << LB) | e), s[sw(e)], s[sw(e + 1)]);\n";
    } else if (!cb && (1 << t) >= 2 * nt) {  // unrolled, thread element split off (see the load)
      o << "  { const u32 e0 = 2u * threadIdx.x, g0 = G(e0), s0 = (u32)sw((int)e0);\n";
      o << "#pragma unroll\n";
      o << "    for (u32 j = 0; j < LNEL / (2u * NT); ++j) { const u32 ej = j * 2u * NT, sj = s0 + (u32)sw((int)ej); "
           "st2(dst + (g0 | G(ej)), s[sj], s[sj + 1u]); } }\n";
    } else {
      o << "#pragma unroll 4\n";
      o << "  for (u32 e = 2u * threadIdx.x; e < LNEL; e += 2u * NT) st2(dst + G((RANK << LB) | e), s[sw(e)], s[sw(e + 1)]);\n";
    }
    if (direct_st) o << "#endif\n";
    o << "}\n";
    // back-to-back barriers (one pass's end, the next one's start) -> one
    std::string src = o.str();
    const std::string two = "  __syncthreads();\n  __syncthreads();\n", one = "  __syncthreads();\n";
    for (size_t p = src.find(two); p != std::string::npos; p = src.find(two, p)) src.replace(p, two.size(), one);
    return src;
  }
};

// ------------------------------------------------------------ driver API
struct Drv {
  CUresult (*moduleLoadData)(CUmodule*, const void*) = nullptr;
  CUresult (*moduleGetFunction)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*funcSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
  CUresult (*launchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                           CUstream, void**, void**) = nullptr;
  CUresult (*launchKernelEx)(const CUlaunchConfig*, CUfunction, void**, void**) = nullptr;
};

template <typename F>
void load_sym(F& f, const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess || !p)
    fail(HSF_ERR_CUDA, std::string("driver entry point ") + name + " unavailable");
  f = reinterpret_cast<F>(p);
}

Drv& drv() {
  static Drv d;
  static std::once_flag once;
  std::call_once(once, [] {
    load_sym(d.moduleLoadData, "cuModuleLoadData");
    load_sym(d.moduleGetFunction, "cuModuleGetFunction");
    load_sym(d.funcSetAttribute, "cuFuncSetAttribute");
    load_sym(d.launchKernel, "cuLaunchKernel");
    load_sym(d.launchKernelEx, "cuLaunchKernelEx");
  });
  return d;
}

uint64_t fnv64(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

std::mutex g_mu;
std::map<std::pair<int, std::string>, void*> g_cache;  // (device, source) -> CUfunction

// ptxas reported local-memory spills (the -v log's "N bytes spill stores")
static bool log_spills(const std::string& log) {
  const std::string key = " bytes spill stores";
  for (size_t p = log.find(key); p != std::string::npos; p = log.find(key, p + 1)) {
    size_t b = p;
    while (b > 0 && std::isdigit((unsigned char)log[b - 1])) --b;
    if (b < p && std::atoi(log.c_str() + b) > 0) return true;
  }
  return false;
}

// A pass with direct register passes whose build spills at the register cap
// (ptxas -v) is rebuilt with HSF_NO_DIRECT: tile load / store through shared
// memory, as before (c3's narrow root passes at 64 registers)
std::vector<char> nvrtc_compile(const std::string& src, std::string& log, bool no_direct = false);
std::vector<char> nvrtc_compile(const std::string& src, std::string& log, bool no_direct) {
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "hsf_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    log = "nvrtcCreateProgram failed";
    return {};
  }
  const bool direct = !no_direct && src.find("HSF_NO_DIRECT") != std::string::npos;
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo", "--fmad=true",
                        no_direct ? "-DHSF_NO_DIRECT" : "--ptxas-options=-v"};
  nvrtcResult r = nvrtcCompileProgram(prog, (no_direct || direct) ? 5 : 4, opts);
  size_t n = 0;
  nvrtcGetProgramLogSize(prog, &n);
  log.assign(n, '\0');
  if (n) nvrtcGetProgramLog(prog, &log[0]);
  std::vector<char> cubin;
  if (r == NVRTC_SUCCESS) {
    size_t cb = 0;
    nvrtcGetCUBINSize(prog, &cb);
    cubin.resize(cb);
    nvrtcGetCUBIN(prog, cubin.data());
  }
  nvrtcDestroyProgram(&prog);
  if (direct && r == NVRTC_SUCCESS && log_spills(log)) return nvrtc_compile(src, log, true);
  return cubin;
}

}  // namespace

static void defer_result(const Gen& g, DeferOut* d) {
  if (!d) return;
  d->active = g.defer;
  d->phase.clear();
  d->scalar = 1.0;
  if (!g.defer) return;
  for (auto& kv : g.carry) d->phase.push_back({kv.first, kv.second});
  d->scalar = g.carry_scalar;
}

// cache-operator experiment knob (jit_prelude.cuh): part of the source, so of the cache key
static std::string ldst_defs() {
  const char* e = std::getenv("HSF_JIT_LDST");
  if (!e) return "";
  const int v = std::atoi(e);
  return "#define HSF_LD_MODE " + std::to_string(v / 10) + "\n#define HSF_ST_MODE " + std::to_string(v % 10) + "\n";
}

std::string jit_pass_source(const Half& H, const Pass& ps, bool c64, int threads, int cluster_bits,
                            const std::vector<cd>* coef, int store_mode, DeferOut* defer) {
  Gen g(H, ps, c64, coef);
  g.defer = defer != nullptr && store_mode == 0;
  std::string src = ldst_defs() + std::string(kPrelude) + "\n" + g.build("hsf_jit_pass", threads, cluster_bits, store_mode);
  defer_result(g, defer);
  return src;
}

std::string jit_tleaf_source(const Half& TL, int leaves, bool c64, const std::vector<cd>* coef, DeferOut* defer) {
  const Pass& ps = TL.trans[0].passes[0];
  Gen g(TL, ps, c64, coef);
  g.defer = defer != nullptr;
  g.multi = leaves;
  g.pb_first = !g.ops.empty() && g.ops[0].kind == OP_RPASS && !std::getenv("HSF_TLEAF_COPY");
  g.TIDs = "TID";
  g.SYNCs = "asm volatile(\"bar.sync %0, 64;\" :: \"r\"(1u + GRP) : \"memory\")";
  std::string src = ldst_defs() + std::string(kPrelude) + "\n" + g.build("hsf_jit_pass", 64 * leaves, 0, 0);
  defer_result(g, defer);
  return src;
}

size_t jit_tleaf_smem_bytes(const Half& TL, int leaves, bool c64) {
  const Pass& ps = TL.trans[0].passes[0];
  const size_t elem = c64 ? 8 : 16;
  // the groups' tiles + tables, then the double-buffered parent tile
  return (size_t)leaves * tleaf_group_bytes(ps.t, ps.tbl_elems, elem) + 2 * elem * padded(ps.t);
}

size_t jit_smem_bytes(const Pass& ps, bool c64, int cluster_bits) {
  const size_t elem = c64 ? 8 : 16;
  return elem * padded(ps.t - cluster_bits) + (size_t)ps.tbl_elems * elem;
}

std::vector<void*> jit_compile_all(int device, const std::vector<std::string>& sources) {
  std::vector<void*> fns(sources.size(), nullptr);
  std::vector<size_t> todo;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (size_t i = 0; i < sources.size(); ++i) {
      auto it = g_cache.find({device, sources[i]});
      if (it != g_cache.end())
        fns[i] = it->second;
      else if (std::find_if(todo.begin(), todo.end(), [&](size_t j) { return sources[j] == sources[i]; }) == todo.end())
        todo.push_back(i);
    }
  }
  if (!todo.empty()) {
    std::vector<std::vector<char>> bins(todo.size());
    std::vector<std::string> logs(todo.size());
    std::atomic<size_t> next{0};
    const unsigned nth = std::max(1u, std::min<unsigned>((unsigned)todo.size(), std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (unsigned w = 0; w < nth; ++w)
      th.emplace_back([&] {
        for (size_t k; (k = next++) < todo.size();) bins[k] = nvrtc_compile(sources[todo[k]], logs[k]);
      });
    for (auto& x : th) x.join();
    Drv& D = drv();
    std::lock_guard<std::mutex> lk(g_mu);
    for (size_t k = 0; k < todo.size(); ++k) {
      if (bins[k].empty())
        fail(HSF_ERR_UNSUPPORTED, "NVRTC compile of a specialised pass failed: " + logs[k].substr(0, 2000));
      CUmodule mod;
      CUfunction f;
      if (D.moduleLoadData(&mod, bins[k].data()) != CUDA_SUCCESS) fail(HSF_ERR_CUDA, "cuModuleLoadData failed");
      if (D.moduleGetFunction(&f, mod, "hsf_jit_pass") != CUDA_SUCCESS) fail(HSF_ERR_CUDA, "cuModuleGetFunction failed");
      if (D.funcSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, 227 * 1024) != CUDA_SUCCESS)
        fail(HSF_ERR_CUDA, "cuFuncSetAttribute failed");
      // HSF_JIT_CARVEOUT=p: preferred shared-memory carveout in percent (the
      // passes stream their global loads, so L1 has nothing to keep); unset =
      // the driver's choice from the launch's dynamic size
      if (const char* e = std::getenv("HSF_JIT_CARVEOUT"))
        D.funcSetAttribute(f, CU_FUNC_ATTRIBUTE_PREFERRED_SHARED_MEMORY_CARVEOUT, std::atoi(e));
      g_cache[{device, sources[todo[k]]}] = (void*)f;  // modules live for the process
    }
    for (size_t i = 0; i < sources.size(); ++i)
      if (!fns[i]) fns[i] = g_cache[{device, sources[i]}];
  }
  return fns;
}

void jit_launch(void* fn, unsigned gx, unsigned gy, unsigned threads, size_t smem, void* stream,
                const JitLaunchArgs& a, int cluster_bits) {
  JitLaunchArgs args = a;
  void* params[] = {&args};
  if (cluster_bits > 0) {  // cluster tier: 2^cb CTAs per tile, one (2^cb, 1, 1) cluster each
    CUlaunchAttribute attr[1];
    std::memset(attr, 0, sizeof(attr));
    attr[0].id = CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION;
    attr[0].value.clusterDim.x = 1u << cluster_bits;
    attr[0].value.clusterDim.y = 1;
    attr[0].value.clusterDim.z = 1;
    CUlaunchConfig cfg;
    std::memset(&cfg, 0, sizeof(cfg));
    cfg.gridDimX = gx << cluster_bits;
    cfg.gridDimY = gy;
    cfg.gridDimZ = 1;
    cfg.blockDimX = threads;
    cfg.blockDimY = 1;
    cfg.blockDimZ = 1;
    cfg.sharedMemBytes = (unsigned)smem;
    cfg.hStream = (CUstream)stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (drv().launchKernelEx(&cfg, (CUfunction)fn, params, nullptr) != CUDA_SUCCESS)
      fail(HSF_ERR_CUDA, "cuLaunchKernelEx (cluster-tier pass) failed");
    return;
  }
  if (drv().launchKernel((CUfunction)fn, gx, gy, 1, threads, 1, 1, (unsigned)smem, (CUstream)stream, params, nullptr) !=
      CUDA_SUCCESS)
    fail(HSF_ERR_CUDA, "cuLaunchKernel (specialised pass) failed");
}

uint64_t jit_source_hash(const std::string& s) { return fnv64(s); }

}  // namespace hsf
