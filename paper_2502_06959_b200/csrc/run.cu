// run.cu — C ABI of libhsf.so (include/hsf.h): plan lifetime, device tables,
// workspace, and hsf_run's launch sequence
//   half A tree -> half B tree -> coefficient fold -> path-sum.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>

#include "hsf_internal.h"
#include "sim_kernels.cuh"
#include "sum_kernels.cuh"
#include "gemm_tc.cuh"
#include "jit.h"
#include "comm.h"

namespace hsf {

static thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }

#define CK(x)                                                                                          \
  do {                                                                                                 \
    cudaError_t e_ = (x);                                                                              \
    if (e_ != cudaSuccess)                                                                             \
      fail(HSF_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_) + " @" + std::to_string(__LINE__)); \
  } while (0)

struct DeviceState {
  int device = -1;
  size_t elem = 8;          // bytes per complex
  void* coef = nullptr;     // complex table (run dtype)
  DevOp* ops[2] = {nullptr, nullptr};
  DevOp* ops_fold[2] = {nullptr, nullptr};  // trailing-diagonal fold variant
  DevOp* ops_tail[2] = {nullptr, nullptr};  // half-sided trailing fold variant (full output)
  void* trail = nullptr;                    // folded units' block diagonals (run dtype)
  // deferred final diagonals of the bitstring-fold variant's last kernel per
  // half ([0] its last tile pass, [1] its T-leaf pass): extra per-sample
  // weight tables appended to `trail` (mask of global bits, table offset)
  DeferOut dfin[2][2];
  std::vector<std::pair<unsigned long long, long long>> dfin_units[2][2];
  void* tail = nullptr;                     // half-sided folded diagonal factors (run dtype)
  float2* tailw[2] = {nullptr, nullptr};    // [T][2^m] tail weights per half (tensor-core runs)
  // half B's last pass (full tree) writing the MN-major split-bf16 GEMM
  // operand directly (full-output tensor-core runs; K4 fused into the leaf pass)
  void* jit_bop = nullptr;
  int jit_bop_nt = 256;
  void* jit_aop = nullptr;  // the same pass writing the swapped path-sum's M operand
  // T-leaf variants (Half::tleaf) of each half's last transition: [variant 0 full / 1 fold][half]
  void* jit_tl[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};

  bool jit = false;                         // specialised pass kernels loaded
  unsigned long long* perm_tab = nullptr;   // caller -> internal index bits (partitions)
  // [variant: 0 full tree, 1 bitstring fold, 2 half-sided tail][half] per flattened pass
  std::vector<void*> jit_fn[3][2];
  std::vector<int> jit_nt[3][2];            //   and its threads per CTA
  std::vector<int> jit_cb[3][2];            //   and its cluster bits (cluster tier, narrow levels)
  void* ws = nullptr;
  size_t ws_bytes = 0;
  // cached per-range path coefficients
  void* cp = nullptr;
  size_t cp_cap = 0;
  uint64_t cp_p0 = ~0ull, cp_p1 = ~0ull;
  int cp_units = -1;
  int cp_heads = 0;
  cudaEvent_t ev[6] = {};
  cudaEvent_t ev_t0 = nullptr;              // timing start (ev[0] is the fork event)
  // CUDA graph of the whole run (both streams), replayed while the run's
  // arguments (pointers, ranges, precision) stay the same
  cudaStream_t cap = nullptr;
  cudaGraphExec_t gexec = nullptr;
  std::vector<uint64_t> gkey;
  int gkernels = -1;                        // kernel nodes of the captured graph
  std::vector<uint64_t> comm_ok;            // communicators whose ranks' plan hashes were compared
  bool capturing = false;
  cudaEvent_t evg[2] = {}, evc[2] = {};  // host-output chunks: GEMM done / D2H done
  cudaStream_t side = nullptr;  // half-B stream; D2H stream of host-output chunks
  cudaStream_t aux = nullptr;   // bitstring prep (H2D, relabel, bucket sort), overlapping the trees
  cudaEvent_t ev_aux = nullptr;
  bool sticky = false;
  unsigned int* bad_bits = nullptr;      // mapped host word: a sample had bits >= 2^n
  unsigned int* bad_bits_dev = nullptr;  //   its device alias
};

void destroy_device(Plan* p) {
  auto* d = (DeviceState*)p->dev;
  if (!d) return;
  int cur = -1;
  cudaGetDevice(&cur);
  if (d->device >= 0) cudaSetDevice(d->device);
  cudaFree(d->coef);
  cudaFree(d->ops[0]);
  cudaFree(d->ops[1]);
  cudaFree(d->ops_fold[0]);
  cudaFree(d->ops_fold[1]);
  cudaFree(d->ops_tail[0]);
  cudaFree(d->ops_tail[1]);
  cudaFree(d->trail);
  cudaFree(d->tail);
  cudaFree(d->tailw[0]);
  cudaFree(d->tailw[1]);
  cudaFree(d->perm_tab);
  cudaFree(d->ws);
  cudaFree(d->cp);
  for (auto& e : d->ev)
    if (e) cudaEventDestroy(e);
  if (d->ev_t0) cudaEventDestroy(d->ev_t0);
  if (d->gexec) cudaGraphExecDestroy(d->gexec);
  if (d->cap) cudaStreamDestroy(d->cap);
  for (int i = 0; i < 2; ++i) {
    if (d->evg[i]) cudaEventDestroy(d->evg[i]);
    if (d->evc[i]) cudaEventDestroy(d->evc[i]);
  }
  if (d->side) cudaStreamDestroy(d->side);
  if (d->aux) cudaStreamDestroy(d->aux);
  if (d->bad_bits) cudaFreeHost(d->bad_bits);
  if (d->ev_aux) cudaEventDestroy(d->ev_aux);
  if (cur >= 0) cudaSetDevice(cur);
  delete d;
  p->dev = nullptr;
}

// half h's fold variant as seen by the operand-prep kernels (path-range
// fields p0 / node0 / W filled by the caller)
static tc::TailParams tail_params(const Plan& P, int h) {
  const Plan::Tail& T = P.tail[h];
  tc::TailParams tp{};
  tp.mapped = 1;
  tp.n = (int)T.mask.size();
  tp.T = (long long)T.T;
  tp.Tt = (long long)T.Tt;
  long long stride = 1;
  for (int u = tp.n - 1; u >= 0; --u) {
    tp.mask[u] = T.mask[u];
    tp.radix[u] = T.radix[u];
    tp.off[u] = T.off[u];
    tp.stride[u] = stride;
    stride *= T.radix[u];
  }
  return tp;
}

static DeviceState* ensure_device(Plan* P, int device) {
  auto* d = (DeviceState*)P->dev;
  if (d && d->sticky) fail(HSF_ERR_CUDA, "plan is unusable after an earlier CUDA error");
  if (device < 0) CK(cudaGetDevice(&device));
  if (d && d->device != device) fail(HSF_ERR_INVALID_ARG, "plan already bound to another device");
  CK(cudaSetDevice(device));
  if (d) return d;
  d = new DeviceState();
  P->dev = d;
  d->device = device;
  const bool c64 = P->opts.dtype == HSF_C64;
  d->elem = c64 ? 8 : 16;
  // coefficient table in the run dtype (fp64 master -> fp32 by RNE)
  size_t n = std::max<size_t>(P->coef.size(), 1);
  CK(cudaMalloc(&d->coef, n * d->elem));
  if (c64) {
    std::vector<float2> h(n);
    for (size_t i = 0; i < P->coef.size(); ++i) h[i] = make_float2((float)P->coef[i].real(), (float)P->coef[i].imag());
    CK(cudaMemcpy(d->coef, h.data(), n * 8, cudaMemcpyHostToDevice));
  } else {
    CK(cudaMemcpy(d->coef, P->coef.data(), P->coef.size() * 16, cudaMemcpyHostToDevice));
  }
  auto upload_ops = [&](const Half& H, DevOp** dst) {
    size_t no = std::max<size_t>(H.dev_ops.size(), 1);
    CK(cudaMalloc(dst, no * sizeof(DevOp)));
    if (!H.dev_ops.empty())
      CK(cudaMemcpy(*dst, H.dev_ops.data(), H.dev_ops.size() * sizeof(DevOp), cudaMemcpyHostToDevice));
  };
  for (int h = 0; h < 2; ++h) {
    upload_ops(P->half[h], &d->ops[h]);
    if (P->fold_u0 >= 0) upload_ops(P->half_fold[h], &d->ops_fold[h]);
    if (P->tail[h].u0 >= 0) upload_ops(P->tail[h].half, &d->ops_tail[h]);
  }
  auto upload_tab = [&](const std::vector<cd>& tab, void** dst) {
    const size_t nt = tab.size();
    CK(cudaMalloc(dst, std::max<size_t>(nt, 1) * d->elem));
    if (c64) {
      std::vector<float2> h(nt);
      for (size_t i = 0; i < nt; ++i) h[i] = make_float2((float)tab[i].real(), (float)tab[i].imag());
      CK(cudaMemcpy(*dst, h.data(), nt * 8, cudaMemcpyHostToDevice));
    } else {
      CK(cudaMemcpy(*dst, tab.data(), nt * 16, cudaMemcpyHostToDevice));
    }
  };
  if (P->fold_u0 >= 0) upload_tab(P->trail_tab, &d->trail);
  if (!P->tail_tab.empty()) upload_tab(P->tail_tab, &d->tail);
  if (P->permuted) {
    std::vector<unsigned long long> tab(4 * 65536, 0);
    for (int k = 0; k < 4; ++k)
      for (unsigned v = 0; v < 65536; ++v) {
        unsigned long long x = 0;
        for (int b = 0; b < 16; ++b) {
          const int q = 16 * k + b;
          if (q < P->n && ((v >> b) & 1u)) x |= 1ull << P->relabel[q];
        }
        tab[(size_t)k * 65536 + v] = x;
      }
    CK(cudaMalloc(&d->perm_tab, tab.size() * 8));
    CK(cudaMemcpy(d->perm_tab, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice));
  }
  if (P->opts.jit) {
    // one specialised kernel per tile pass (jit.cpp), compiled once per process
    std::vector<std::string> src;
    std::vector<std::pair<int, int>> owner;
    for (int v = 0; v < 3; ++v) {
      if (v == 1 && P->fold_u0 < 0) continue;
      for (int h = 0; h < 2; ++h) {
        if (v == 2 && P->tail[h].u0 < 0) continue;
        const Half& H = v == 0 ? P->half[h] : v == 1 ? P->half_fold[h] : P->tail[h].half;
        for (const auto& tr : H.trans) {
          // narrow levels (few nodes x tiles, e.g. a root that hoisting made
          // heavy) get 512-thread CTAs: twice the threads on the few SMs busy
          const double ctas = (double)range_prod(P->ranks, 0, tr.level_out);
          for (const auto& ps : tr.passes) {
            const double n_cta = ctas * std::ldexp(1.0, H.m - ps.t);
            // Cluster tier (opt-in, HSF_CLUSTER=1): very narrow tiled levels split
            // each tile over a cluster of 2 or 4 CTAs (DSMEM for the ops on the
            // top tile positions).  Parity-tested, but measured no faster on c3's
            // narrow roots (their passes are bound by each thread's op chain, not
            // by one SM's issue rate), so the default is 512-thread CTAs there.
            const char* ce = std::getenv("HSF_CLUSTER");
            const bool tiled = ps.t < H.m && ps.t >= 12 && ce && ce[0] == '1';
            int cb = 0;
            if (tiled && n_cta * 4 <= num_sms()) cb = 2;
            else if (tiled && n_cta * 2 <= num_sms()) cb = 1;
            int nt = cb ? std::max(128, 1 << (ps.t - cb - 4)) : (n_cta < 2.0 * num_sms() ? 512 : 256);
            if (!cb) nt = std::min(nt, std::max(128, 1 << (ps.t - 2)));  // small narrow-level tiles (t = 10, 11)
            // the fold variant's last pass leaves its final diagonals to the gather
            const bool lastp = v == 1 && &tr == &H.trans.back() && &ps == &tr.passes.back();
            src.push_back(jit_pass_source(H, ps, c64, nt, cb, &P->coef, 0, lastp ? &d->dfin[0][h] : nullptr));
            owner.push_back({v, h});
            d->jit_nt[v][h].push_back(nt);
            d->jit_cb[v][h].push_back(cb);
          }
        }
      }
    }
    // operand-store variant of half B's last pass (same launch shape)
    const Half& HB = P->half[1];
    const bool bop = c64 && !d->jit_cb[0][1].empty() && d->jit_cb[0][1].back() == 0;
    if (bop) {
      d->jit_bop_nt = d->jit_nt[0][1].back();
      src.push_back(jit_pass_source(HB, HB.trans.back().passes.back(), c64, d->jit_bop_nt, 0, &P->coef, 1));
      owner.push_back({-1, 1});
      if (P->n_low >= 8) {
        src.push_back(jit_pass_source(HB, HB.trans.back().passes.back(), c64, d->jit_bop_nt, 0, &P->coef, 3));
        owner.push_back({-1, 3});
      }
    }
    // T-leaf variants (bitstring runs: the half the block gather reads transposed)
    for (int v = 0; v < 2 && c64; ++v) {
      if (v == 1 && P->fold_u0 < 0) continue;
      for (int h = 0; h < 2; ++h) {
        const Half& H = v ? P->half_fold[h] : P->half[h];
        if (!H.tleaf) continue;
        // (no deferral here: the T side's D_fin would be per-sample table
        // lookups in the gather, and this pass is write-bound, not issue-bound)
        src.push_back(jit_tleaf_source(*H.tleaf, H.tleaf_R, c64, &P->coef));
        owner.push_back({-2 - (2 * v + h), 0});
      }
    }
    std::vector<void*> fns = jit_compile_all(device, src);
    for (size_t i = 0; i < fns.size(); ++i) {
      if (owner[i].first == -1)
        (owner[i].second == 3 ? d->jit_aop : d->jit_bop) = fns[i];
      else if (owner[i].first <= -2)
        d->jit_tl[(-2 - owner[i].first) / 2][(-2 - owner[i].first) % 2] = fns[i];
      else
        d->jit_fn[owner[i].first][owner[i].second].push_back(fns[i]);
    }
    d->jit = true;
    // D_fin tables over contiguous ranges of <= 10 of the half's qubits
    // (index = one shift and mask in the gather), entry = product of the
    // pending phases of the range's set bits (the scalar in the first range
    // used), appended after the folded units' tables
    std::vector<cd> tab = P->trail_tab;
    bool any = false;
    for (int kind = 0; kind < 2; ++kind)
      for (int h = 0; h < 2; ++h) {
        const DeferOut& df = d->dfin[kind][h];
        if (!df.active || (df.phase.empty() && df.scalar == cd(1.0))) continue;
        any = true;
        const int first = P->half[h].first_qubit, mq = P->half[h].m;
        std::vector<cd> ph(mq, cd(1.0));
        for (const auto& q : df.phase) ph[q.first] = q.second;
        bool scalar_done = false;
        for (int lo = 0; lo < mq; lo += 10) {
          const int hi = std::min(mq, lo + 10);
          bool used = !scalar_done && df.scalar != cd(1.0);
          for (int q = lo; q < hi; ++q) used = used || ph[q] != cd(1.0);
          if (!used) continue;
          const unsigned long long mask = ((1ull << (hi - lo)) - 1ull) << (first + lo);
          d->dfin_units[kind][h].push_back({mask, (long long)tab.size()});
          for (size_t idx = 0; idx < (1ull << (hi - lo)); ++idx) {
            cd w = scalar_done ? cd(1.0) : df.scalar;
            for (int j = 0; j < hi - lo; ++j)
              if ((idx >> j) & 1) w *= ph[lo + j];
            tab.push_back(w);
          }
          scalar_done = true;
        }
      }
    if (any) {
      cudaFree(d->trail);
      d->trail = nullptr;
      upload_tab(tab, &d->trail);
    }
  }
  for (auto& e : d->ev) CK(cudaEventCreateWithFlags(&e, cudaEventDefault));
  CK(cudaEventCreateWithFlags(&d->ev_t0, cudaEventDefault));
  CK(cudaStreamCreateWithFlags(&d->cap, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    CK(cudaEventCreateWithFlags(&d->evg[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&d->evc[i], cudaEventDisableTiming));
  }
  CK(cudaStreamCreateWithFlags(&d->side, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&d->aux, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&d->ev_aux, cudaEventDisableTiming));
  CK(cudaHostAlloc((void**)&d->bad_bits, sizeof(unsigned int), cudaHostAllocMapped));
  *d->bad_bits = 0;
  CK(cudaHostGetDevicePointer((void**)&d->bad_bits_dev, d->bad_bits, 0));
  return d;
}

// ----------------------------------------------------------- workspace
struct Layout {
  uint64_t p0, p1, K;          // path range of the path-sum (folded runs: full range / fold_T)
  bool fold = false;           // trailing-diagonal fold active (bitstring runs)
  int U_tree = 0;              // units behind p0, p1 (c_p table)
  std::vector<int32_t> ranks;  // their radices
  // per half: evaluated tree (0 full, 1 bitstring fold, 2 half-sided tail),
  // its units' radices and its node range at the leaf level
  int var[2] = {0, 0};
  std::vector<int32_t> hranks[2];
  uint64_t hp0[2] = {0, 0}, hp1[2] = {0, 0};
  const Half* half[2] = {nullptr, nullptr};
  bool bop = false;            // half B's last pass writes the MN-major GEMM operand (with a JIT kernel)
  bool swap = false;           // few output rows: GEMM with the roles swapped (half B's 2^nB rows as M,
                               // half A's rows as N with the complex rotation), then a transpose
  size_t off_swapT = 0;        // its [2^nB][swap_cols] complex64 output
  bool aop = false;            // swapped: M operand stored by half B's last pass (jit_aop)
  bool bits_mode;
  uint64_t r0, r1;
  hsf_precision prec;
  size_t scratch_elems[2] = {0, 0};  // per ping-pong buffer, per half
  size_t off_scratch[2][2] = {{0, 0}, {0, 0}};  // [half][ping/pong]: the halves run concurrently
  size_t off_leaves[2] = {0, 0};
  size_t off_T[2] = {0, 0};    // transposed operands (bitstring mode)
  size_t off_bits = 0, off_out = 0, off_tc = 0;
  size_t off_pbits = 0, off_pout = 0;  // relabelled bitstrings / internal-order output (partitions)
  int direct = -1;             // block gather (gather_block_c64_kernel): half read from its leaves, -1 => none
  long long Kp = 0;            // its transposed other half's padded row length
  long long n_blocks = 0;      // blocks of block_rows rows of the direct half
  int block_rows = 16;
  bool tleaf[2] = {false, false};  // that half's last transition = its T-leaf pass (no leaves, no transpose)
  size_t off_grp = 0;          // counts[n_blocks] | offs[n_blocks + 1] | cursor[n_blocks] | sidx[n] (int32)
  size_t off_sbits = 0;        // sbits[n] (uint64): the samples' bitstrings in block order
  size_t tc_bytes = 0;
  uint64_t chunk_rows = 0;     // full mode, host output: rows per staged D2H chunk
  size_t chunk_bytes = 0;
  size_t total = 0;
};

// block gather launch shape (tuning: HSF_GATHER_CFG = 100 * (RB == 32 ? 3 : 1)
// + 10 * min CTAs per SM + U samples in flight per warp)
static int gather_cfg() {
  if (const char* e = std::getenv("HSF_GATHER_CFG")) return std::atoi(e);
  return 344;
}
static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }
// split-bf16 operand planes per precision mode
// (4 = tf32x3: hi + lo planes of fp32-storage tf32 values)
static int tc_planes(hsf_precision p) {
  return p == HSF_PREC_TF32X3 ? 4 : p == HSF_PREC_BF16X6 ? 3 : p == HSF_PREC_BF16X3 ? 2 : 1;
}
constexpr size_t kHostChunkBytes = (size_t)16 << 20;  // D2H of chunk i overlaps the path-sum of chunk i+1 (c2 e2e: 32 MB 2.74, 16 MB 2.64, 8 MB 2.65 ms)

static uint64_t nodes_at(const std::vector<int32_t>& ranks, int L, uint64_t p0, uint64_t p1) {
  uint64_t S = suffix_prod(ranks, L);
  return (p1 - 1) / S - p0 / S + 1;
}

// swapped path-sum: GEMM columns = the run's output rows, padded to even (16 B
// rows of the fp32 [2^nB][2 * cols] GEMM output)
static long long swap_cols(const Layout& L) { return (long long)((L.r1 - L.r0 + 1) & ~1ull); }

static Layout make_layout(const Plan& P, const hsf_run_args& a, size_t elem) {
  Layout L{};
  L.p0 = a.path_begin;
  L.p1 = a.path_end;
  if (L.p0 == 0 && L.p1 == 0) L.p1 = P.n_paths;
  if (L.p0 >= L.p1 || L.p1 > P.n_paths) fail(HSF_ERR_INVALID_ARG, "bad path range");
  L.bits_mode = a.n_bitstrings > 0;
  // the folded tree evaluates path groups of fold_T consecutive paths (the
  // folded units are the fastest digits), so the range must be aligned
  L.fold = L.bits_mode && P.fold_u0 >= 0 && L.p0 % P.fold_T == 0 && L.p1 % P.fold_T == 0;
  L.U_tree = L.fold ? P.fold_u0 : (int)P.units.size();
  L.ranks.assign(P.ranks.begin(), P.ranks.begin() + L.U_tree);
  for (int h = 0; h < 2; ++h) L.half[h] = L.fold ? &P.half_fold[h] : &P.half[h];
  if (L.fold) {
    L.p0 /= P.fold_T;
    L.p1 /= P.fold_T;
  }
  L.K = L.p1 - L.p0;
  L.prec = a.precision;
  if ((int)L.prec < (int)HSF_PREC_AUTO || (int)L.prec > (int)HSF_PREC_TF32X3)
    fail(HSF_ERR_INVALID_ARG, "unknown precision mode " + std::to_string((int)L.prec));
  if (L.prec == HSF_PREC_AUTO) L.prec = (P.opts.dtype == HSF_C64) ? HSF_PREC_BF16X3 : HSF_PREC_SIMT;
  if (P.opts.dtype == HSF_C128 && L.prec != HSF_PREC_SIMT) fail(HSF_ERR_UNSUPPORTED, "complex128 path-sum is SIMT fp64 only");
  // half-sided trailing fold: full-output tensor-core runs whose path range
  // holds whole groups of T consecutive paths (the folded units are the
  // fastest digits)
  for (int h = 0; h < 2; ++h) {
    // (head fold: whole periods of T * Tt paths, the tree is evaluated whole)
    const Plan::Tail& T = P.tail[h];
    const uint64_t per = T.v0 > 0 ? T.T * T.Tt : T.T;
    const bool tail = !L.bits_mode && L.prec != HSF_PREC_SIMT && T.u0 >= 0 && L.p0 % per == 0 && L.p1 % per == 0;
    L.var[h] = L.fold ? 1 : tail ? 2 : 0;
    if (tail) {
      L.half[h] = &T.half;
      L.hranks[h].assign(P.ranks.begin(), P.ranks.begin() + T.u0);
      for (int u = 0; u < T.v0; ++u) L.hranks[h][u] = 1;
      L.hp0[h] = T.v0 > 0 ? 0 : L.p0 / T.T;
      L.hp1[h] = T.v0 > 0 ? T.Tt : L.p1 / T.T;
    } else {
      L.hranks[h] = L.ranks;
      L.hp0[h] = L.p0;
      L.hp1[h] = L.p1;
    }
  }
  {
    // swapped path-sum for prefix outputs (<= 128 rows of A): half B's leaves
    // become the un-rotated (re, im planes) MN-major M operand, stored by B's
    // last pass, and the few A rows the rotated K-major N operand of one
    // narrow pair tile (tc_swap_buffers).  The big operand is half the bytes
    // of the rotated one and streams once instead of 16x-padded M tiles
    // re-reading it (q33-3 9.40 -> 7.09 ms); HSF_TC_SWAP=0 / 1 forces off / on
    const uint64_t nr = (a.row_end > a.row_begin ? a.row_end - a.row_begin : 1ull << (P.n - P.n_low));
    const char* sw = std::getenv("HSF_TC_SWAP");
    const bool want = sw ? sw[0] == '1' : true;
    L.swap = want && nr <= 128 && !L.bits_mode && P.opts.dtype == HSF_C64 && L.prec != HSF_PREC_SIMT &&
             L.prec != HSF_PREC_TF32X3 && a.n_out_shards == 0 && !P.permuted && tc_mn((long long)L.K) &&
             P.n_low >= 8;
  }
  L.bop = !L.bits_mode && !L.swap && (L.prec == HSF_PREC_BF16X3 || L.prec == HSF_PREC_BF16X1) &&
          P.opts.dtype == HSF_C64 && L.var[1] == 0 && tc_mn((long long)L.K);
  // the swapped path-sum's M operand written by half B's last pass (HSF_TC_AOP=0 disables)
  const char* aop_env = std::getenv("HSF_TC_AOP");
  L.aop = L.swap && (L.prec == HSF_PREC_BF16X3 || L.prec == HSF_PREC_BF16X1) && L.var[1] == 0 &&
          !(aop_env && aop_env[0] == '0');
  if (!L.bits_mode && a.bitstrings) fail(HSF_ERR_INVALID_ARG, "bitstrings given with n_bitstrings == 0");
  if (L.bits_mode && !a.bitstrings) fail(HSF_ERR_INVALID_ARG, "n_bitstrings > 0 but bitstrings is NULL");
  if (L.bits_mode && P.n > 63) fail(HSF_ERR_INVALID_ARG, "bitstring runs need n <= 63");
  const int nA = P.n - P.n_low, nB = P.n_low;
  L.r0 = a.row_begin;
  L.r1 = a.row_end;
  if (L.r0 == 0 && L.r1 == 0) L.r1 = 1ull << nA;
  if (!L.bits_mode && (L.r0 >= L.r1 || L.r1 > (1ull << nA))) fail(HSF_ERR_INVALID_ARG, "bad row range");
  size_t off = 0;
  for (int h = 0; h < 2; ++h) {
    const Half& H = *L.half[h];
    const size_t st = (size_t)1 << H.m;
    for (size_t i = 0; i + 1 < H.trans.size(); ++i)
      L.scratch_elems[h] =
          std::max(L.scratch_elems[h], (size_t)nodes_at(L.hranks[h], H.trans[i].level_out, L.hp0[h], L.hp1[h]) * st);
    for (int b = 0; b < 2; ++b) {
      L.off_scratch[h][b] = off;
      off = align_up(off + L.scratch_elems[h] * elem);
    }
  }
  for (int h = 0; h < 2; ++h) {
    L.off_leaves[h] = off;
    off = align_up(off + ((size_t)(L.hp1[h] - L.hp0[h]) << L.half[h]->m) * elem);
  }
  if (L.bits_mode) {
    // block gather: >= 4 samples per block of the direct half (the one whose
    // tree the planner estimates to finish last: its leaves are read in place,
    // the other half is transposed beside its tree), complex64, K <= 512
    // (padded to a power of two >= 64), <= 2^15 blocks (the bucket sort's
    // shared histograms), samples < 2^31
    const int mA = L.half[0]->m, mB = L.half[1]->m;
    int dir = L.half[1]->est_ms >= L.half[0]->est_ms ? 1 : 0;
    if (const char* e = std::getenv("HSF_GATHER_DIRECT")) dir = std::atoi(e);  // tests: 0 / 1, -1 = per-sample gather
    const int mD = dir == 1 ? mB : mA;
    const int rb = gather_cfg() / 100 == 3 ? 32 : 16;
    if (dir >= 0 && P.opts.dtype == HSF_C64 && L.K <= 512 && mD >= 5 && (1ll << mD) / rb <= 32768 &&
        a.n_bitstrings < (1ull << 31) && (long long)a.n_bitstrings >= (4ll << mD) / rb) {
      L.direct = dir;
      L.Kp = 64;
      while (L.Kp < (long long)L.K) L.Kp *= 2;
      L.block_rows = rb;
      L.n_blocks = (1ll << mD) / rb;
      const int th = 1 - dir;
      const Half& HT = *L.half[th];
      const char* te = std::getenv("HSF_TLEAF");
      // (only without K padding: the T-leaf pass writes the K real columns)
      L.tleaf[th] = HT.tleaf && P.opts.jit && L.var[th] <= 1 && (long long)L.K == L.Kp &&
                    L.hp0[th] % (uint64_t)HT.tleaf_R == 0 &&
                    L.hp1[th] % (uint64_t)HT.tleaf_R == 0 && !(te && te[0] == '0');
    }
    for (int h = 0; h < 2; ++h) {
      if (h == L.direct) continue;
      L.off_T[h] = off;
      off = align_up(off + ((size_t)(L.direct >= 0 ? L.Kp : L.K) << L.half[h]->m) * elem);
    }
    if (!a.bits_on_device) {
      L.off_bits = off;
      off = align_up(off + a.n_bitstrings * 8);
    }
    if (!a.out_on_device) {
      L.off_out = off;
      off = align_up(off + a.n_bitstrings * elem);
    }
    if (P.permuted) {
      L.off_pbits = off;
      off = align_up(off + a.n_bitstrings * 8);
    }
    if (L.direct >= 0) {
      L.off_grp = off;
      off = align_up(off + (size_t)(3 * L.n_blocks + 1 + (long long)a.n_bitstrings) * 4);
      L.off_sbits = off;
      off = align_up(off + (size_t)a.n_bitstrings * 8);
    }
  } else {
    if (P.permuted) {
      if (!a.out_on_device || L.r0 != 0 || L.r1 != (1ull << nA))
        fail(HSF_ERR_UNSUPPORTED, "non-contiguous partitions need a device output and all rows in full-output runs");
      L.off_pout = off;
      off = align_up(off + ((size_t)1 << P.n) * elem);
    }
    if (L.prec != HSF_PREC_SIMT) {
      L.tc_bytes = L.swap ? tc_workspace_bytes((long long)L.K, 1ll << nB, swap_cols(L), tc_planes(L.prec))
                            : tc_workspace_bytes((long long)L.K, (long long)(L.r1 - L.r0), 1ll << nB, tc_planes(L.prec));
      L.off_tc = off;
      off = align_up(off + L.tc_bytes);
      if (L.swap) {
        L.off_swapT = off;
        off = align_up(off + ((size_t)swap_cols(L) << nB) * elem);
      }
    }
    if (!a.out_on_device && a.n_out_shards == 0) {
      // host output: rows are produced in chunks of <= kHostChunkBytes into two
      // device staging buffers; the D2H copy of one chunk overlaps the
      // path-sum of the next (bounded device memory for any output size)
      const size_t row_bytes = ((size_t)1 << nB) * elem;
      size_t chunk = kHostChunkBytes;
      if (const char* e = std::getenv("HSF_HOST_CHUNK_BYTES")) chunk = std::max<size_t>(1, std::strtoull(e, nullptr, 10));
      uint64_t cr = std::max<uint64_t>(1, chunk / row_bytes);
      if (L.prec != HSF_PREC_SIMT && !L.swap) cr = std::max<uint64_t>(128, cr / 128 * 128);  // whole tensor-core M tiles
      L.chunk_rows = std::min<uint64_t>(cr, L.r1 - L.r0);
      L.chunk_bytes = align_up(L.chunk_rows * row_bytes);
      L.off_out = off;
      off = align_up(off + 2 * L.chunk_bytes);
    }
  }
  L.total = off;
  return L;
}

static void ensure_ws(DeviceState* d, size_t bytes) {
  if (d->ws_bytes >= bytes) return;
  if (d->ws) CK(cudaFree(d->ws));
  d->ws = nullptr;
  d->ws_bytes = 0;
  cudaError_t e = cudaMalloc(&d->ws, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(HSF_ERR_OUT_OF_MEMORY, "device workspace of " + std::to_string(bytes) + " bytes");
  }
  d->ws_bytes = bytes;
}

// c_p = prod_u c_{u,d_u} over the tree's units for tree paths p in [p0, p1),
// fp64 on the host -> run dtype
// Tail weight table W[t][i] of half h (complex64 tensor-core runs with the
// half-sided fold), built at the first run that uses it -- outside any graph
// capture -- when it has <= 2^22 entries; else the operand prep loops over
// the folded units per element.
static void ensure_tailw(Plan* P, DeviceState* d, int h) {
  if (d->tailw[h] || d->elem != 8) return;
  const Plan::Tail& T = P->tail[h];
  const long long wld = 1ll << P->half[h].m;
  const char* nt = std::getenv("HSF_TAIL_NO_TABLE");  // tests: per-unit weight loop
  if (T.u0 < 0 || T.mask.empty() || (double)T.T * (double)wld > (double)(1 << 22) || (nt && nt[0] == '1')) return;
  CK(cudaMalloc(&d->tailw[h], (size_t)T.T * wld * sizeof(float2)));
  const tc::TailParams tp = tail_params(*P, h);
  const long long nel = (long long)T.T * wld;
  tc::tail_weights_kernel<<<(unsigned)((nel + 255) / 256), 256>>>(d->tailw[h], wld, tp, (const float2*)d->tail);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
}

// heads: bit h set => half h's head-scalar units (Plan::Tail::v0) are folded
// into c_p as well
static void ensure_cp(Plan* P, DeviceState* d, uint64_t p0, uint64_t p1, int U_tree, int heads, cudaStream_t st) {
  if (d->cp_p0 == p0 && d->cp_p1 == p1 && d->cp_units == U_tree && d->cp_heads == heads) return;
  const uint64_t K = p1 - p0;
  if (d->cp_cap < K) {
    if (d->cp) CK(cudaFree(d->cp));
    CK(cudaMalloc(&d->cp, K * d->elem));
    d->cp_cap = K;
  }
  const int U = U_tree;
  std::vector<cd> c(K);
  for (uint64_t p = p0; p < p1; ++p) {
    uint64_t x = p;
    cd v = 1.0;
    for (int u = U - 1; u >= 0; --u) {
      const int dg = (int)(x % P->ranks[u]);
      v *= P->units[u].c[dg];
      for (int h = 0; h < 2; ++h)
        if (((heads >> h) & 1) && u < P->tail[h].v0) v *= P->tail[h].head[u][dg];
      x /= P->ranks[u];
    }
    c[p - p0] = v;
  }
  if (P->opts.dtype == HSF_C64) {
    std::vector<float2> h(K);
    for (uint64_t i = 0; i < K; ++i) h[i] = make_float2((float)c[i].real(), (float)c[i].imag());
    CK(cudaMemcpyAsync(d->cp, h.data(), K * 8, cudaMemcpyHostToDevice, st));
  } else {
    CK(cudaMemcpyAsync(d->cp, c.data(), K * 16, cudaMemcpyHostToDevice, st));
  }
  CK(cudaStreamSynchronize(st));
  d->cp_p0 = p0;
  d->cp_p1 = p1;
  d->cp_units = U_tree;
  d->cp_heads = heads;
}

template <typename R>
static void run_half(const Plan& P, DeviceState* d, int h, const Layout& L, cudaStream_t st) {
  using C = typename cplx<R>::T;
  const Half& H = *L.half[h];
  const int var = L.var[h];
  DevOp* dops = var == 0 ? d->ops[h] : var == 1 ? d->ops_fold[h] : d->ops_tail[h];
  const std::vector<int32_t>& ranks = L.hranks[h];
  const uint64_t hp0 = L.hp0[h], hp1 = L.hp1[h];
  char* ws = (char*)d->ws;
  const size_t st_elems = (size_t)1 << H.m;
  const void* prev_buf = nullptr;
  int prev_level = -1;
  size_t pass_ord = 0;
  const std::vector<void*>* jf = d->jit ? &d->jit_fn[var][h] : nullptr;
  // Row light cone (full-output runs of half A over a row range): the rows'
  // constant index bits F (values those of r0) are all the path-sum reads.
  // A pass computes an output element from input elements with the same
  // non-tile bits (its ops stay inside its tile), so pass k needs only the
  // tiles whose non-tile bits in N_k agree with r0, N_last = F and
  // N_{k-1} = N_k minus pass k's tile qubits: need[k] = N_k.  (q33-3, 16
  // rows: the leaf level's first pass computes 4 of 32 tiles per node.)
  std::vector<uint32_t> need;
  const bool cone = h == 0 && !L.bits_mode && (L.r1 - L.r0) < (1ull << H.m);
  if (cone) {
    size_t np = 0;
    for (const Transition& tr : H.trans) np += tr.passes.size();
    need.assign(np, 0);
    const uint64_t diff = L.r0 ^ (L.r1 - 1);
    int hb = 0;
    while (hb < 64 && (diff >> hb) != 0) ++hb;
    uint32_t N = (uint32_t)(((1ull << H.m) - 1) & ~((1ull << hb) - 1));
    size_t k = np;
    for (size_t ti = H.trans.size(); ti-- > 0;)
      for (size_t pi = H.trans[ti].passes.size(); pi-- > 0;) {
        need[--k] = N;
        const Pass& ps = H.trans[ti].passes[pi];
        uint32_t tm = 0;
        if (ps.t < H.m)
          for (int q : ps.T) tm |= 1u << q;
        else
          tm = ~0u;
        N &= ~tm;
      }
  }
  for (size_t ti = 0; ti < H.trans.size(); ++ti) {
    const Transition& tr = H.trans[ti];
    const bool last = (ti + 1 == H.trans.size());
    if (last && L.tleaf[h] && d->jit_tl[var][h]) {
      // T-leaf: one CTA per (2^10-amplitude tile, parent) evaluates the
      // parent's R leaves and writes them transposed into the gather operand
      const Half& TL = *H.tleaf;
      const int Rl = H.tleaf_R;
      const uint64_t S_in = suffix_prod(ranks, tr.level_in);
      JitLaunchArgs ja{prev_buf, ws + L.off_T[h], d->coef, (long long)hp0, 0, (long long)(hp0 / S_in),
                       (long long)range_prod(ranks, tr.level_in, tr.level_out), 0u,
                       h != L.direct ? d->cp : nullptr, L.Kp};  // c_p rides on the transposed half
      // persistent CTAs over (tile, parent) items (tile_free carries the parent count)
      const uint64_t parents = (hp1 - hp0) / (uint64_t)Rl;
      ja.tile_free = (unsigned)parents;
      const size_t smem = jit_tleaf_smem_bytes(TL, Rl, true);
      const int per_sm = std::max(1, std::min(2, (int)((227u << 10) / smem)));
      const uint64_t items = parents << (H.m - 10);
      jit_launch(d->jit_tl[var][h], (unsigned)std::min<uint64_t>(items, (uint64_t)per_sm * num_sms()), 1u,
                 (unsigned)(64 * Rl), smem, st, ja, 0);
      break;
    }
    void* out = ws + (last ? L.off_leaves[h] : L.off_scratch[h][ti & 1]);
    const uint64_t S_out = suffix_prod(ranks, tr.level_out);
    const uint64_t first_out = hp0 / S_out;
    const uint64_t n_out = (hp1 - 1) / S_out - first_out + 1;
    for (size_t pi = 0; pi < tr.passes.size(); ++pi, ++pass_ord) {
      const Pass& ps = tr.passes[pi];
      PassParams pp{};
      pp.dst = out;
      pp.ops = dops + ps.op_begin;
      pp.n_ops = (int)(ps.op_end - ps.op_begin);
      pp.coef = d->coef;
      pp.m = H.m;
      pp.t = ps.t;
      pp.state_elems = (long long)st_elems;
      if (ps.t < H.m) {
        pp.n_hi = ps.t - 5;
        for (int j = 5; j < ps.t; ++j) pp.T_hi[j - 5] = ps.T[j];
        pp.n_nt = 0;
        for (int q = 0; q < H.m; ++q)
          if (std::find(ps.T.begin(), ps.T.end(), q) == ps.T.end()) pp.nonT[pp.n_nt++] = q;
        if (pp.n_nt > kMaxNonTile) fail(HSF_ERR_UNSUPPORTED, "half too large for the tile kernel");
      }
      const int n_ops = (int)(ps.op_end - ps.op_begin);
      size_t smem = (sizeof(C) << ps.t) + (ps.t < H.m ? (sizeof(uint32_t) << (ps.t - 5)) : 0);
      smem = ((smem + 15) & ~(size_t)15) + (size_t)n_ops * (sizeof(DevOp) + sizeof(void*));
      smem = ((smem + 15) & ~(size_t)15) + (size_t)ps.tbl_elems * sizeof(C);
      pp.tbl_elems = (int)ps.tbl_elems;
      uint64_t tiles = 1ull << (H.m - ps.t);
      pp.tile0 = 0;
      pp.tile_free = 0xFFFFFFFFu;
      if (cone && ps.t < H.m && need[pass_ord] && !(last && pi + 1 == tr.passes.size())) {
        uint32_t t0 = 0, fm = 0;
        for (int j = 0; j < pp.n_nt; ++j) {
          const int q = pp.nonT[j];
          if ((need[pass_ord] >> q) & 1u)
            t0 |= (uint32_t)((L.r0 >> q) & 1ull) << j;
          else
            fm |= 1u << j;
        }
        if (fm != (1u << pp.n_nt) - 1) {
          pp.tile0 = t0;
          pp.tile_free = fm;
          tiles = 1ull << __builtin_popcount(fm);
        }
      }
      // Row-restricted leaf pass: in full-output runs only rows [r0, r1) of
      // half A's leaves reach the path-sum, so the last pass of A's tree
      // computes only the tiles holding them (ops of a pass stay inside its
      // tile; tile index = the rows' non-tile bits, monotone in the row)
      if (h == 0 && !L.bits_mode && last && pi + 1 == tr.passes.size() && ps.t < H.m &&
          (L.r1 - L.r0) < (1ull << H.m)) {
        auto tile_of = [&](uint64_t i) {
          uint64_t tt = 0;
          for (int j = 0; j < pp.n_nt; ++j) tt |= ((i >> pp.nonT[j]) & 1ull) << j;
          return tt;
        };
        const uint64_t t0 = tile_of(L.r0), t1 = tile_of(L.r1 - 1);
        pp.tile0 = (unsigned)t0;
        tiles = t1 - t0 + 1;
      }
      // narrow levels (few CTAs) use one 1024-thread CTA per (node, tile) to
      // shorten the dependent chain of small launches at the top of the tree
      const bool wide = tiles * n_out < 2ull * (uint64_t)num_sms() && ps.t >= 11;
      auto kern = wide ? (ps.heavy ? hsf_pass_kernel<R, kSimThreadsWide, true> : hsf_pass_kernel<R, kSimThreadsWide, false>)
                       : (ps.heavy ? hsf_pass_kernel<R, kSimThreads, true> : hsf_pass_kernel<R, kSimThreads, false>);
      const int nthr = wide ? kSimThreadsWide : kSimThreads;
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      for (uint64_t y0 = 0; y0 < n_out; y0 += 65535) {
        const uint64_t ny = std::min<uint64_t>(65535, n_out - y0);
        pp.node_first = (long long)(first_out + y0);
        pp.node_local0 = (long long)y0;
        if (pi == 0) {
          if (prev_level < 0) {
            pp.src = nullptr;
          } else {
            pp.src = prev_buf;
            const uint64_t S_in = suffix_prod(ranks, prev_level);
            pp.src_first = (long long)(hp0 / S_in);
            pp.src_div = (long long)range_prod(ranks, prev_level, tr.level_out);
          }
        } else {  // in place on this level's buffer
          pp.src = out;
          pp.src_first = (long long)first_out;
          pp.src_div = 1;
        }
        const bool bop = h == 1 && L.bop && d->jit_bop && last && pi + 1 == tr.passes.size();
        const bool aop = h == 1 && L.aop && d->jit_aop && last && pi + 1 == tr.passes.size();
        if (aop) {  // swapped path-sum: write the MN-major M operand instead of the leaves
          TcBuffers t = tc_swap_buffers((long long)L.K, 1ll << H.m, swap_cols(L), tc_planes(L.prec), ws + L.off_tc,
                                        L.tc_bytes);
          JitLaunchArgs ja{pp.src, t.a_hi, pp.coef, pp.node_first, pp.node_local0, pp.src_first, pp.src_div, pp.tile0,
                           t.b_lo == nullptr ? nullptr : t.a_lo, t.d.rows_pad / 2};
          jit_launch(d->jit_aop, (unsigned)tiles, (unsigned)ny, (unsigned)d->jit_bop_nt, jit_smem_bytes(ps, true, 0), st,
                     ja, 0);
        } else if (bop) {  // K4 fused: write the MN-major split-bf16 B operand instead of the leaves
          TcBuffers t = tc_buffers((long long)L.K, (long long)(L.r1 - L.r0), 1ll << H.m, tc_planes(L.prec),
                                   ws + L.off_tc, L.tc_bytes);
          JitLaunchArgs ja{pp.src, t.b_hi, pp.coef, pp.node_first, pp.node_local0, pp.src_first, pp.src_div, pp.tile0,
                           t.b_lo, t.d.nrows_b_pad / 2};
          jit_launch(d->jit_bop, (unsigned)tiles, (unsigned)ny, (unsigned)d->jit_bop_nt, jit_smem_bytes(ps, true, 0), st,
                     ja, 0);
        } else if (jf) {
          JitLaunchArgs ja{pp.src, pp.dst, pp.coef, pp.node_first, pp.node_local0, pp.src_first, pp.src_div,
                           pp.tile0};
          ja.tile_free = pp.tile_free;
          const int cb = d->jit_cb[var][h][pass_ord];
          jit_launch((*jf)[pass_ord], (unsigned)tiles, (unsigned)ny, (unsigned)d->jit_nt[var][h][pass_ord],
                     jit_smem_bytes(ps, sizeof(R) == 4, cb), st, ja, cb);
        } else {
          dim3 grid((unsigned)tiles, (unsigned)ny);
          kern<<<grid, nthr, smem, st>>>(pp);
          CK(cudaGetLastError());
        }
      }
    }
    prev_buf = out;
    prev_level = tr.level_out;
  }
}

// Path-sum operand preparation for one half (runs on that half's stream):
// bitstring mode -> transpose (+ c_p fold for A) to [2^m][K]; full mode on the
// tensor cores -> split-bf16 K-major operands; SIMT full mode reads the
// node-major leaves directly (nothing to prepare).
template <typename R>
static void prep_half(Plan* P, DeviceState* d, const Layout& L, int h, cudaStream_t st) {
  using C = typename cplx<R>::T;
  char* ws = (char*)d->ws;
  const int m = P->half[h].m;
  const long long K = (long long)L.K;
  const C* leaves = (const C*)(ws + L.off_leaves[h]);
  if (L.bits_mode) {
    if (h == L.direct) return;  // read in place by the block gather
    // c_p (a3) is folded into the transposed half: half A in the per-sample
    // gather, the non-direct half in the block gather (whose staging then is
    // a plain copy)
    const bool with_cp = L.direct >= 0 ? h != L.direct : h == 0;
    if (L.tleaf[h] && d->jit_tl[L.var[h]][h]) return;  // written transposed by the half's T-leaf pass
    C* T = (C*)(ws + L.off_T[h]);
    const long long ldo = L.direct >= 0 ? L.Kp : K;
    const char* tv = std::getenv("HSF_TRANSPOSE_V1");
    if (sizeof(R) == 4 && m >= 1 && !(tv && tv[0] == '1')) {  // 16 B accesses (c5: 0.43 ms per half before)
      dim3 g((unsigned)(((1ll << m) + 63) / 64), (unsigned)((ldo + 31) / 32));
      transpose_fold_c64_kernel<<<g, dim3(32, 8), 0, st>>>((const float2*)leaves, (float2*)T,
                                                           with_cp ? (const float2*)d->cp : nullptr, K, 1ll << m, ldo);
    } else {
      if (ldo != K) fail(HSF_ERR_INVALID_ARG, "padded transpose needs the complex64 kernel");
      dim3 g((unsigned)(((1ll << m) + 31) / 32), (unsigned)((K + 31) / 32));
      transpose_fold_kernel<C><<<g, dim3(32, 8), 0, st>>>(leaves, T, with_cp ? (const C*)d->cp : nullptr, K, 1ll << m);
    }
    CK(cudaGetLastError());
  } else if (L.prec != HSF_PREC_SIMT) {
    const int nB = P->n_low;
    tc::TailParams tp = L.var[h] == 2 ? tail_params(*P, h) : tc::TailParams{};
    tp.p0 = (long long)L.p0;
    if (L.var[h] == 2) {
      tp.node0 = (long long)L.hp0[h];
      tp.W = d->tailw[h];
      tp.wld = 1ll << m;
    } else {
      tp.T = 1;
      tp.Tt = 1;
    }
    if (L.swap) {  // roles swapped: B's leaves -> M operand, A's rows (rotated, c_p) -> N operand
      TcBuffers t = tc_swap_buffers(K, 1ll << nB, swap_cols(L), tc_planes(L.prec), ws + L.off_tc, L.tc_bytes);
      if (h == 1) {
        if (!(L.aop && d->jit_aop))  // else written by half B's last pass
          tc_prep_a(t, (const float2*)leaves, nullptr, K, 1ll << m, 0, 1ll << m, tp, (const float2*)d->tail, st);
      } else
        tc_prep_b(t, (const float2*)leaves, K, (long long)(L.r1 - L.r0), tp, (const float2*)d->tail, st,
                  (const float2*)d->cp, (long long)L.r0, 1ll << m);
    } else if (h == 0) {
      TcBuffers t = tc_buffers(K, (long long)(L.r1 - L.r0), 1ll << nB, tc_planes(L.prec), ws + L.off_tc, L.tc_bytes);
      tc_prep_a(t, (const float2*)leaves, (const float2*)d->cp, K, 1ll << m, (long long)L.r0, (long long)(L.r1 - L.r0),
                tp, (const float2*)d->tail, st);
    } else if (!(L.bop && d->jit_bop)) {  // else written by half B's last pass
      TcBuffers t = tc_buffers(K, (long long)(L.r1 - L.r0), 1ll << nB, tc_planes(L.prec), ws + L.off_tc, L.tc_bytes);
      tc_prep_b(t, (const float2*)leaves, K, 1ll << m, tp, (const float2*)d->tail, st);
    }
  }
}

// Bitstring-run input prep, independent of the path trees (runs on the aux
// stream beside them): H2D of host bitstrings, the relabelling of
// non-contiguous partitions, the bits < 2^n check and the bucket sort of the
// block gather.
// Returns the device bitstrings in internal bit order.
static const unsigned long long* prep_bits(Plan* P, DeviceState* d, const Layout& L, const hsf_run_args& a,
                                           cudaStream_t st) {
  char* ws = (char*)d->ws;
  const int nB = P->n_low;
  const unsigned long long* bits = (const unsigned long long*)a.bitstrings;
  if (!a.bits_on_device) {
    bits = (const unsigned long long*)(ws + L.off_bits);
    CK(cudaMemcpyAsync((void*)bits, a.bitstrings, a.n_bitstrings * 8, cudaMemcpyHostToDevice, st));
  }
  const long long ns = (long long)a.n_bitstrings;
  if (P->permuted) {  // caller bit order -> internal (relabelled) bit order
    unsigned long long* pb = (unsigned long long*)(ws + L.off_pbits);
    permute_bits_kernel<<<(unsigned)std::min<long long>((ns + 255) / 256, 148ll * 8), 256, 0, st>>>(bits, pb, ns,
                                                                                                 d->perm_tab);
    CK(cudaGetLastError());
    bits = pb;
  }
  // precondition bits < 2^n (hsf.h): flagged in mapped host memory, checked
  // when the run synchronises
  check_bits_kernel<<<(unsigned)std::min<long long>((ns + 255) / 256, 148ll * 8), 256, 0, st>>>(bits, ns, P->n,
                                                                                              d->bad_bits_dev);
  if (L.direct >= 0) {
    const long long nblk = L.n_blocks;
    int* counts = (int*)(ws + L.off_grp);
    int* offs = counts + nblk;
    int* cursor = offs + nblk + 1;
    int* sidx = cursor + nblk;
    unsigned long long* sbits = (unsigned long long*)(ws + L.off_sbits);
    const int rb = L.block_rows == 32 ? 5 : 4;
    const int shift = L.direct == 1 ? rb : nB + rb;  // blocks of the direct half
    const unsigned long long kmask = (unsigned long long)nblk - 1ull;
    CK(cudaMemsetAsync(counts, 0, (size_t)nblk * 4, st));
    // per-CTA shared histograms of nblk ints (<= 128 KB: nblk <= 2^15, checked in make_layout)
    const size_t hsm = (size_t)nblk * 4;
    static bool hattr = false;
    if (!hattr) {
      CK(cudaFuncSetAttribute(bucket_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 << 10));
      CK(cudaFuncSetAttribute(bucket_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 << 10));
      hattr = true;
    }
    const int per_sm = std::max(1, std::min(2, (int)((200u << 10) / std::max<size_t>(hsm, 1))));
    const unsigned gb = (unsigned)std::max(1ll, std::min<long long>((ns + 4095) / 4096, (long long)per_sm * num_sms()));
    bucket_count_kernel<<<gb, 1024, hsm, st>>>(bits, ns, shift, kmask, (int)nblk, counts);
    bucket_scan_kernel<<<1, 1024, 0, st>>>(counts, offs, cursor, nblk);
    bucket_scatter_kernel<<<gb, 1024, hsm, st>>>(bits, ns, shift, kmask, (int)nblk, cursor, sidx, sbits);
    CK(cudaGetLastError());
  }
  return bits;
}

// bitstring path-sum (K6) into `out` (device)
template <typename R>
static void run_core_bits(Plan* P, DeviceState* d, const Layout& L, const hsf_run_args& a, cudaStream_t st,
                          typename cplx<R>::T* out, const unsigned long long* bits) {
  using C = typename cplx<R>::T;
  char* ws = (char*)d->ws;
  const int nB = P->n_low;
  const long long K = (long long)L.K;
  const C* AT = (const C*)(ws + L.off_T[0]);
  const C* BT = (const C*)(ws + L.off_T[1]);
  const long long ns = (long long)a.n_bitstrings;
  long long blocks = std::min<long long>((ns + 7) / 8, 148ll * 64);
  TrailParams tw{};
  if (L.fold) {
    tw.n = (int)P->trail_mask.size();
    for (int u = 0; u < tw.n; ++u) {
      tw.mask[u] = P->trail_mask[u];
      tw.off[u] = P->trail_off[u];
    }
    // the deferred final diagonals of the kernels that produced the leaves
    // (the direct half's are applied to its staged rows by the block gather)
    for (int h = 0; h < 2 && d->jit; ++h) {
      const int kind = (L.tleaf[h] && d->jit_tl[1][h]) ? 1 : 0;
      if (h == L.direct && sizeof(R) == 4) continue;
      for (const auto& un : d->dfin_units[kind][h]) {
        if (tw.n >= kMaxTrail) fail(HSF_ERR_UNSUPPORTED, "too many per-sample weight tables");
        tw.mask[tw.n] = un.first;
        tw.off[tw.n] = un.second;
        ++tw.n;
      }
    }
  }
  const unsigned long long maskA = (P->n - nB >= 64) ? ~0ull : (1ull << (P->n - nB)) - 1ull;
  if (sizeof(R) == 4 && L.direct >= 0) {  // bucket sort done by prep_bits
    const long long nblk = L.n_blocks;
    BlockGatherParams bp{};
    bp.D = (const float2*)(ws + L.off_leaves[L.direct]);
    bp.ldD = 1ll << L.half[L.direct]->m;
    bp.K = K;
    bp.cpD = nullptr;  // c_p is in the transposed half
    bp.T = (const float4*)(ws + L.off_T[1 - L.direct]);
    bp.offs = (const int*)(ws + L.off_grp) + nblk;
    bp.sidx = bp.offs + 2 * nblk + 1;
    bp.sbits = (const unsigned long long*)(ws + L.off_sbits);
    bp.out = (float2*)out;
    bp.n_blocks = nblk;
    bp.n_low = nB;
    bp.direct_b = L.direct;
    bp.maskA = maskA;
    bp.maskB = (1ull << nB) - 1ull;
    bp.accumulate = a.accumulate;
    if (const char* e = std::getenv("HSF_GATHER_DEBUG")) bp.debug = std::atoi(e);
    bp.n_shards = a.n_out_shards;
    bp.shard_len = (long long)a.shard_rows;
    for (int o = 0; o < a.n_out_shards; ++o) bp.shard[o] = (float2*)a.out_shards[o];
    bp.multicast = a.shards_multicast;
    if (const char* e = std::getenv("HSF_GATHER_LD")) bp.ldmode = std::atoi(e);
    if (L.fold && d->jit) {  // the direct half's deferred final diagonal, per staged row
      const int hd = L.direct, kind = (L.tleaf[hd] && d->jit_tl[1][hd]) ? 1 : 0;
      const int first = P->half[hd].first_qubit;
      bp.dtab = (const float2*)d->trail;
      for (const auto& un : d->dfin_units[kind][hd]) {
        if (bp.dnr >= 4) fail(HSF_ERR_UNSUPPORTED, "too many deferred-diagonal tables");
        const int lo = __builtin_ctzll(un.first);
        bp.dlo[bp.dnr] = lo - first;
        bp.dmask[bp.dnr] = (unsigned)(un.first >> lo);
        bp.doff[bp.dnr] = un.second;
        ++bp.dnr;
      }
    }
    const size_t smem = (size_t)L.block_rows * L.Kp * sizeof(float2);
    auto launch = [&](auto kern, int nt) {
      static std::vector<const void*> attr;  // kernels whose SMEM limit is raised (all share one type)
      if (std::find(attr.begin(), attr.end(), (const void*)kern) == attr.end()) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr.push_back((const void*)kern);
      }
      int per_sm = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nt, smem));
      const long long grid = std::min<long long>(nblk, (long long)std::max(1, per_sm) * num_sms());
      kern<<<(unsigned)grid, nt, smem, st>>>(bp, tw, (const float2*)d->trail);
    };
    // tuning (HSF_GATHER_CFG = 100 * (RB == 32 ? 3 : 1) + 10 * MINB + U)
    // default U by row length (c5, Kp = 128: U = 4 -> gather 1.09 ms, U = 2 1.38;
    // c3, Kp = 256: U = 2 -> 0.25 ms, U = 4 0.45 -- 64 float4 of rows per
    // thread spill at 4 CTAs per SM)
    // min CTAs/SM: 4 (64 registers) for Kp <= 128; 3 for Kp = 256 (c3: 0.254 vs 0.273 ms)
    const int cfg = gather_cfg(),
              MB = std::getenv("HSF_GATHER_CFG") ? (cfg / 10) % 10 : (L.Kp >= 256 ? 3 : 4);
    const int U = std::getenv("HSF_GATHER_CFG") ? cfg % 10 : L.Kp <= 64 ? 8 : L.Kp == 128 ? 4 : L.Kp == 256 ? 2 : 1;
#define HSF_GB(NF, U_, RB, MB_) launch(gather_block_c64_kernel<NF, U_, RB, 256, MB_>, 256)
#define HSF_GB_MB(NF, U_, RB)     \
  if (MB == 2) HSF_GB(NF, U_, RB, 2); \
  else if (MB == 3) HSF_GB(NF, U_, RB, 3); \
  else HSF_GB(NF, U_, RB, 4);
#define HSF_GB_RB(NF, U_)            \
  if (L.block_rows == 16) {          \
    HSF_GB_MB(NF, U_, 16)            \
  } else {                           \
    HSF_GB_MB(NF, U_, 32)            \
  }
    switch (L.Kp) {
      case 64: if (U == 8) { HSF_GB_RB(1, 8) } else { HSF_GB_RB(1, 4) } break;
      case 128: if (U == 8) { HSF_GB_RB(2, 8) } else if (U == 4) { HSF_GB_RB(2, 4) } else { HSF_GB_RB(2, 2) } break;
      case 256: if (U == 4) { HSF_GB_RB(4, 4) } else { HSF_GB_RB(4, 2) } break;
      case 512: if (U == 2) { HSF_GB_RB(8, 2) } else { HSF_GB_RB(8, 1) } break;
#undef HSF_GB_RB
#undef HSF_GB_MB
#undef HSF_GB
      default: fail(HSF_ERR_INVALID_ARG, "block gather row length");
    }
  } else if (sizeof(R) == 4 && K % 64 == 0) {
    gather_dot_c64_vec_kernel<<<(unsigned)blocks, 256, 0, st>>>((const float4*)AT, (const float4*)BT, bits,
                                                                (float2*)out, ns, K, nB, tw, (const float2*)d->trail,
                                                                a.accumulate, maskA);
  } else {
    gather_dot_kernel<C><<<(unsigned)blocks, 256, 0, st>>>(AT, BT, bits, out, ns, K, nB, tw, (const C*)d->trail,
                                                           a.accumulate, maskA);
  }
  CK(cudaGetLastError());
}

// full-output path-sum (K5 / K5s) of rows [L.r0 + lo, L.r0 + lo + nrows) into `out`
// (device, row-major [nrows][2^nB]); lo is a multiple of the tensor-core M tile
template <typename R>
static void run_core_full(Plan* P, DeviceState* d, const Layout& L, cudaStream_t st, uint64_t lo, uint64_t nrows,
                          typename cplx<R>::T* out, bool accumulate, const hsf_run_args* shards = nullptr) {
  using C = typename cplx<R>::T;
  char* ws = (char*)d->ws;
  const int nA = P->n - P->n_low, nB = P->n_low;
  const long long K = (long long)L.K;
  if (L.prec == HSF_PREC_SIMT) {
    const C* leavesA = (const C*)(ws + L.off_leaves[0]);
    const C* leavesB = (const C*)(ws + L.off_leaves[1]);
    dim3 grid((unsigned)(((1ll << nB) + 63) / 64), (unsigned)((nrows + 63) / 64));
    simt_gemm_kernel<C, R><<<grid, 256, 0, st>>>(leavesA, leavesB, (const C*)d->cp, out, K, 1ll << nA, 1ll << nB,
                                                 (long long)(L.r0 + lo), (long long)nrows, accumulate ? 1 : 0);
    CK(cudaGetLastError());
  } else {
    if (sizeof(R) != 4) fail(HSF_ERR_UNSUPPORTED, "tensor-core path-sum needs complex64");
    if (L.swap) {  // outT[j][i] over all 2^nB columns and the run's rows, then out[i][j]
      // (host-output chunks: the GEMM runs with the first chunk, each chunk transposes its rows)
      const long long Rw = swap_cols(L), MBl = 1ll << nB;
      float2* outT = (float2*)(ws + L.off_swapT);
      if (lo == 0)
        tc_gemm(tc_swap_buffers(K, MBl, Rw, tc_planes(L.prec), ws + L.off_tc, L.tc_bytes), outT, Rw, 0, MBl, st);
      swap_transpose_kernel<<<dim3((unsigned)((MBl + 31) / 32), (unsigned)((nrows + 31) / 32)), dim3(32, 8), 0, st>>>(
          outT + lo, (float2*)out, (long long)nrows, MBl, Rw, accumulate ? 1 : 0);
      CK(cudaGetLastError());
      return;
    }
    TcBuffers t = tc_buffers(K, (long long)(L.r1 - L.r0), 1ll << nB, tc_planes(L.prec), ws + L.off_tc,
                             L.tc_bytes);
    if (shards && shards->n_out_shards > 0)
      tc_gemm(t, nullptr, 1ll << nB, (long long)lo, (long long)nrows, st, true, shards->out_shards,
              shards->n_out_shards, (long long)shards->shard_rows);
    else
      tc_gemm(t, (float2*)out, 1ll << nB, (long long)lo, (long long)nrows, st, accumulate);
  }
}

template <typename R>
static void run_all(Plan* P, DeviceState* d, const Layout& L, const hsf_run_args& a, cudaStream_t st, bool timed) {
  using C = typename cplx<R>::T;
  // timing events become graph nodes when the run is being captured
  auto rec = [&](cudaEvent_t e, cudaStream_t s) {
    CK(cudaEventRecordWithFlags(e, s, d->capturing ? cudaEventRecordExternal : cudaEventRecordDefault));
  };
  if (timed) rec(d->ev_t0, st);
  // half B (and its operand prep) on the side stream, half A on the caller's
  // stream; the two path trees are independent until the path-sum
  CK(cudaEventRecord(d->ev[0], st));
  CK(cudaStreamWaitEvent(d->side, d->ev[0], 0));
  const unsigned long long* bits_d = nullptr;
  if (L.bits_mode) {  // bitstring prep on the aux stream, beside both trees
    CK(cudaStreamWaitEvent(d->aux, d->ev[0], 0));
    bits_d = prep_bits(P, d, L, a, d->aux);
    CK(cudaEventRecord(d->ev_aux, d->aux));
  }
  run_half<R>(*P, d, 1, L, d->side);
  if (timed) rec(d->ev[2], d->side);
  prep_half<R>(P, d, L, 1, d->side);
  CK(cudaEventRecord(d->ev[5], d->side));
  run_half<R>(*P, d, 0, L, st);
  if (timed) rec(d->ev[1], st);
  prep_half<R>(P, d, L, 0, st);
  CK(cudaStreamWaitEvent(st, d->ev[5], 0));
  if (timed) rec(d->ev[3], st);
  char* ws = (char*)d->ws;
  if (L.bits_mode) {
    C* out = a.n_out_shards > 0 ? nullptr : a.out_on_device ? (C*)a.out : (C*)(ws + L.off_out);
    CK(cudaStreamWaitEvent(st, d->ev_aux, 0));
    run_core_bits<R>(P, d, L, a, st, out, bits_d);
    if (!a.out_on_device && a.n_out_shards == 0)
      CK(cudaMemcpyAsync(a.out, out, (size_t)a.n_bitstrings * sizeof(C), cudaMemcpyDeviceToHost, st));
  } else if (a.out_on_device && P->permuted) {
    // internal-order result into the workspace, then back to the caller's qubit order
    C* tmp = (C*)(ws + L.off_pout);
    run_core_full<R>(P, d, L, st, 0, L.r1 - L.r0, tmp, false);
    const long long nout = 1ll << P->n;
    permute_out_kernel<C><<<(unsigned)std::min<long long>((nout + 255) / 256, 148ll * 32), 256, 0, st>>>(
        tmp, (C*)a.out, nout, d->perm_tab, a.accumulate);
    CK(cudaGetLastError());
  } else if (a.n_out_shards > 0) {  // fused reduce-scatter into the owners' shards
    run_core_full<R>(P, d, L, st, 0, L.r1 - L.r0, nullptr, true, &a);
  } else if (a.out_on_device) {
    run_core_full<R>(P, d, L, st, 0, L.r1 - L.r0, (C*)a.out, a.accumulate != 0);
  } else {
    // host output: double-buffered chunks, path-sum on `st`, D2H on `side`
    const uint64_t rows = L.r1 - L.r0;
    const size_t row_bytes = sizeof(C) << P->n_low;
    int c = 0;
    for (uint64_t lo = 0; lo < rows; lo += L.chunk_rows, ++c) {
      const uint64_t nr = std::min<uint64_t>(L.chunk_rows, rows - lo);
      C* buf = (C*)(ws + L.off_out + (size_t)(c & 1) * L.chunk_bytes);
      if (c >= 2) CK(cudaStreamWaitEvent(st, d->evc[c & 1], 0));
      run_core_full<R>(P, d, L, st, lo, nr, buf, false);
      CK(cudaEventRecord(d->evg[c & 1], st));
      CK(cudaStreamWaitEvent(d->side, d->evg[c & 1], 0));
      CK(cudaMemcpyAsync((char*)a.out + lo * row_bytes, buf, nr * row_bytes, cudaMemcpyDeviceToHost, d->side));
      CK(cudaEventRecord(d->evc[c & 1], d->side));
    }
    for (int i = 0; i < std::min(c, 2); ++i) CK(cudaStreamWaitEvent(st, d->evc[i], 0));
  }
  if (a.comm && a.coll != HSF_COLL_NONE) {  // the exchange step (contributions added up)
    Comm* cm = reinterpret_cast<Comm*>(a.comm);
    const bool f64 = sizeof(R) == 8;
    const size_t n = L.bits_mode ? (size_t)a.n_bitstrings : ((size_t)(L.r1 - L.r0) << P->n_low);
    if (a.coll == HSF_COLL_ALLREDUCE)
      comm_allreduce(cm, a.out, 2 * n, f64, st);
    else
      comm_reduce_scatter(cm, a.out, a.coll_out, 2 * n / comm_nranks(cm), f64, st);
  }
  if (timed) rec(d->ev[4], st);
}

static void run(Plan* P, const hsf_run_args& a) {
  DeviceState* d = ensure_device(P, a.device);
  Layout L = make_layout(*P, a, d->elem);
  if (a.n_out_shards < 0 || a.n_out_shards > 8) fail(HSF_ERR_INVALID_ARG, "n_out_shards must be in 0..8");
  if (a.n_out_shards > 0 && L.bits_mode) {
    // fused exchange of bitstring runs: the block gather reduce-adds each
    // sample into its owner's shard (samples [o * shard_rows, (o+1) * shard_rows))
    if (L.direct < 0 || P->opts.dtype != HSF_C64)
      fail(HSF_ERR_UNSUPPORTED, "owner-sharded bitstring output needs the complex64 block gather");
    if (!a.out_shards || a.shard_rows == 0 || a.shard_rows * (uint64_t)a.n_out_shards < a.n_bitstrings ||
        a.shard_rows * (uint64_t)(a.n_out_shards - 1) >= a.n_bitstrings)
      fail(HSF_ERR_INVALID_ARG, "out_shards: n_out_shards pointers of shard_rows samples covering all samples");
    for (int o = 0; o < a.n_out_shards; ++o)
      if (!a.out_shards[o]) fail(HSF_ERR_INVALID_ARG, "out_shards[o] is NULL");
    if (a.shards_multicast && a.n_out_shards != 1)
      fail(HSF_ERR_INVALID_ARG, "a multicast output is one shard holding every sample");
  } else if (a.n_out_shards > 0) {
    if (a.shards_multicast) fail(HSF_ERR_UNSUPPORTED, "multicast output is for bitstring runs");
    if (L.prec == HSF_PREC_SIMT || P->permuted || L.r0 != 0 || L.r1 != (1ull << (P->n - P->n_low)))
      fail(HSF_ERR_UNSUPPORTED, "fused reduce-scatter needs a full-output tensor-core run over all rows of a "
                                "contiguous cut");
    if (!a.out_shards || a.shard_rows == 0 || a.shard_rows % 256 ||
        a.shard_rows * (uint64_t)a.n_out_shards != (1ull << (P->n - P->n_low)))
      fail(HSF_ERR_INVALID_ARG, "out_shards: n_out_shards pointers of shard_rows rows (a multiple of 256) "
                                "covering all 2^nA rows");
    for (int o = 0; o < a.n_out_shards; ++o)
      if (!a.out_shards[o]) fail(HSF_ERR_INVALID_ARG, "out_shards[o] is NULL");
  } else if (!a.out) {
    fail(HSF_ERR_INVALID_ARG, "out is NULL");
  }
  if (a.accumulate && !a.out_on_device && a.n_out_shards == 0)
    fail(HSF_ERR_INVALID_ARG, "accumulate needs a device output buffer");
  if ((int)a.coll < (int)HSF_COLL_NONE || (int)a.coll > (int)HSF_COLL_REDUCE_SCATTER)
    fail(HSF_ERR_INVALID_ARG, "unknown collective");
  if (a.coll != HSF_COLL_NONE) {
    if (!a.comm) fail(HSF_ERR_INVALID_ARG, "collective without a communicator");
    Comm* cm = reinterpret_cast<Comm*>(a.comm);
    if (!a.out_on_device || a.n_out_shards > 0 || P->permuted)
      fail(HSF_ERR_UNSUPPORTED, "the exchange step needs a device output (no out_shards, contiguous cut)");
    if (comm_device(cm) != d->device) fail(HSF_ERR_INVALID_ARG, "communicator bound to another device");
    if (a.coll == HSF_COLL_REDUCE_SCATTER) {
      if (L.bits_mode) fail(HSF_ERR_INVALID_ARG, "reduce-scatter is for full outputs");
      if ((L.r1 - L.r0) % (uint64_t)comm_nranks(cm)) fail(HSF_ERR_INVALID_ARG, "rows not divisible by nranks");
      if (!a.coll_out) fail(HSF_ERR_INVALID_ARG, "reduce-scatter needs coll_out");
    }
    const uint64_t key = comm_serial(cm);
    if (std::find(d->comm_ok.begin(), d->comm_ok.end(), key) == d->comm_ok.end()) {
      if (!comm_same_hash(cm, P->hash, (cudaStream_t)a.cuda_stream))
        fail(HSF_ERR_PLAN_MISMATCH, "ranks of the communicator hold different plans (plan_hash differs)");
      d->comm_ok.push_back(key);
    }
  }
  ensure_ws(d, L.total);
  cudaStream_t st = (cudaStream_t)a.cuda_stream;
  int heads = 0;
  for (int h = 0; h < 2; ++h)
    if (L.var[h] == 2 && P->tail[h].v0 > 0) heads |= 1 << h;
  ensure_cp(P, d, L.p0, L.p1, L.U_tree, heads, st);
  for (int h = 0; h < 2; ++h)
    if (L.var[h] == 2) ensure_tailw(P, d, h);
  const bool timed = a.phase_ms != nullptr;
  try {
    const char* ng = std::getenv("HSF_NO_GRAPH");
    // page-locked host buffers of a bitstring run (H2D of the samples, D2H of
    // the amplitudes) are captured as graph memcpy nodes too; pageable ones
    // are not capturable, those runs launch directly
    auto pinned = [](const void* ptr) {
      if (!ptr) return false;
      cudaPointerAttributes at{};
      if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
      }
      return at.type == cudaMemoryTypeHost;
    };
    const bool out_ok = a.out_on_device || a.n_out_shards > 0 || (L.bits_mode && pinned(a.out));
    const bool bits_ok = !L.bits_mode || a.bits_on_device || pinned(a.bitstrings);
    const bool graph = P->opts.graphs && out_ok && bits_ok && !(ng && ng[0] == '1');
    if (graph) {
      // the key holds everything the captured launches depend on
      std::vector<uint64_t> key = {(uint64_t)(uintptr_t)a.out, (uint64_t)(uintptr_t)a.bitstrings, a.n_bitstrings,
                                   L.p0, L.p1, L.r0, L.r1, (uint64_t)L.prec, (uint64_t)a.accumulate,
                                   (uint64_t)timed, (uint64_t)L.fold, (uint64_t)(uintptr_t)d->ws,
                                   (uint64_t)(uintptr_t)d->cp, (uint64_t)L.total, (uint64_t)a.n_out_shards,
                                   a.shard_rows, (uint64_t)L.swap, (uint64_t)L.bop,
                                   (uint64_t)a.out_on_device, (uint64_t)a.bits_on_device,
                                   (uint64_t)(uintptr_t)a.comm, (uint64_t)a.coll, (uint64_t)(uintptr_t)a.coll_out,
                                   (uint64_t)a.shards_multicast};
      for (int o = 0; o < a.n_out_shards; ++o) key.push_back((uint64_t)(uintptr_t)a.out_shards[o]);
      if (!d->gexec || key != d->gkey) {
        if (d->gexec) CK(cudaGraphExecDestroy(d->gexec));
        d->gexec = nullptr;
        d->gkey.clear();
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(d->cap, cudaStreamCaptureModeThreadLocal));
        d->capturing = true;
        try {
          if (P->opts.dtype == HSF_C64)
            run_all<float>(P, d, L, a, d->cap, timed);
          else
            run_all<double>(P, d, L, a, d->cap, timed);
        } catch (...) {
          d->capturing = false;
          cudaStreamEndCapture(d->cap, &g);
          if (g) cudaGraphDestroy(g);
          throw;
        }
        d->capturing = false;
        CK(cudaStreamEndCapture(d->cap, &g));
        {
          size_t nn = 0;
          CK(cudaGraphGetNodes(g, nullptr, &nn));
          std::vector<cudaGraphNode_t> nodes(nn);
          if (nn) CK(cudaGraphGetNodes(g, nodes.data(), &nn));
          int nk = 0;
          for (auto nd : nodes) {
            cudaGraphNodeType ty;
            CK(cudaGraphNodeGetType(nd, &ty));
            nk += ty == cudaGraphNodeTypeKernel ? 1 : 0;
          }
          d->gkernels = nk;
        }
        cudaError_t e = cudaGraphInstantiate(&d->gexec, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) fail(HSF_ERR_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
        d->gkey = key;
      }
      CK(cudaGraphLaunch(d->gexec, st));
    } else if (P->opts.dtype == HSF_C64) {
      run_all<float>(P, d, L, a, st, timed);
    } else {
      run_all<double>(P, d, L, a, st, timed);
    }
    if (timed || !a.out_on_device) {
      CK(cudaStreamSynchronize(st));
      if (L.bits_mode && *(volatile unsigned int*)d->bad_bits) {
        *d->bad_bits = 0;
        fail(HSF_ERR_INVALID_ARG, "bitstrings must be < 2^n (a sample has a bit set at or above qubit n)");
      }
    }
    if (timed) {
      float tA, tB, tprep, tcore, ttot;
      CK(cudaEventElapsedTime(&tA, d->ev_t0, d->ev[1]));
      CK(cudaEventElapsedTime(&tB, d->ev_t0, d->ev[2]));
      CK(cudaEventElapsedTime(&tprep, d->ev_t0, d->ev[3]));
      CK(cudaEventElapsedTime(&tcore, d->ev[3], d->ev[4]));
      CK(cudaEventElapsedTime(&ttot, d->ev_t0, d->ev[4]));
      a.phase_ms[0] = tA;
      a.phase_ms[1] = tB;
      a.phase_ms[2] = tprep - std::max(tA, tB);
      a.phase_ms[3] = tcore;
      a.phase_ms[4] = ttot;
    }
  } catch (Error& e) {
    if (e.st == HSF_ERR_CUDA) d->sticky = true;
    throw;
  }
}

}  // namespace hsf

using namespace hsf;

#define ABI_GUARD(...)                         \
  try {                                        \
    __VA_ARGS__;                               \
    return HSF_OK;                             \
  } catch (const Error& e) {                   \
    set_last_error(e.msg);                     \
    return e.st;                               \
  } catch (const std::bad_alloc&) {            \
    set_last_error("host allocation failed");  \
    return HSF_ERR_OUT_OF_MEMORY;              \
  } catch (const std::exception& e) {          \
    set_last_error(e.what());                  \
    return HSF_ERR_INVALID_ARG;                \
  } catch (...) {                              \
    set_last_error("unknown C++ exception");   \
    return HSF_ERR_INVALID_ARG;                \
  }

extern "C" {

hsf_status hsf_plan_opts_default(hsf_plan_opts* o) {
  if (!o) return HSF_ERR_INVALID_ARG;
  o->dtype = HSF_C64;
  o->svd_rel_tol = 1e-12;
  o->max_dense_block_qubits = 10;
  o->log2_path_budget = 26;
  o->individual = 0;
  o->tile_qubits = 0;
  o->fuse_gates = 1;
  o->hoist_gates = 1;
  o->fold_trailing_diag = 1;
  o->jit = 1;
  o->graphs = 1;
  o->analytic_cascades = 1;
  o->smem_tier = 0;
  o->block_route = 0;
  o->partition_b = 0;
  return HSF_OK;
}

hsf_status hsf_plan(const char* text, size_t len, int32_t n_low, int64_t n_blocks, const int64_t* off,
                    const int64_t* ids, const hsf_plan_opts* opts, hsf_plan_t** out) {
  ABI_GUARD({
    if (!text || !out) fail(HSF_ERR_INVALID_ARG, "NULL argument");
    if (n_blocks < -1) fail(HSF_ERR_INVALID_ARG, "n_blocks < -1");
    *out = nullptr;
    hsf_plan_opts o;
    hsf_plan_opts_default(&o);
    if (opts) o = *opts;
    if (o.block_route < 0 || o.block_route > 2) fail(HSF_ERR_INVALID_ARG, "block_route must be 0, 1 or 2");
    if (o.tile_qubits != 0 && (o.tile_qubits < 10 || o.tile_qubits > 13))
      fail(HSF_ERR_INVALID_ARG, "tile_qubits must be 0 (auto) or in [10,13]");
    if (o.dtype != HSF_C64 && o.dtype != HSF_C128) fail(HSF_ERR_INVALID_ARG, "bad dtype");
    if (!(o.svd_rel_tol >= 0 && o.svd_rel_tol < 1)) fail(HSF_ERR_INVALID_ARG, "bad svd_rel_tol");
    if (o.max_dense_block_qubits < 1 || o.max_dense_block_qubits > 12) fail(HSF_ERR_INVALID_ARG, "bad max_dense_block_qubits");
    *out = reinterpret_cast<hsf_plan_t*>(build_plan(text, len, n_low, n_blocks, off, ids, o));
  })
}

hsf_status hsf_plan_info_get(const hsf_plan_t* plan, hsf_plan_info* info) {
  ABI_GUARD({
    if (!plan || !info) fail(HSF_ERR_INVALID_ARG, "NULL argument");
    const Plan* P = reinterpret_cast<const Plan*>(plan);
    info->n_qubits = P->n;
    info->n_a = P->n - P->n_low;
    info->n_b = P->n_low;
    info->n_units = (int32_t)P->units.size();
    info->n_paths = P->n_paths;
    info->log2_n_paths_individual = P->log2_individual;
    info->ranks = P->ranks.data();
    info->support_a = P->sa.data();
    info->support_b = P->sb.data();
    info->sigma_offsets = P->sigma_off.data();
    info->sigmas = P->sigmas.data();
    info->levels_a = (int32_t)P->half[0].materialized.size();
    info->levels_b = (int32_t)P->half[1].materialized.size();
    info->passes_a = P->half[0].n_passes;
    info->passes_b = P->half[1].n_passes;
    info->ops_a = (int32_t)P->half[0].ops.size();
    info->ops_b = (int32_t)P->half[1].ops.size();
    info->plan_hash = P->hash;
    info->fold_units = P->fold_u0 >= 0 ? (int32_t)P->units.size() - P->fold_u0 : 0;
    info->tree_bytes_a = P->half[0].tree_bytes;
    info->tree_bytes_b = P->half[1].tree_bytes;
    info->fold_tree_bytes_a = P->fold_u0 >= 0 ? P->half_fold[0].tree_bytes : 0.0;
    info->fold_tree_bytes_b = P->fold_u0 >= 0 ? P->half_fold[1].tree_bytes : 0.0;
    info->fold_passes_a = P->fold_u0 >= 0 ? P->half_fold[0].n_passes : 0;
    info->fold_passes_b = P->fold_u0 >= 0 ? P->half_fold[1].n_passes : 0;
    for (int h = 0; h < 2; ++h) {
      const Plan::Tail& T = P->tail[h];
      const bool on = T.u0 >= 0;
      const int nu = on ? (int)P->units.size() - T.u0 : 0;
      (h ? info->tail_units_b : info->tail_units_a) = nu;
      (h ? info->head_units_b : info->head_units_a) = on ? T.v0 : 0;
      (h ? info->tail_passes_b : info->tail_passes_a) = on ? T.half.n_passes : 0;
      (h ? info->tail_tree_bytes_b : info->tail_tree_bytes_a) = on ? T.half.tree_bytes : 0.0;
    }
    info->tree_flops_a = P->half[0].tree_flops;
    info->tree_flops_b = P->half[1].tree_flops;
    info->fold_tree_flops_a = P->fold_u0 >= 0 ? P->half_fold[0].tree_flops : 0.0;
    info->fold_tree_flops_b = P->fold_u0 >= 0 ? P->half_fold[1].tree_flops : 0.0;
    info->tail_tree_flops_a = P->tail[0].u0 >= 0 ? P->tail[0].half.tree_flops : 0.0;
    info->tail_tree_flops_b = P->tail[1].u0 >= 0 ? P->tail[1].half.tree_flops : 0.0;
    info->n_analytic_units = 0;
    for (int32_t x : P->unit_analytic) info->n_analytic_units += x;
    info->unit_analytic = P->unit_analytic.data();
    info->unit_sequential = P->unit_sequential.data();
    for (int h = 0; h < 2; ++h) {
      const Half& H = P->half[h];
      (h ? info->whole_state_b : info->whole_state_a) =
          !H.trans.empty() && !H.trans[0].passes.empty() && H.trans[0].passes[0].t == H.m ? 1 : 0;
    }
    info->n_joint_blocks = 0;
    for (const auto& un : P->units) info->n_joint_blocks += un.gids.size() > 1 ? 1 : 0;
  })
}

hsf_status hsf_run(hsf_plan_t* plan, const hsf_run_args* args) {
  ABI_GUARD({
    if (!plan || !args) fail(HSF_ERR_INVALID_ARG, "NULL argument");
    run(reinterpret_cast<Plan*>(plan), *args);
  })
}

// ---- CUDA IPC of output shards (fused reduce-scatter plumbing) ----------
typedef CUresult (*PFN_memGetAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);

hsf_status hsf_ipc_export(const void* dev_ptr, void* handle_out, uint64_t* offset_out) {
  ABI_GUARD({
    if (!dev_ptr || !handle_out || !offset_out) fail(HSF_ERR_INVALID_ARG, "NULL argument");
    static PFN_memGetAddressRange range = nullptr;
    if (!range) {
      void* f = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess || !f)
        fail(HSF_ERR_CUDA, "cuMemGetAddressRange entry point unavailable");
      range = (PFN_memGetAddressRange)f;
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, (CUdeviceptr)(uintptr_t)dev_ptr) != CUDA_SUCCESS)
      fail(HSF_ERR_INVALID_ARG, "pointer is not device memory of this context");
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, (void*)(uintptr_t)base));
    std::memcpy(handle_out, &h, sizeof(h));
    *offset_out = (uint64_t)((uintptr_t)dev_ptr - (uintptr_t)base);
  })
}

hsf_status hsf_ipc_import(const void* handle, uint64_t offset, void** dev_ptr_out) {
  ABI_GUARD({
    if (!handle || !dev_ptr_out) fail(HSF_ERR_INVALID_ARG, "NULL argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* base = nullptr;
    CK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *dev_ptr_out = (char*)base + offset;
  })
}

hsf_status hsf_ipc_release(void* dev_ptr, uint64_t offset) {
  ABI_GUARD({
    if (!dev_ptr) fail(HSF_ERR_INVALID_ARG, "NULL argument");
    CK(cudaIpcCloseMemHandle((char*)dev_ptr - offset));
  })
}

hsf_status hsf_run_describe(const hsf_plan_t* plan, const hsf_run_args* args, hsf_run_desc* out) {
  ABI_GUARD({
    if (!plan || !args || !out) fail(HSF_ERR_INVALID_ARG, "NULL argument");
    const Plan* P = reinterpret_cast<const Plan*>(plan);
    const size_t elem = P->opts.dtype == HSF_C64 ? 8 : 16;
    const Layout L = make_layout(*P, *args, elem);
    hsf_run_desc& o = *out;
    std::memset(&o, 0, sizeof(o));
    const int nA = P->n - P->n_low, nB = P->n_low;
    const double K = (double)L.K, MB = std::ldexp(1.0, nB);
    o.K = L.K;
    o.direct_half = L.direct;
    o.tleaf_half = L.tleaf[0] ? 0 : L.tleaf[1] ? 1 : -1;
    o.tleaf_leaves = o.tleaf_half >= 0 ? L.half[o.tleaf_half]->tleaf_R : 0;
    o.tree_variant_a = L.var[0];
    o.tree_variant_b = L.var[1];
    for (int h = 0; h < 2; ++h) {  // this range's share of the evaluated tree
      const Half& H = *L.half[h];
      const double tot = (double)range_prod(L.hranks[h], 0, (int)L.hranks[h].size());
      const double frac = (double)(L.hp1[h] - L.hp0[h]) / std::max(1.0, tot);
      o.sim_bytes[h] = H.tree_bytes * frac;
      o.sim_flops[h] = H.tree_flops * frac;
    }
    if (L.bits_mode) {
      const double ns = (double)args->n_bitstrings;
      o.rows = args->n_bitstrings;
      o.core_flops_useful = o.core_flops_executed = 8.0 * K * ns;
      if (L.direct >= 0) {
        o.core = HSF_CORE_BLOCK_GATHER;
        const double mD = L.half[L.direct]->m, mT = L.half[1 - L.direct]->m;
        // D's leaves once, one padded T row + sample index, bits and result per sample
        o.core_bytes = K * std::ldexp(1.0, (int)mD) * elem + ns * ((double)L.Kp * elem + 4 + 8 + elem);
        // the T half's transpose (none when its T-leaf pass writes the rows: the
        // leaf level's bytes, counted in sim_bytes, are then the operand's)
        o.prep_bytes = L.tleaf[1 - L.direct] ? 0.0 : 2.0 * K * std::ldexp(1.0, (int)mT) * elem;
      } else {
        o.core = HSF_CORE_GATHER;
        o.core_bytes = ns * (2.0 * K * elem + 8 + elem);
        o.prep_bytes = 2.0 * K * (std::ldexp(1.0, L.half[0]->m) + std::ldexp(1.0, L.half[1]->m)) * elem;
      }
    } else {
      const double rows = (double)(L.r1 - L.r0);
      o.rows = L.r1 - L.r0;
      o.core_flops_useful = 8.0 * K * rows * MB;
      if (L.prec == HSF_PREC_SIMT) {
        o.core = HSF_CORE_SIMT;
        o.core_flops_executed = o.core_flops_useful;
        o.core_bytes = K * (rows + MB) * elem + rows * MB * elem;
      } else {
        const int planes = tc_planes(L.prec);
        const int prods = L.prec == HSF_PREC_BF16X6 ? 6 : L.prec == HSF_PREC_BF16X1 ? 1 : 3;
        const double esz = L.prec == HSF_PREC_TF32X3 ? 4.0 : 2.0;
        const double pl = L.prec == HSF_PREC_TF32X3 ? 2.0 : (double)planes;
        o.tc_products = prods;
        const double Kp = (double)((L.K + 31) / 32 * 32);
        if (L.swap) {
          o.core = HSF_CORE_TC_SWAPPED;
          const double R = (double)swap_cols(L);
          const double bn = std::ceil(2.0 * R / 32.0) * 32.0;
          o.core_flops_executed = prods * 2.0 * MB * bn * 2.0 * Kp;
          // M operand (half B's planes, 2K rows) read once, the narrow N operand,
          // the fp32 [2^nB][2R] GEMM output written and read by the transpose, the result
          o.core_bytes = pl * esz * 2.0 * Kp * (MB + bn) + 2.0 * MB * 2.0 * R * 4.0 + rows * MB * elem;
        } else {
          o.core = rows > 128 ? HSF_CORE_TC_PAIR : HSF_CORE_TC_SINGLE;
          const double rp = std::ceil(rows / 128.0) * 128.0;
          o.core_flops_executed = prods * 2.0 * rp * (2.0 * MB) * (2.0 * Kp);
          // operand planes read once (A'' rows x 2K, B'' 2 MB rows x 2K) + the output written
          o.core_bytes = pl * esz * 2.0 * Kp * (rp + 2.0 * MB) + rows * MB * elem;
        }
        o.prep_bytes = K * (rows + MB) * elem + pl * esz * 2.0 * Kp * (rows + 2.0 * MB);
      }
    }
    o.kernel_launches = -1;
    const auto* d = (const DeviceState*)P->dev;
    if (d && d->gexec) o.kernel_launches = d->gkernels;
  })
}

size_t hsf_workspace_bytes(const hsf_plan_t* plan, const hsf_run_args* args) {
  try {
    if (!plan || !args) return 0;
    const Plan* P = reinterpret_cast<const Plan*>(plan);
    return make_layout(*P, *args, P->opts.dtype == HSF_C64 ? 8 : 16).total;
  } catch (const Error& e) {
    set_last_error(e.msg);
    return 0;
  }
}

void hsf_plan_free(hsf_plan_t* plan) {
  if (!plan) return;
  Plan* P = reinterpret_cast<Plan*>(plan);
  try {
    destroy_device(P);
  } catch (...) {
  }
  delete P;
}

const char* hsf_status_str(hsf_status s) {
  switch (s) {
    case HSF_OK: return "HSF_OK";
    case HSF_ERR_INVALID_ARG: return "HSF_ERR_INVALID_ARG";
    case HSF_ERR_PARSE: return "HSF_ERR_PARSE";
    case HSF_ERR_UNSUPPORTED_GATE: return "HSF_ERR_UNSUPPORTED_GATE";
    case HSF_ERR_DUPLICATE_QUBIT: return "HSF_ERR_DUPLICATE_QUBIT";
    case HSF_ERR_NONCONVEX_BLOCK: return "HSF_ERR_NONCONVEX_BLOCK";
    case HSF_ERR_BLOCK_TOO_LARGE: return "HSF_ERR_BLOCK_TOO_LARGE";
    case HSF_ERR_SVD_NO_CONVERGENCE: return "HSF_ERR_SVD_NO_CONVERGENCE";
    case HSF_ERR_PATH_BUDGET: return "HSF_ERR_PATH_BUDGET";
    case HSF_ERR_OUT_OF_MEMORY: return "HSF_ERR_OUT_OF_MEMORY";
    case HSF_ERR_CUDA: return "HSF_ERR_CUDA";
    case HSF_ERR_UNSUPPORTED: return "HSF_ERR_UNSUPPORTED";
    case HSF_ERR_NCCL: return "HSF_ERR_NCCL";
    case HSF_ERR_PLAN_MISMATCH: return "HSF_ERR_PLAN_MISMATCH";
  }
  return "HSF_ERR_UNKNOWN";
}

size_t hsf_last_error(char* buf, size_t len) {
  const std::string& m = g_last_error;
  if (buf && len) {
    size_t n = std::min(len - 1, m.size());
    std::memcpy(buf, m.data(), n);
    buf[n] = 0;
  }
  return m.size();
}

size_t hsf_debug_pass_source(const hsf_plan_t* plan, int32_t variant, int32_t half, int32_t pass, char* buf,
                             size_t len) {
  try {
    const Plan* P = reinterpret_cast<const Plan*>(plan);
    if (variant & 64) {  // bit 6: the T-leaf variant of that tree's last transition
      const int v = variant & 3;
      if (!P || half < 0 || half > 1 || v > 1 || (v == 1 && P->fold_u0 < 0)) return 0;
      const Half& H = v ? P->half_fold[half] : P->half[half];
      if (!H.tleaf) return 0;
      const std::string s = jit_tleaf_source(*H.tleaf, H.tleaf_R, P->opts.dtype == HSF_C64, &P->coef);
      if (buf && len) {
        const size_t n = std::min(len - 1, s.size());
        std::memcpy(buf, s.data(), n);
        buf[n] = 0;
      }
      return s.size();
    }
    const int cbq = (variant >> 2) & 3;  // bits 2-3: cluster-tier variant with 2^cb CTAs per tile
    const int store = (variant >> 4) & 3;  // bits 4-5: store mode (1 B operand, 2 transposed leaf)
    variant &= 3;                        // 0 full tree, 1 bitstring fold, 2 half-sided tail
    if (!P || half < 0 || half > 1 || variant > 2 || (variant == 1 && P->fold_u0 < 0) ||
        (variant == 2 && P->tail[half].u0 < 0))
      return 0;
    const Half& H = variant == 0 ? P->half[half] : variant == 1 ? P->half_fold[half] : P->tail[half].half;
    int k = 0;
    for (const auto& tr : H.trans)
      for (const auto& ps : tr.passes)
        if (k++ == pass) {
          const int nt = cbq ? std::max(128, 1 << (ps.t - cbq - 4)) : 256;
          DeferOut df;
          const bool lastp = variant == 1 && &tr == &H.trans.back() && &ps == &tr.passes.back();
          const std::string s = jit_pass_source(H, ps, P->opts.dtype == HSF_C64, nt, ps.t < H.m ? cbq : 0, &P->coef,
                                                store, lastp ? &df : nullptr);
          if (buf && len) {
            const size_t n = std::min(len - 1, s.size());
            std::memcpy(buf, s.data(), n);
            buf[n] = 0;
          }
          return s.size();
        }
    return 0;
  } catch (...) {
    return 0;
  }
}

const char* hsf_version(void) { return "libhsf 0.1 sm_100a (tcgen05 bf16x3 path-sum, SMEM/tile-pass simulator)"; }

}  // extern "C"
