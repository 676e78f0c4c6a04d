// hsf_internal.h — host-side plan structures shared by plan.cpp and run.cu.
// Not part of the ABI (include/hsf.h is).
#pragma once

#include <complex>
#include <memory>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/hsf.h"

namespace hsf {

using cd = std::complex<double>;

struct Error {
  hsf_status st;
  std::string msg;
};
[[noreturn]] void fail(hsf_status st, const std::string& msg);
void set_last_error(const std::string& msg);

// ---------------------------------------------------------------- circuit
struct Gate {
  std::string name;
  int k = 0;
  std::vector<int> q;   // as listed in the file: q[0] = MSB of the local index
  std::vector<cd> U;    // 2^k x 2^k row-major
  bool diag = false;    // every off-diagonal entry exactly zero
};

// ------------------------------------------------------------ cut units
struct Unit {
  std::vector<int> gids;           // member gates (file order)
  std::vector<int> support, Sa, Sb;// ascending global qubit ids
  bool diag_route = false;         // all members diagonal => diagonal factors
  bool analytic = false;           // factors from the closed-form cascade route (Eq. 11)
  bool sequential = false;         // factors from the sequential (MPO-style) route
  int rank = 0;
  std::vector<double> sigma;       // kept singular values (descending)
  std::vector<cd> c;               // sigma_m / sqrt(2^|S|)
  // per term: dense (2^k x 2^k row-major) or diagonal (2^k) matrices with
  // local index LSB = smallest support qubit of that side
  std::vector<std::vector<cd>> X, Y;
  double log2_individual = 0;      // only for reporting
};

// ------------------------------------------------------------ device ops
// OP_DENSE : SMEM sweep of a dense k-qubit op (q = tile positions)
// OP_DIAG  : diagonal op, elementwise (q = half-local qubits, any position)
// OP_RPASS : register pass header: q[0..3] = tile positions of the 4 register
//            qubits, k = number of following OP_R1 / OP_DIAG ops applied to
//            2^4 amplitudes held in registers per thread
// OP_R1    : 1-qubit dense op inside a register pass, q[0] = register slot
enum OpKind : int32_t { OP_DENSE = 0, OP_DIAG = 1, OP_RPASS = 2, OP_R1 = 3 };
constexpr int kRegQ = 4;          // register qubits per pass (16 amplitudes/thread)
constexpr int kMaxPassOps = 128;  // ops per kernel pass (all staged in SMEM)
constexpr int kSmemTableQ = 8;     // diag tables with <= 2^8 entries are staged in SMEM
constexpr int kSmemTableBytes = 48 * 1024;  // per-pass cap on staged tables
constexpr int kMaxOpQ = 13;      // widest diagonal op (2^13 entries)
constexpr int kMaxDenseQ = 5;    // widest dense op in the SMEM kernels
constexpr int kMaxFoldUnits = 8;  // folded trailing diagonal units (bitstring runs)
constexpr int kMaxTrail = 16;    // folded trailing diagonal units + deferred-diagonal tables (bitstring runs)
constexpr int kMaxTail = 16;     // half-sided trailing diagonal factors (full-output operand prep)
constexpr double kTailPrefixBytes = 16.0 * (1 << 20);  // prefix-leaf budget (HSF_TAIL_PREFIX_BYTES mode)
constexpr double kTailTableEntries = 1 << 20;           // default: tail weight table W[T][2^m] cap

// One operation of a half-circuit program (half-local qubits, LSB-first:
// q[j] is bit j of the op's local index).
struct HostOp {
  int kind = OP_DENSE;
  int k = 0;
  int q[kMaxOpQ] = {0};
  int unit = -1;        // >= 0: Schmidt factor of this unit, matrix selected by digit
  int64_t table = 0;    // complex offset of the digit-0 matrix in the coef table
  int64_t stride = 0;   // complex elements between digit matrices
};

// POD mirrored byte-for-byte on the device (see sim_kernels.cuh).
struct DevOp {
  int32_t kind, k;
  int32_t q[kMaxOpQ];   // dense: tile positions; diag: half-local qubit ids
  int32_t radix;        // 1 for fixed ops
  int32_t nruns;        // diag: contiguous qubit runs (1..3 => fast index), 0 => generic
  uint8_t rshift[4];    // run r covers index bits [roff[r], roff[r]+rlen[r]) taken
  uint8_t rlen[4];      //   from state bits [rshift[r], rshift[r]+rlen[r])
  uint8_t roff[4];
  int32_t soff;         // diag: element offset of this op's table in the pass's SMEM
                        // table area, -1 => read from global (L2)
  int64_t div;          // factor digit = (node_global / div) % radix
  int64_t table, stride;
};
static_assert(sizeof(DevOp) == 112, "DevOp layout");

struct Pass {
  int t = 0;                 // tile qubits (t == m => whole state in SMEM)
  std::vector<int> T;        // T[i] = half qubit of tile position i
  int64_t op_begin = 0, op_end = 0;  // into Half::dev_ops
  int64_t tbl_elems = 0;             // SMEM table area (complex elements)
  bool heavy = false;                // needs register passes / 3..5-qubit dense ops
};

struct Transition {
  int level_in = -1;         // -1 => start from |0...0>
  int level_out = 0;
  std::vector<Pass> passes;
};

struct Half {
  int m = 0;                 // qubits in this half
  int first_qubit = 0;       // global id of half-local qubit 0
  std::vector<HostOp> ops;   // after fusion
  std::vector<int64_t> seg_end;      // seg_end[l] = ops index after seg_l, l = 0..U
  std::vector<int> materialized;     // ascending levels; always contains U
  std::vector<Transition> trans;
  std::vector<DevOp> dev_ops;
  int n_passes = 0;
  double est_ms = 0;                 // planner's cost-model estimate of the tree (all paths)
  int last_gate_level = 0;           // deepest level holding a local gate
  double tree_bytes = 0;             // state bytes the tile passes read + write (all paths)
  double tree_flops = 0;             // their floating-point operations (all paths; FMA = 2)
  // T-leaf variant of the last transition (bitstring runs, the half the block
  // gather reads transposed): one pass over 2^10-amplitude tiles evaluating all
  // tleaf_R leaves of a parent per CTA and writing them transposed ([2^m][Kp]
  // rows, c_p folded for half A) -- no leaf buffer, no transpose kernel
  std::shared_ptr<struct Half> tleaf;
  int tleaf_R = 0;
};

struct Plan {
  int n = 0, n_low = 0;
  // non-contiguous partition: new index of caller qubit q (identity if none)
  std::vector<int> relabel;
  bool permuted = false;
  hsf_plan_opts opts{};
  std::vector<Gate> gates;
  std::vector<Unit> units;          // schedule order
  std::vector<int32_t> ranks, sa, sb;
  std::vector<int32_t> unit_analytic;  // per unit: closed-form cascade factors
  std::vector<int32_t> unit_sequential;  // per unit: sequential (MPO-style) route
  std::vector<int64_t> sigma_off;
  std::vector<double> sigmas;
  uint64_t n_paths = 1;
  double log2_individual = 0;
  std::vector<cd> coef;             // all device matrices (fp64 master copy)
  Half half[2];                     // 0 = A (high), 1 = B (low)
  // trailing-diagonal fold (bitstring runs; see build_plan)
  int fold_u0 = -1;                 // tree depth of the folded variant, -1 => none
  uint64_t fold_T = 1;              // product of the folded units' ranks
  Half half_fold[2];
  std::vector<uint64_t> trail_mask; // per folded unit: global support bits
  std::vector<int64_t> trail_off;   // per folded unit: offset into trail_tab
  std::vector<cd> trail_tab;        // per folded unit: block diagonal D_u over its support
  // half-sided trailing fold (full-output tensor-core runs; see build_plan):
  // units [u0, U) whose half-h factors are diagonal with no gate of half h
  // after them are applied while the GEMM operand is prepared
  struct Tail {
    int u0 = -1;                    // tree depth of half h, -1 => no variant (U => head fold only)
    int v0 = 0;                     // head-scalar units [0, v0) (radix 1 in this tree)
    uint64_t T = 1;                 // product of the tail units' ranks
    uint64_t Tt = 1;                // product of the tree units' ranks [v0, u0)
    std::vector<std::vector<cd>> head;  // per head unit, per digit: its scalar on half h
    Half half;                      // half h's tree over units [v0, u0)
    std::vector<uint32_t> mask;     // per folded unit: half-local support bits
    std::vector<int32_t> radix;     // per folded unit: rank
    std::vector<int64_t> off;       // per folded unit: offset of digit 0 in tail_tab
  } tail[2];
  std::vector<cd> tail_tab;         // diagonal factors (X for A, Y for B), 2^|S_h| per digit
  uint64_t hash = 0;
  void* dev = nullptr;              // device state (run.cu)
};

Plan* build_plan(const char* text, size_t len, int n_low, int64_t n_blocks, const int64_t* off,
                 const int64_t* ids, const hsf_plan_opts& opts);

// node-count helpers (levels 0..U; level l = after the first l units)
inline uint64_t suffix_prod(const std::vector<int32_t>& r, int from) {
  uint64_t s = 1;
  for (size_t v = from; v < r.size(); ++v) s *= (uint64_t)r[v];
  return s;
}
inline uint64_t range_prod(const std::vector<int32_t>& r, int from, int to) {  // [from, to)
  uint64_t s = 1;
  for (int v = from; v < to; ++v) s *= (uint64_t)r[v];
  return s;
}

void destroy_device(Plan* p);

}  // namespace hsf
