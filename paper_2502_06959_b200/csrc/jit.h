// jit.h — run-time specialised simulator passes (jit.cpp).  Not ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <complex>
#include <string>
#include <vector>

#include "hsf_internal.h"

namespace hsf {

// Mirrors JitArgs in jit_prelude.cuh (passed by value to the kernel).
struct JitLaunchArgs {
  const void* src;
  void* dst;
  const void* coef;
  long long node_first, node_local0, src_first, src_div;
  unsigned tile0;
  void* dst_lo = nullptr;
  long long ldw = 0;
  unsigned tile_free = 0xFFFFFFFFu;  // see PassParams::tile_free
};

// Deferred final diagonals (last pass of a bitstring-fold half): the
// register passes' left diagonals still pending when the pass ends are not
// applied; the leaves are then D_fin^-1-scaled and the gather multiplies each
// sample by D_fin(i_half) = scalar x prod_q (bit q of i ? phase[q] : 1).
struct DeferOut {
  bool active = false;
  std::vector<std::pair<int, std::complex<double>>> phase;  // half-local qubit, phase of |1>
  std::complex<double> scalar = 1.0;
};

// CUDA source of the kernel "hsf_jit_pass" specialised to one tile pass.
// coef (plan master table, optional): fixed gate matrices become literals
// store_mode 1: write the MN-major split-bf16 B operand instead of the leaf
// (JitArgs dst / dst_lo / ldw; row pair 2k, 2k+1 for output node k);
// store_mode 3: the swapped path-sum's MN-major M operand (st_aop)
std::string jit_pass_source(const Half& H, const Pass& ps, bool c64, int threads = 256, int cluster_bits = 0,
                            const std::vector<cd>* coef = nullptr, int store_mode = 0, DeferOut* defer = nullptr);
// T-leaf variant (Half::tleaf): one CTA per (tile, parent) evaluates the
// parent's `leaves` leaves and writes them transposed into the gather operand
// (JitArgs dst = operand [2^m][ldw], dst_lo = c_p of half A or nullptr)
// (64 threads per leaf: launch with 64 * leaves threads)
std::string jit_tleaf_source(const Half& TL, int leaves, bool c64, const std::vector<cd>* coef,
                             DeferOut* defer = nullptr);
size_t jit_tleaf_smem_bytes(const Half& TL, int leaves, bool c64);
// dynamic shared memory of that kernel (tile + staged diagonal tables)
size_t jit_smem_bytes(const Pass& ps, bool c64, int cluster_bits = 0);
// NVRTC-compile (cached per device and source, parallel) and load; returns CUfunctions
std::vector<void*> jit_compile_all(int device, const std::vector<std::string>& sources);
void jit_launch(void* fn, unsigned gx, unsigned gy, unsigned threads, size_t smem, void* stream,
                const JitLaunchArgs& a, int cluster_bits = 0);
uint64_t jit_source_hash(const std::string& s);

}  // namespace hsf
