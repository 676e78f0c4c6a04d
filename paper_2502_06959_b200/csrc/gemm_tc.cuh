// gemm_tc.cuh — tensor-core (tcgen05) split-bf16 complex path-sum (K4 + K5).
// Placeholder until the tcgen05 kernel lands: reports HSF_ERR_UNSUPPORTED.
#pragma once
#include <cuda_runtime.h>

#include "hsf_internal.h"

namespace hsf {

inline size_t tc_workspace_bytes(long long K, long long rows, long long MB, bool x3) {
  (void)K; (void)rows; (void)MB; (void)x3;
  return 0;
}

inline void tc_path_sum(const float2*, const float2*, const float2*, float2*, long long, long long, long long,
                        long long, long long, bool, void*, size_t, cudaStream_t) {
  fail(HSF_ERR_UNSUPPORTED, "tcgen05 path-sum not built yet");
}

}  // namespace hsf
