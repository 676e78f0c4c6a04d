"""B200-native joint-cut Hybrid Schroedinger-Feynman path evaluator
(arXiv 2502.06959).  Host planner + CUDA sm_100a kernels in libhsf.so behind
the C ABI include/hsf.h; this package is the thin Python binding."""
from .hsf import Plan, HsfError, lib, version  # noqa: F401
from .dist import path_range_for_rank, row_range_for_rank, make_shard, run_sharded  # noqa: F401
