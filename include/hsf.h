/*
 * hsf.h — C ABI of libhsf.so: joint-cut Hybrid Schroedinger-Feynman (HSF)
 * path evaluation on NVIDIA B200 (sm_100a).
 *
 * Method: arXiv 2502.06959 (PAPER.md, cited as P:<line>).
 *   - HSF partitions the qubits into halves a (high) and b (low); every gate
 *     crossing the cut is replaced by a bipartite (Schmidt) representation
 *     A = sum_m sigma_m X_m (x) Y_m  (Eq. 4).  Each choice of one
 *     term per cut unit is a "path"; n_p = prod_i r_i.  The result is
 *     the sum over paths of c_p psi_A^p (x) psi_B^p.
 *   - Joint cutting groups gates into blocks, multiplies them and
 *     Schmidt-decomposes the block unitary via reshape (Eq. 5-6,
 *     P:163-172), SVD (Eq. 7) and absorption of U, V* into the factors
 *     (Eq. 8-9).
 *
 * Conventions:
 *   - qubit 0 is the least-significant bit of a basis index;
 *   - n_low = number of qubits in half B = qubits [0, n_low); half A = the
 *     paper's partition a = qubits [n_low, n); the paper's cut position
 *     l = n_low - 1;
 *   - full output index i = i_A * 2^n_low + i_B, row-major [2^nA][2^nB];
 *   - complex numbers are interleaved (re, im), complex64 = 2 x float32,
 *     complex128 = 2 x float64;
 *   - bitstring bit q = qubit q (uint64, so n <= 63 for bitstring runs);
 *   - paths are numbered mixed-radix over the cut units in schedule order,
 *     last unit fastest.
 *
 * Errors: every call returns hsf_status; HSF_OK == 0.  No C++ exception or
 * abort crosses the ABI.  A thread-local message describing the last error is
 * available through hsf_last_error().  On error the output buffer contents are
 * undefined; the plan stays valid unless the status is HSF_ERR_CUDA.
 *
 * Threading: a plan is immutable after hsf_plan() except for its device
 * workspace; hsf_run() calls on one plan must be serialised by the caller.
 */
#ifndef HSF_H_
#define HSF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HSF_OK = 0,
  HSF_ERR_INVALID_ARG = 1,       /* null pointer, bad size, bad cut, bad range */
  HSF_ERR_PARSE = 2,             /* malformed circuit text (message has the line) */
  HSF_ERR_UNSUPPORTED_GATE = 3,  /* unknown gate name or arity */
  HSF_ERR_DUPLICATE_QUBIT = 4,   /* a gate lists a qubit twice / qubit out of range */
  HSF_ERR_NONCONVEX_BLOCK = 5,   /* a block is not convex in the wire DAG */
  HSF_ERR_BLOCK_TOO_LARGE = 6,   /* dense block > max_dense_block_qubits, or a
                                    dense factor on > 5 qubits of one half */
  HSF_ERR_SVD_NO_CONVERGENCE = 7,
  HSF_ERR_PATH_BUDGET = 8,       /* n_p exceeds 2^log2_path_budget */
  HSF_ERR_OUT_OF_MEMORY = 9,     /* host or device allocation failed */
  HSF_ERR_CUDA = 10,             /* CUDA runtime error (sticky for the plan) */
  HSF_ERR_UNSUPPORTED = 11,      /* valid request this build does not handle */
  HSF_ERR_NCCL = 12,             /* NCCL missing or an NCCL call failed (communicator) */
  HSF_ERR_PLAN_MISMATCH = 13     /* the ranks of a communicator hold different plans */
} hsf_status;

typedef enum { HSF_C64 = 0, HSF_C128 = 1 } hsf_dtype;

/* Arithmetic of the full-output path-sum Psi = (Psi_A diag(c)) Psi_B^T
 * (P:109).  Half-state simulation always runs in the plan dtype. */
typedef enum {
  HSF_PREC_AUTO = 0,    /* c64: BF16X3 ; c128: FP64 SIMT */
  HSF_PREC_SIMT = 1,    /* CUDA-core FMA in the plan dtype (fp32 / fp64) */
  HSF_PREC_BF16X3 = 2,  /* tcgen05 bf16 MMA, fp32 accumulate in TMEM, operands
                           split hi+lo, 3 products (hi*hi + hi*lo + lo*hi) */
  HSF_PREC_BF16X1 = 3,  /* tcgen05 bf16 MMA, single product (error study only) */
  HSF_PREC_BF16X6 = 4,  /* tcgen05 bf16 MMA, operands split hi+lo+lo2, 6 products
                           (+ lo*lo + hi*lo2 + lo2*hi): 2x the MMA work; the error then
                           sits at the tensor core's fp32 accumulation floor */
  HSF_PREC_TF32X3 = 5   /* tcgen05 kind::tf32 MMA (half the bf16 rate), operands split
                           hi+lo tf32 (cvt.rna), 3 products, K-major fp32 storage */
} hsf_precision;

typedef struct {
  hsf_dtype dtype;               /* default HSF_C64 */
  double svd_rel_tol;            /* drop sigma_m <= tol * sigma_0; default 1e-12 */
  int32_t max_dense_block_qubits;/* default 10 (dense block assembly O(D^3)) */
  double log2_path_budget;       /* default 26 */
  int32_t individual;            /* 1 => ignore blocks, cut every crossing gate alone */
  int32_t tile_qubits;           /* in [10,13]: amplitudes per SMEM tile = 2^tile_qubits for
                                    halves larger than the SMEM-resident limit (2^14
                                    complex64 / 2^13 complex128 amplitudes: whole state in
                                    one CTA) and for any half with m > tile_qubits (forces
                                    the tiled tier); 0 => auto (default): 12, widened to 13
                                    for complex64 where that saves an HBM pass */
  int32_t fuse_gates;            /* 1 (default) => host gate fusion */
  int32_t hoist_gates;           /* 1 (default) => commutation-aware path tree: a local gate
                                    is hoisted above every cut unit whose factors it commutes
                                    with (disjoint support, or both diagonal), so it runs once
                                    per shared prefix node; 0 => schedule order */
  int32_t fold_trailing_diag;    /* 1 (default) => bitstring runs fold trailing all-diagonal
                                    units with no gate after them into a per-sample weight
                                    (the block's diagonal at the sample's bits) instead of
                                    extending the path tree; and full-output tensor-core runs
                                    fold trailing units whose factors on one half are diagonal
                                    with no gate of that half after them into that half's
                                    operand prep (leaf = prefix leaf x diagonal factors);
                                    results are identical up to rounding */
  int32_t jit;                   /* 1 (default) => every simulator tile pass runs as a kernel
                                    specialised to its op list (generated CUDA, NVRTC for
                                    sm_100a, compiled at the first hsf_run on a device and
                                    cached per process); 0 => generic interpreter kernel */
  uint64_t partition_b;          /* 0 (default) => contiguous cut: half B = qubits [0, n_low).
                                    Otherwise the bit mask of half B's qubits (any subset,
                                    popcount == n_low): qubits are relabelled internally (B
                                    qubits keep their order at [0, n_low), A qubits at
                                    [n_low, n)); bitstrings and full outputs stay in the
                                    caller's qubit order.  Full-output runs then need a device
                                    output and all rows. */
  int32_t graphs;                /* 1 (default) => runs with device buffers are captured once
                                    into a CUDA graph (both streams, all launches) and replayed
                                    while pointers, ranges and precision stay the same */
  int32_t analytic_cascades;     /* 1 (default) => a block that is a cascade of two-qubit gates
                                    on one common qubit, each block-diagonal in that qubit's
                                    computational basis (CNOT, CZ, CP, RZZ; Eq. 11),
                                    gets its rank-<=2 Schmidt factors in closed form (no block
                                    assembly or SVD; sigma equal to the SVD's); 0 => numeric
                                    route for every block */
  int32_t smem_tier;             /* K1 tier (whole half state in one CTA's shared memory,
                                    north_star part (1)): 0 (default) => halves up to 2^13
                                    complex64 / 2^12 complex128 always, 2^14 / 2^13 (128 KiB,
                                    one CTA per SM) where the planner's cost model prefers it
                                    to 2^12-2^13 tiles; 1 => every half that fits */
  int32_t block_route;           /* dense (non-diagonal, non-cascade) blocks: 0 (default) =>
                                    sequential route from 8 support qubits on, assembly below;
                                    1 => assembly of the 2^s x 2^s block + SVD of the reshaped
                                    matrix (Eq. 6-9; s <= max_dense_block_qubits); 2 =>
                                    sequential (MPO-style) route: factors built gate by gate
                                    across the cut and recompressed to the operator-Schmidt
                                    form after each crossing gate (no block assembly).
                                    Either way dense factors are <= 5 qubits per side. */
} hsf_plan_opts;

typedef struct hsf_plan_s hsf_plan_t; /* opaque */
typedef struct hsf_comm_s hsf_comm_t; /* opaque: NCCL communicator of the exchange step */

/* The exchange step after the path-sum (every path's contribution is
 * added up; paths split across ranks need one sum over ranks). */
typedef enum {
  HSF_COLL_NONE = 0,           /* the run's partial result stays in `out` */
  HSF_COLL_ALLREDUCE = 1,      /* out <- sum over ranks of out (in place); bitstrings and
                                  small full outputs */
  HSF_COLL_REDUCE_SCATTER = 2  /* coll_out <- rank r's row shard [r R / G, (r+1) R / G) of the
                                  sum over ranks of out (R = the run's rows) */
} hsf_collective;

/* Fill *opts with the defaults listed above. */
hsf_status hsf_plan_opts_default(hsf_plan_opts* opts);

/*
 * hsf_plan — parse the circuit, classify gates, contract and schedule the
 * joint-cut blocks, Schmidt-decompose every cut unit (host fp64: assembly or
 * diagonal route, reshape Eq. 6, one-sided Jacobi SVD Eq. 7, truncation and
 * normalisation Eq. 8-9), count paths and build the per-half device
 * programs.  Host only: touches no GPU.
 *
 *   circuit_text, text_len : circuit file contents (format in DESIGN.md)
 *   n_low                  : qubits in half B; 1 <= n_low < n
 *   n_blocks               : number of joint blocks (0 => every crossing gate
 *                            is its own unit; -1 => automatic cascades: the
 *                            fewest groups of commuting diagonal two-qubit
 *                            crossing gates sharing one qubit (minimum vertex
 *                            cover), other crossing gates alone)
 *   block_offsets          : CSR offsets, length n_blocks+1 (may be NULL iff
 *                            n_blocks == 0)
 *   block_gate_ids         : gate indices (0-based, file order) of each block
 *   opts                   : NULL => defaults
 *   out                    : receives a new plan; free with hsf_plan_free
 * Inputs are copied; the caller keeps ownership.
 */
hsf_status hsf_plan(const char* circuit_text, size_t text_len, int32_t n_low, int64_t n_blocks,
                    const int64_t* block_offsets, const int64_t* block_gate_ids,
                    const hsf_plan_opts* opts, hsf_plan_t** out);

typedef struct {
  int32_t n_qubits, n_a, n_b;
  int32_t n_units;
  uint64_t n_paths;             /* joint-cut paths n_p^j (exact, <= budget) */
  double log2_n_paths_individual; /* log2 of n_p^t = prod of individual ranks */
  const int32_t* ranks;         /* [n_units] Schmidt ranks r_u (plan-owned) */
  const int32_t* support_a;     /* [n_units] |S_a| */
  const int32_t* support_b;     /* [n_units] |S_b| */
  const int64_t* sigma_offsets; /* [n_units+1] into sigmas */
  const double* sigmas;         /* kept singular values, descending per unit */
  int32_t levels_a, levels_b;   /* materialised path-tree levels per half */
  int32_t passes_a, passes_b;   /* device passes over all levels per half */
  int32_t ops_a, ops_b;         /* device ops after fusion */
  uint64_t plan_hash;           /* FNV-1a of the device program + tables */
  int32_t fold_units;           /* trailing diagonal units folded in bitstring runs (0 = none) */
  int32_t n_joint_blocks;       /* units holding more than one gate (the paper's "blocks";
                                   n_units - n_joint_blocks = its "separate cuts") */
  double tree_bytes_a, tree_bytes_b; /* state bytes the simulator tile passes read + write
                                   for all paths (full tree; roofline numerator) */
  double fold_tree_bytes_a, fold_tree_bytes_b; /* same for the folded tree (0 if none) */
  int32_t fold_passes_a, fold_passes_b;        /* device passes of the folded tree (0 if none) */
  int32_t tail_units_a, tail_units_b;          /* trailing units whose diagonal factors on that half
                                                  are applied in the full-output operand prep
                                                  (half-sided fold; 0 = none) */
  int32_t tail_passes_a, tail_passes_b;        /* device passes of that half's shortened tree
                                                  (head and tail folds) */
  double tail_tree_bytes_a, tail_tree_bytes_b; /* tree_bytes of the shortened trees (0 if none) */
  int32_t head_units_a, head_units_b;          /* leading units whose factors on that half act on
                                                  computational-basis qubits: scalars folded into
                                                  c_p in full-output tensor-core runs (head fold) */
  double tree_flops_a, tree_flops_b;           /* floating-point operations of the simulator passes
                                                  for all paths (FMA = 2; dense k-qubit op 8*2^k,
                                                  register-pass 1-qubit gate 16, diagonal 6 per
                                                  amplitude): the compute-roofline numerator */
  double fold_tree_flops_a, fold_tree_flops_b; /* same for the bitstring folded tree (0 if none) */
  double tail_tree_flops_a, tail_tree_flops_b; /* same for the half-sided fold trees (0 if none) */
  int32_t n_analytic_units;     /* units decomposed by the analytic cascade route */
  const int32_t* unit_analytic; /* [n_units] 1 if that unit's factors are closed-form */
  const int32_t* unit_sequential; /* [n_units] 1 if that unit's factors came from the sequential
                                     (MPO-style) route */
  int32_t whole_state_a, whole_state_b; /* 1: K1 tier -- each pass holds the whole half state in one
                                           CTA's shared memory (2^m <= 2^14 complex64 / 2^13
                                           complex128); 0: K2 tiles streamed through HBM/L2 */
} hsf_plan_info;

/* Pointers in *info stay valid until hsf_plan_free. */
hsf_status hsf_plan_info_get(const hsf_plan_t* plan, hsf_plan_info* info);

typedef struct {
  /* Bitstring mode: n_bitstrings > 0.  out receives n_bitstrings complex
   * amplitudes in input order (duplicates allowed).  Full mode: bitstrings ==
   * NULL and n_bitstrings == 0; out receives rows [row_begin,row_end) of the
   * [2^nA][2^nB] output, i.e. (row_end-row_begin) * 2^nB complex values. */
  const uint64_t* bitstrings;
  uint64_t n_bitstrings;
  int32_t bits_on_device;       /* 1 => device pointer, 0 => host pointer */
  void* out;                    /* caller-owned, plan dtype */
  int32_t out_on_device;        /* 1 => device pointer, 0 => host pointer: full-mode
                                   rows are computed in chunks of <= 16 MiB (env
                                   HSF_HOST_CHUNK_BYTES overrides) into two device
                                   staging buffers and copied back while the next
                                   chunk is computed (bounded device memory);
                                   pinned host memory gives overlapped copies */
  uint64_t path_begin, path_end;/* paths evaluated [begin,end); 0,0 => all.  The
                                   result is the partial sum over this range. */
  uint64_t row_begin, row_end;  /* full mode only; 0,0 => all 2^nA rows */
  void* cuda_stream;            /* cudaStream_t; NULL => legacy default stream */
  hsf_precision precision;
  int32_t device;               /* CUDA device ordinal; -1 => current */
  double* phase_ms;             /* optional [5], ms from CUDA events (synchronises):
                                   [0] start -> half-A leaves done (caller stream)
                                   [1] start -> half-B leaves done (side stream;
                                       the two path trees run concurrently)
                                   [2] operand prep after the later tree (K4)
                                   [3] core path-sum kernel (tcgen05 GEMM /
                                       SIMT GEMM / gather)
                                   [4] total */
  int32_t accumulate;           /* 1 => out += this run's result (device output only;
                                   e.g. path ranges run in chunks, or partial sums
                                   combined on one GPU); 0 => out is overwritten */
  /* Fused reduce-scatter (full output, tensor-core precisions, all rows):
   * n_out_shards in 1..8 device pointers, possibly another GPU's memory
   * (CUDA IPC / peer access); output rows [o*shard_rows, (o+1)*shard_rows)
   * are reduce-added (TMA .add, fp32 element-wise) into out_shards[o] by the
   * GEMM epilogue itself, tile by tile -- the K-split partial sums of several
   * ranks land in each owner's shard without a separate collective.
   * shard_rows * n_out_shards == 2^nA, shard_rows a multiple of 256.  The
   * caller zeroes the shards before the ranks' runs and synchronises after.
   * `out` is ignored; n_out_shards == 0 => normal output. */
  void* const* out_shards;
  int32_t n_out_shards;
  uint64_t shard_rows;
  /* Exchange step (device output only): with comm != NULL and coll !=
   * HSF_COLL_NONE, the sum over the communicator's ranks is enqueued on
   * cuda_stream right after the path-sum (captured into the run's CUDA graph
   * with it).  Every rank calls hsf_run with the same plan, collective,
   * output size and row range and its own path range.  The first run of a plan
   * on a communicator compares the ranks' plan hashes (HSF_ERR_PLAN_MISMATCH).
   * coll_out: REDUCE_SCATTER destination, device, (rows / nranks) * 2^nB
   * complex values (rows divisible by nranks); ignored otherwise. */
  hsf_comm_t* comm;
  hsf_collective coll;
  void* coll_out;
  /* 1 => out_shards[0] is the multicast address of an NVLS buffer
   * (hsf_mcast_bind) and n_out_shards == 1: a bitstring run's block gather
   * reduce-adds every sample with multimem.red into all ranks' copies (each
   * rank then holds the whole sum: a fused all-reduce).  Zero the buffers and
   * barrier before, barrier after, as for out_shards. */
  int32_t shards_multicast;
} hsf_run_args;

/* hsf_run — evaluate the paths [path_begin, path_end) on the GPU: path-tree
 * half-state simulation of both halves, coefficient fold
 * c_p = prod_u c_{u,d_u}, then the Kronecker path-sum
 * into `out`.  Enqueued on cuda_stream; returns after the stream work has
 * been enqueued if out_on_device, after completion otherwise.  The plan owns
 * its device tables and workspace (grown on demand, freed by hsf_plan_free). */
hsf_status hsf_run(hsf_plan_t* plan, const hsf_run_args* args);

/* What hsf_run does for these args (the launch sequence make_layout picks)
 * and the method's algorithmic work of each phase -- the numerators of the
 * rooflines bench.py reports.  Bytes count each operand / result element
 * once at its storage width; flops count FMA = 2. */
typedef enum {
  HSF_CORE_SIMT = 0,          /* K5s: CUDA-core complex GEMM (fp32 / fp64) */
  HSF_CORE_TC_PAIR = 1,       /* K5: tcgen05 CTA-pair GEMM (cta_group::2) */
  HSF_CORE_TC_SINGLE = 2,     /* K5: tcgen05 single-CTA GEMM (<= 128 rows) */
  HSF_CORE_TC_SWAPPED = 3,    /* K5w: narrow-N swapped GEMM + transpose (prefix outputs) */
  HSF_CORE_GATHER = 4,        /* K6: per-sample gather (both halves transposed) */
  HSF_CORE_BLOCK_GATHER = 5   /* K6b: block gather (one half read from its leaves) */
} hsf_core_kind;

typedef struct {
  int32_t core;               /* hsf_core_kind */
  int32_t direct_half;        /* block gather: half read from its leaves (0 A, 1 B); else -1 */
  int32_t tree_variant_a, tree_variant_b; /* 0 full tree, 1 bitstring fold, 2 half-sided fold */
  uint64_t K;                 /* columns of the path-sum (tree paths of the range) */
  uint64_t rows;              /* full output: rows of half A evaluated; bitstrings: samples */
  int32_t tc_products;        /* split-bf16 / tf32 products per real MMA (0 = SIMT / gather) */
  int32_t kernel_launches;    /* kernels of the run's captured CUDA graph (-1: the run is not
                                 graph-captured yet, or launches directly) */
  double sim_bytes[2], sim_flops[2];    /* per half: simulator passes over this range */
  double prep_bytes;          /* operand preparation (transposes / split-bf16 planes) */
  double core_bytes;          /* path-sum kernel: operands read once + result written */
  double core_flops_useful;   /* 8 K per output amplitude (complex multiply-add) */
  double core_flops_executed; /* tensor-core flops actually issued (split products, padding) */
  int32_t tleaf_half;         /* bitstring runs: the half whose last transition is a T-leaf pass
                                 (writes the gather operand rows directly), -1 none */
  int32_t tleaf_leaves;       /* its leaves per parent (2, 4 or 8) */
} hsf_run_desc;

hsf_status hsf_run_describe(const hsf_plan_t* plan, const hsf_run_args* args, hsf_run_desc* out);

/* Bytes of device workspace hsf_run would need for these args (0 on error). */
size_t hsf_workspace_bytes(const hsf_plan_t* plan, const hsf_run_args* args);

void hsf_plan_free(hsf_plan_t* plan);

const char* hsf_status_str(hsf_status s);

/* Copy the calling thread's last error message into buf (NUL-terminated,
 * truncated to len); returns the full message length. */
size_t hsf_last_error(char* buf, size_t len);

/* Debug/inspection: CUDA source of the specialised kernel of tile pass `pass`
 * (flattened over transitions) of half `half` (0 = A, 1 = B) of tree variant
 * `variant` (0 = full tree, 1 = bitstring trailing-diagonal fold, 2 = the
 * half-sided trailing fold of full-output runs; + 4·cb for the cluster tier
 * with 2^cb CTAs per tile; + 16·s for the store variant s: 1 = split-bf16 B
 * operand, 3 = the swapped path-sum's M operand; + 64: the T-leaf variant of
 * that tree's last transition, `pass` ignored).  Copies at most
 * len-1 bytes + NUL into buf (may be NULL) and returns the full length; 0 if
 * the pass does not exist.  Host only. */
size_t hsf_debug_pass_source(const hsf_plan_t* plan, int32_t variant, int32_t half, int32_t pass, char* buf,
                             size_t len);

/* CUDA IPC of fused reduce-scatter shards (plumbing for out_shards across
 * processes): hsf_ipc_export writes the 64-byte IPC handle of the allocation
 * holding dev_ptr and dev_ptr's offset in it; another process of the same
 * node maps it with hsf_ipc_import (peer access enabled lazily) and unmaps it
 * with hsf_ipc_release(ptr, offset).  The exporter keeps the allocation alive. */
hsf_status hsf_ipc_export(const void* dev_ptr, void* handle_out, uint64_t* offset_out);
hsf_status hsf_ipc_import(const void* handle, uint64_t offset, void** dev_ptr_out);
hsf_status hsf_ipc_release(void* dev_ptr, uint64_t offset);

/* NCCL communicator of the exchange step (one per rank and GPU).  Rank 0
 * calls hsf_comm_unique_id and sends the 128 bytes to every rank out of band
 * (e.g. torch.distributed); every rank then calls hsf_comm_create with its
 * rank (collective: blocks until all ranks joined).  device: CUDA ordinal, -1
 * = current.  NCCL is loaded at run time (libnccl.so.2; HSF_ERR_NCCL if
 * absent).  Free after the last run that uses it. */
hsf_status hsf_comm_unique_id(void* id_out128);
hsf_status hsf_comm_create(const void* id128, int32_t nranks, int32_t rank, int32_t device, hsf_comm_t** out);
void hsf_comm_free(hsf_comm_t* comm);

/* NVLink SHARP multicast buffers (the fused all-reduce of bitstring runs,
 * hsf_run_args.shards_multicast).  Collective set-up, every rank in order:
 * rank 0 hsf_mcast_create (returns a 64-byte fabric handle, sent to the other
 * ranks out of band), the others hsf_mcast_import(handle); every rank
 * hsf_mcast_add_device; barrier; every rank hsf_mcast_bind (allocates `bytes`
 * on its device, binds it, maps the local and the multicast address, zeroes
 * it); barrier.  HSF_ERR_UNSUPPORTED without multicast support (no NVSwitch /
 * fabric).  hsf_mcast_free unmaps and releases (after every rank's last use). */
typedef struct hsf_mcast_s hsf_mcast_t;
hsf_status hsf_mcast_create(size_t bytes, int32_t nranks, int32_t device, void* handle_out64, hsf_mcast_t** out);
hsf_status hsf_mcast_import(const void* handle64, size_t bytes, int32_t nranks, int32_t device, hsf_mcast_t** out);
hsf_status hsf_mcast_add_device(hsf_mcast_t* m);
hsf_status hsf_mcast_bind(hsf_mcast_t* m, void** local_out, void** multicast_out);
void hsf_mcast_free(hsf_mcast_t* m);

/* Library build identification string (compile flags, arch). */
const char* hsf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HSF_H_ */
