"""Thin ctypes binding of libhsf.so (include/hsf.h).  Argument marshalling only:
every step of the HSF path runs in the library's CUDA kernels.  There is no
CPU fallback: if the library or a GPU is missing, calls raise.

PyTorch is used only for device memory and streams (``torch.Tensor`` data
pointers, ``torch.cuda.current_stream()``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# HSF_DEBUG_LIB=1 loads the debug build (bounded mbarrier waits that trap;
# build.build(debug=True))
LIB_PATH = os.path.join(_HERE, "lib", "libhsf_debug.so" if os.environ.get("HSF_DEBUG_LIB") == "1" else "libhsf.so")

HSF_C64, HSF_C128 = 0, 1
PREC = {"auto": 0, "simt": 1, "bf16x3": 2, "bf16x1": 3, "bf16x6": 4, "tf32x3": 5}
STATUS = {}


class HsfError(RuntimeError):
    def __init__(self, status: int, name: str, msg: str):
        super().__init__(f"{name}: {msg}")
        self.status = status
        self.name = name


class _Opts(C.Structure):
    _fields_ = [("dtype", C.c_int), ("svd_rel_tol", C.c_double), ("max_dense_block_qubits", C.c_int32),
                ("log2_path_budget", C.c_double), ("individual", C.c_int32), ("tile_qubits", C.c_int32),
                ("fuse_gates", C.c_int32), ("hoist_gates", C.c_int32), ("fold_trailing_diag", C.c_int32),
                ("jit", C.c_int32), ("partition_b", C.c_uint64),
                ("graphs", C.c_int32), ("analytic_cascades", C.c_int32), ("smem_tier", C.c_int32),
                ("block_route", C.c_int32)]


class _Info(C.Structure):
    _fields_ = [("n_qubits", C.c_int32), ("n_a", C.c_int32), ("n_b", C.c_int32), ("n_units", C.c_int32),
                ("n_paths", C.c_uint64), ("log2_n_paths_individual", C.c_double),
                ("ranks", C.POINTER(C.c_int32)), ("support_a", C.POINTER(C.c_int32)),
                ("support_b", C.POINTER(C.c_int32)), ("sigma_offsets", C.POINTER(C.c_int64)),
                ("sigmas", C.POINTER(C.c_double)), ("levels_a", C.c_int32), ("levels_b", C.c_int32),
                ("passes_a", C.c_int32), ("passes_b", C.c_int32), ("ops_a", C.c_int32), ("ops_b", C.c_int32),
                ("plan_hash", C.c_uint64), ("fold_units", C.c_int32),
                ("n_joint_blocks", C.c_int32), ("tree_bytes_a", C.c_double), ("tree_bytes_b", C.c_double),
                ("fold_tree_bytes_a", C.c_double), ("fold_tree_bytes_b", C.c_double),
                ("fold_passes_a", C.c_int32), ("fold_passes_b", C.c_int32),
                ("tail_units_a", C.c_int32), ("tail_units_b", C.c_int32),
                ("tail_passes_a", C.c_int32), ("tail_passes_b", C.c_int32),
                ("tail_tree_bytes_a", C.c_double), ("tail_tree_bytes_b", C.c_double),
                ("head_units_a", C.c_int32), ("head_units_b", C.c_int32),
                ("tree_flops_a", C.c_double), ("tree_flops_b", C.c_double),
                ("fold_tree_flops_a", C.c_double), ("fold_tree_flops_b", C.c_double),
                ("tail_tree_flops_a", C.c_double), ("tail_tree_flops_b", C.c_double),
                ("n_analytic_units", C.c_int32), ("unit_analytic", C.POINTER(C.c_int32)),
                ("unit_sequential", C.POINTER(C.c_int32)),
                ("whole_state_a", C.c_int32), ("whole_state_b", C.c_int32)]


class _RunArgs(C.Structure):
    _fields_ = [("bitstrings", C.c_void_p), ("n_bitstrings", C.c_uint64), ("bits_on_device", C.c_int32),
                ("out", C.c_void_p), ("out_on_device", C.c_int32), ("path_begin", C.c_uint64),
                ("path_end", C.c_uint64), ("row_begin", C.c_uint64), ("row_end", C.c_uint64),
                ("cuda_stream", C.c_void_p), ("precision", C.c_int), ("device", C.c_int32),
                ("phase_ms", C.POINTER(C.c_double)), ("accumulate", C.c_int32),
                ("out_shards", C.POINTER(C.c_void_p)), ("n_out_shards", C.c_int32), ("shard_rows", C.c_uint64),
                ("comm", C.c_void_p), ("coll", C.c_int), ("coll_out", C.c_void_p), ("shards_multicast", C.c_int32)]

COLL = {None: 0, "none": 0, "allreduce": 1, "reduce_scatter": 2}


class _RunDesc(C.Structure):
    _fields_ = [("core", C.c_int32), ("direct_half", C.c_int32), ("tree_variant_a", C.c_int32),
                ("tree_variant_b", C.c_int32), ("K", C.c_uint64), ("rows", C.c_uint64), ("tc_products", C.c_int32),
                ("kernel_launches", C.c_int32), ("sim_bytes", C.c_double * 2), ("sim_flops", C.c_double * 2),
                ("prep_bytes", C.c_double), ("core_bytes", C.c_double), ("core_flops_useful", C.c_double),
                ("core_flops_executed", C.c_double), ("tleaf_half", C.c_int32), ("tleaf_leaves", C.c_int32)]


CORE_KINDS = ["simt", "tc_pair", "tc_single", "tc_swapped", "gather", "block_gather"]

_lib = None

EXPORTS = ["hsf_plan_opts_default", "hsf_plan", "hsf_plan_info_get", "hsf_run", "hsf_workspace_bytes",
           "hsf_plan_free", "hsf_status_str", "hsf_last_error", "hsf_version", "hsf_debug_pass_source",
           "hsf_ipc_export", "hsf_ipc_import", "hsf_ipc_release", "hsf_run_describe", "hsf_comm_unique_id",
           "hsf_comm_create", "hsf_comm_free", "hsf_mcast_create", "hsf_mcast_import", "hsf_mcast_add_device",
           "hsf_mcast_bind", "hsf_mcast_free"]


def lib():
    """Load libhsf.so (built in-tree by paper_2502_06959_b200/build.py)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libhsf.so not built ({LIB_PATH}); run `python -m paper_2502_06959_b200.build`")
    L = C.CDLL(LIB_PATH)
    L.hsf_plan_opts_default.argtypes = [C.POINTER(_Opts)]
    L.hsf_plan.argtypes = [C.c_char_p, C.c_size_t, C.c_int32, C.c_int64, C.POINTER(C.c_int64),
                           C.POINTER(C.c_int64), C.POINTER(_Opts), C.POINTER(C.c_void_p)]
    L.hsf_plan_info_get.argtypes = [C.c_void_p, C.POINTER(_Info)]
    L.hsf_run.argtypes = [C.c_void_p, C.POINTER(_RunArgs)]
    L.hsf_workspace_bytes.argtypes = [C.c_void_p, C.POINTER(_RunArgs)]
    L.hsf_run_describe.argtypes = [C.c_void_p, C.POINTER(_RunArgs), C.POINTER(_RunDesc)]
    L.hsf_comm_unique_id.argtypes = [C.c_void_p]
    L.hsf_comm_create.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]
    L.hsf_comm_free.argtypes = [C.c_void_p]
    L.hsf_comm_free.restype = None
    L.hsf_mcast_create.argtypes = [C.c_size_t, C.c_int32, C.c_int32, C.c_void_p, C.POINTER(C.c_void_p)]
    L.hsf_mcast_import.argtypes = [C.c_void_p, C.c_size_t, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]
    L.hsf_mcast_add_device.argtypes = [C.c_void_p]
    L.hsf_mcast_bind.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]
    L.hsf_mcast_free.argtypes = [C.c_void_p]
    L.hsf_mcast_free.restype = None
    L.hsf_workspace_bytes.restype = C.c_size_t
    L.hsf_plan_free.argtypes = [C.c_void_p]
    L.hsf_plan_free.restype = None
    L.hsf_status_str.argtypes = [C.c_int]
    L.hsf_status_str.restype = C.c_char_p
    L.hsf_last_error.argtypes = [C.c_char_p, C.c_size_t]
    L.hsf_last_error.restype = C.c_size_t
    L.hsf_version.restype = C.c_char_p
    L.hsf_debug_pass_source.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_char_p, C.c_size_t]
    L.hsf_debug_pass_source.restype = C.c_size_t
    L.hsf_ipc_export.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64)]
    L.hsf_ipc_import.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_void_p)]
    L.hsf_ipc_release.argtypes = [C.c_void_p, C.c_uint64]
    for f in ("hsf_plan_opts_default", "hsf_plan", "hsf_plan_info_get", "hsf_run", "hsf_ipc_export", "hsf_ipc_import",
              "hsf_ipc_release", "hsf_run_describe", "hsf_comm_unique_id", "hsf_comm_create", "hsf_mcast_create",
              "hsf_mcast_import", "hsf_mcast_add_device", "hsf_mcast_bind"):
        getattr(L, f).restype = C.c_int
    _lib = L
    return L


def _check(st: int):
    if st != 0:
        L = lib()
        buf = C.create_string_buffer(4096)
        L.hsf_last_error(buf, 4096)
        raise HsfError(st, L.hsf_status_str(st).decode(), buf.value.decode(errors="replace"))


def ipc_export(t) -> tuple:
    """CUDA IPC handle (64 bytes) + offset of a device tensor's memory (hsf_ipc_export)."""
    h = (C.c_char * 64)()
    off = C.c_uint64()
    _check(lib().hsf_ipc_export(C.c_void_p(t.data_ptr()), h, C.byref(off)))
    return bytes(h), int(off.value)


def ipc_import(handle: bytes, offset: int) -> int:
    """Device pointer to another process's exported memory (hsf_ipc_import)."""
    p = C.c_void_p()
    hb = C.create_string_buffer(bytes(handle), 64)
    _check(lib().hsf_ipc_import(hb, C.c_uint64(offset), C.byref(p)))
    return int(p.value)


def ipc_release(ptr: int, offset: int) -> None:
    _check(lib().hsf_ipc_release(C.c_void_p(ptr), C.c_uint64(offset)))


class Comm:
    """hsf_comm_create(): the library's NCCL communicator for the exchange step
    (one per rank).  `unique_id()` on rank 0, broadcast the 128 bytes, then
    every rank constructs Comm(uid, nranks, rank)."""

    @staticmethod
    def unique_id() -> bytes:
        b = (C.c_char * 128)()
        _check(lib().hsf_comm_unique_id(b))
        return bytes(b)

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int = -1):
        h = C.c_void_p()
        ub = C.create_string_buffer(bytes(uid), 128)
        _check(lib().hsf_comm_create(ub, nranks, rank, device, C.byref(h)))
        self._h = h
        self.nranks, self.rank = nranks, rank

    @property
    def handle(self):
        return self._h.value

    def close(self):
        if self._h is not None and self._h.value and _lib is not None:
            _lib.hsf_comm_free(self._h)
        self._h = None

    def __del__(self):
        self.close()


class Multicast:
    """NVLS multicast buffer (hsf_mcast_*): `create` on rank 0 returns the
    64-byte fabric handle, `import_` on the other ranks; then every rank
    add_device(), a barrier, bind() (-> local and multicast addresses), a
    barrier.  dist.MulticastBuffer drives the sequence over torch.distributed."""

    def __init__(self, nbytes: int, nranks: int, device: int = -1, handle: bytes | None = None):
        h = C.c_void_p()
        self.nbytes = nbytes
        if handle is None:
            hb = (C.c_char * 64)()
            _check(lib().hsf_mcast_create(nbytes, nranks, device, hb, C.byref(h)))
            self.handle = bytes(hb)
        else:
            _check(lib().hsf_mcast_import(C.create_string_buffer(bytes(handle), 64), nbytes, nranks, device,
                                          C.byref(h)))
            self.handle = bytes(handle)
        self._h = h
        self.local = self.multicast = None

    def add_device(self):
        _check(lib().hsf_mcast_add_device(self._h))

    def bind(self):
        lo, mc = C.c_void_p(), C.c_void_p()
        _check(lib().hsf_mcast_bind(self._h, C.byref(lo), C.byref(mc)))
        self.local, self.multicast = int(lo.value), int(mc.value)
        return self.local, self.multicast

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value and _lib is not None:
            _lib.hsf_mcast_free(self._h)
        self._h = None

    def __del__(self):
        self.close()


def version() -> str:
    return lib().hsf_version().decode()


class Plan:
    """hsf_plan(): host-side joint-cut plan.  `n_low` is the size
    of half B = qubits [0, n_low), or a list of the qubits forming half B (any
    partition; relabelled internally, results in the caller's order).  `blocks` is a list of
    gate-index lists, or "auto" (automatic cascades of commuting diagonal
    crossing gates); `individual=True` cuts every crossing gate alone."""

    def __init__(self, circuit_text: str, n_low: int, blocks=None, dtype: str = "c64", individual: bool = False,
                 svd_rel_tol: float = 1e-12, tile_qubits: int = 0, fuse_gates: bool = True,
                 log2_path_budget: float = 26.0, max_dense_block_qubits: int = 10, hoist_gates: bool = True,
                 fold_trailing_diag: bool = True, jit: bool = True, graphs: bool = True,
                 analytic_cascades: bool = True, smem_tier: int = 0, block_route: int = 0):
        L = lib()
        o = _Opts()
        _check(L.hsf_plan_opts_default(C.byref(o)))
        if isinstance(n_low, (list, tuple, set, frozenset)):  # half B = these qubits (any subset)
            qs = sorted(set(int(q) for q in n_low))
            o.partition_b = sum(1 << q for q in qs)
            n_low = len(qs)
        o.dtype = HSF_C64 if dtype == "c64" else HSF_C128
        o.svd_rel_tol = svd_rel_tol
        o.individual = int(individual)
        o.tile_qubits = tile_qubits
        o.fuse_gates = int(fuse_gates)
        o.hoist_gates = int(hoist_gates)
        o.fold_trailing_diag = int(fold_trailing_diag)
        o.jit = int(jit)
        o.graphs = int(graphs)
        o.analytic_cascades = int(analytic_cascades)
        o.smem_tier = int(smem_tier)
        o.block_route = int(block_route)
        o.log2_path_budget = log2_path_budget
        o.max_dense_block_qubits = max_dense_block_qubits
        auto = isinstance(blocks, str)
        if auto and blocks != "auto":
            raise ValueError("blocks must be a list of gate-index lists or 'auto'")
        blocks = [] if auto else (blocks or [])
        offs = np.zeros(len(blocks) + 1, dtype=np.int64)
        for i, b in enumerate(blocks):
            offs[i + 1] = offs[i] + len(b)
        ids = np.array([g for b in blocks for g in b] or [0], dtype=np.int64)
        txt = circuit_text.encode()
        h = C.c_void_p()
        _check(L.hsf_plan(txt, len(txt), n_low, -1 if auto else len(blocks), offs.ctypes.data_as(C.POINTER(C.c_int64)),
                          ids.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(o), C.byref(h)))
        self._h = h
        self.dtype = dtype
        self._info = _Info()
        _check(L.hsf_plan_info_get(self._h, C.byref(self._info)))
        i = self._info
        self.n, self.n_a, self.n_b = i.n_qubits, i.n_a, i.n_b
        self.n_paths = int(i.n_paths)
        self.ranks = [i.ranks[u] for u in range(i.n_units)]
        self.log2_n_paths_individual = i.log2_n_paths_individual
        self.sigmas = [[i.sigmas[j] for j in range(i.sigma_offsets[u], i.sigma_offsets[u + 1])]
                       for u in range(i.n_units)]
        self.support = [(i.support_a[u], i.support_b[u]) for u in range(i.n_units)]
        self.levels = (i.levels_a, i.levels_b)
        self.passes = (i.passes_a, i.passes_b)
        self.ops = (i.ops_a, i.ops_b)
        self.plan_hash = int(i.plan_hash)
        self.fold_units = int(i.fold_units)
        self.n_joint_blocks = int(i.n_joint_blocks)
        self.n_units = int(i.n_units)
        self.tree_bytes = (float(i.tree_bytes_a), float(i.tree_bytes_b))
        self.fold_tree_bytes = (float(i.fold_tree_bytes_a), float(i.fold_tree_bytes_b))
        self.fold_passes = (int(i.fold_passes_a), int(i.fold_passes_b))
        self.tail_units = (int(i.tail_units_a), int(i.tail_units_b))
        self.tail_passes = (int(i.tail_passes_a), int(i.tail_passes_b))
        self.tail_tree_bytes = (float(i.tail_tree_bytes_a), float(i.tail_tree_bytes_b))
        self.head_units = (int(i.head_units_a), int(i.head_units_b))
        self.tree_flops = (float(i.tree_flops_a), float(i.tree_flops_b))
        self.fold_tree_flops = (float(i.fold_tree_flops_a), float(i.fold_tree_flops_b))
        self.tail_tree_flops = (float(i.tail_tree_flops_a), float(i.tail_tree_flops_b))
        self.n_analytic_units = int(i.n_analytic_units)
        self.unit_analytic = [bool(i.unit_analytic[u]) for u in range(i.n_units)]
        self.unit_sequential = [bool(i.unit_sequential[u]) for u in range(i.n_units)]
        self.whole_state = (bool(i.whole_state_a), bool(i.whole_state_b))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.hsf_plan_free(h)
            self._h = None

    # -------------------------------------------------------------- run
    def _args(self, out_ptr, out_dev, bits_ptr, n_bits, bits_dev, path_range, row_range, precision, stream, device,
              phase, accumulate=False):
        a = _RunArgs()
        a.bitstrings = bits_ptr
        a.n_bitstrings = n_bits
        a.bits_on_device = int(bits_dev)
        a.out = out_ptr
        a.out_on_device = int(out_dev)
        a.path_begin, a.path_end = path_range if path_range else (0, 0)
        a.row_begin, a.row_end = row_range if row_range else (0, 0)
        a.cuda_stream = stream
        a.precision = PREC[precision]
        a.device = device
        a.phase_ms = phase
        a.accumulate = int(accumulate)
        return a

    def run(self, out, bitstrings=None, path_range=None, row_range=None, precision: str = "auto", stream=None,
            timings: bool = False, accumulate: bool = False, out_shards=None, comm=None, coll=None,
            coll_out=None, multicast=None):
        """hsf_run(): evaluate paths [path_range) into `out`.

        `out` / `bitstrings` are torch tensors (device or host) or numpy arrays
        (host).  Returns per-phase ms [simA, simB, prep, core, total] if `timings`.

        out_shards: fused exchange (hsf.h) -- a list of 1..8 destinations,
        each a device tensor or an int device pointer (e.g. another GPU's
        buffer opened via CUDA IPC).  Full output: 2^nA / len(out_shards)
        rows each, the GEMM epilogue reduce-adds each row shard into its
        owner.  Bitstrings: ceil(n / len(out_shards)) samples each, the block
        gather reduce-adds each sample into its owner.  `out` may be None.

        multicast: an NVLS multicast address (Multicast.bind()): a bitstring
        run's block gather reduce-adds every sample into all ranks' copies
        (multimem.red; the fused all-reduce).  `out` may be None.

        comm / coll / coll_out: the exchange step inside the run (hsf.h):
        coll = "allreduce" (out summed over the communicator's ranks in place)
        or "reduce_scatter" (this rank's row shard of the sum into coll_out)."""
        import torch

        keep = []  # host arrays converted here stay alive until hsf_run returns
        cdt = {"c64": (torch.complex64, np.complex64), "c128": (torch.complex128, np.complex128)}[self.dtype]

        def ptr(x, kind):
            if isinstance(x, torch.Tensor):
                if not x.is_contiguous():
                    raise ValueError(f"{kind} tensor must be contiguous")
                if kind == "out" and x.dtype != cdt[0]:
                    raise TypeError(f"out must be {cdt[0]} for a {self.dtype} plan, got {x.dtype}")
                if kind == "bitstrings" and x.dtype not in (torch.int64, torch.uint64):
                    raise TypeError(f"bitstrings must be int64 / uint64, got {x.dtype}")
                if x.is_cuda and torch.cuda.is_available() and x.device.index != dev:
                    raise ValueError(f"{kind} is on {x.device}, the run on cuda:{dev}")
                return x.data_ptr(), x.is_cuda, x.numel()
            if not isinstance(x, np.ndarray):
                raise TypeError(f"{kind} must be a torch tensor or a numpy array")
            if kind == "out":
                if x.dtype != cdt[1]:
                    raise TypeError(f"out must be {np.dtype(cdt[1])} for a {self.dtype} plan, got {x.dtype}")
                if not x.flags.c_contiguous or not x.flags.writeable:
                    raise ValueError("out must be a writeable C-contiguous array")
            else:
                if x.dtype not in (np.int64, np.uint64):
                    raise TypeError(f"bitstrings must be int64 / uint64, got {x.dtype}")
                x = np.ascontiguousarray(x)
                keep.append(x)
            return x.ctypes.data, False, x.size

        dev = torch.cuda.current_device() if torch.cuda.is_available() else -1
        if path_range is not None and int(path_range[0]) == int(path_range[1]):
            # hsf_run reads (0, 0) as "all paths": an empty range must not reach it
            raise ValueError(f"empty path_range {path_range}")
        shards_arr = None
        if multicast is not None:
            out_shards = [int(multicast)]
        if out_shards:
            ps = [s if isinstance(s, int) else s.data_ptr() for s in out_shards]
            shards_arr = (C.c_void_p * len(ps))(*ps)
            op, odev = None, True
        else:
            if out is None:
                raise ValueError("out is None")
            op, odev, n_out = ptr(out, "out")
        bp, bdev, nb = (None, False, 0) if bitstrings is None else ptr(bitstrings, "bitstrings")
        if not out_shards:
            if bitstrings is not None:
                need = nb
            else:
                r0, r1 = row_range if row_range else (0, 1 << self.n_a)
                need = (r1 - r0) << self.n_b
            if n_out < need:
                raise ValueError(f"out holds {n_out} amplitudes, the run writes {need}")
        st = stream if stream is not None else (torch.cuda.current_stream().cuda_stream if torch.cuda.is_available() else None)
        phase = (C.c_double * 5)() if timings else None
        a = self._args(op, odev, bp, nb, bdev, path_range, row_range, precision, st, dev,
                       C.cast(phase, C.POINTER(C.c_double)) if timings else None, accumulate)
        if shards_arr is not None:
            a.out_shards = C.cast(shards_arr, C.POINTER(C.c_void_p))
            a.n_out_shards = len(out_shards)
            # full output: rows of half A per shard; bitstrings: samples per shard
            a.shard_rows = (-(-nb // len(out_shards)) if bitstrings is not None
                            else (1 << self.n_a) // len(out_shards))
            a.shards_multicast = int(multicast is not None)
        if coll not in COLL:
            raise ValueError(f"unknown collective {coll!r}")
        if COLL[coll]:
            if comm is None:
                raise ValueError("a collective needs comm=")
            a.comm = comm.handle
            a.coll = COLL[coll]
            if coll == "reduce_scatter":
                if coll_out is None:
                    raise ValueError("reduce_scatter needs coll_out")
                cp_, cdev, cn = ptr(coll_out, "out")
                if not cdev or cn * comm.nranks != n_out:
                    raise ValueError("coll_out must be a device tensor of out.numel() / nranks values")
                a.coll_out = cp_
        _check(lib().hsf_run(self._h, C.byref(a)))
        return list(phase) if timings else None

    def pass_source(self, half: int, pass_index: int, variant: int = 0) -> str | None:
        """CUDA source of one specialised simulator pass kernel (inspection)."""
        L = lib()
        n = L.hsf_debug_pass_source(self._h, variant, half, pass_index, None, 0)
        if not n:
            return None
        buf = C.create_string_buffer(n + 1)
        L.hsf_debug_pass_source(self._h, variant, half, pass_index, buf, n + 1)
        return buf.value.decode()

    def describe(self, bitstrings_count: int = 0, path_range=None, row_range=None, precision="auto") -> dict:
        """hsf_run_describe(): the launch sequence and algorithmic work of a run
        with these arguments (after a run with the same arguments,
        `kernel_launches` counts the kernels of its captured graph)."""
        a = self._args(1, True, 1 if bitstrings_count else None, bitstrings_count, True, path_range, row_range,
                       precision, None, -1, None)
        d = _RunDesc()
        _check(lib().hsf_run_describe(self._h, C.byref(a), C.byref(d)))
        return {"core": CORE_KINDS[d.core], "direct_half": d.direct_half,
                "tree_variant": (d.tree_variant_a, d.tree_variant_b), "K": int(d.K), "rows": int(d.rows),
                "tc_products": d.tc_products, "kernel_launches": d.kernel_launches,
                "sim_bytes": tuple(d.sim_bytes), "sim_flops": tuple(d.sim_flops), "prep_bytes": d.prep_bytes,
                "core_bytes": d.core_bytes, "core_flops_useful": d.core_flops_useful,
                "core_flops_executed": d.core_flops_executed, "tleaf_half": d.tleaf_half,
                "tleaf_leaves": d.tleaf_leaves}

    def workspace_bytes(self, bitstrings_count: int = 0, path_range=None, row_range=None, precision="auto") -> int:
        a = self._args(1, True, 1 if bitstrings_count else None, bitstrings_count, True, path_range, row_range,
                       precision, None, -1, None)
        return int(lib().hsf_workspace_bytes(self._h, C.byref(a)))
