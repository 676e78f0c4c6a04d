"""Multi-GPU partition of the HSF path evaluation (DESIGN.md
"Multi-GPU").  One process per GPU; torch.distributed (NCCL on the box, gloo
in the CPU tests) is plumbing only: it carries the single exchange step the
method has -- the sum over paths of the partial amplitude vectors (P:109,
"adding up all contributions") -- or nothing at all when the output is
row-sharded.

Modes (`mode`):
  "allreduce"       paths split in contiguous ranges (whole subtrees); every
                    rank evaluates its range into a full-size partial output,
                    then one all-reduce(sum).  Bitstring runs (c3, c5), tiny
                    full runs (c1).
  "reduce_scatter"  paths split; full-size partial output; one
                    reduce-scatter(sum): rank r keeps rows
                    [r*2^nA/G, (r+1)*2^nA/G) of the [2^nA][2^nB] output.  The
                    literal BASELINE.json c4 reading; K-split c2.
  "rows"            every rank evaluates ALL paths but writes only its row
                    shard (rows as above) -- no collective on the data path.
                    The recommended c4 mode.
  "fused_bits"      bitstring runs: paths split as in allreduce, no partial
                    vector and no collective call: the block gather reduce-adds
                    (vector red.add) each sample's partial amplitude straight
                    into its owner's shard over peer memory; rank r holds
                    samples [r L, (r+1) L), L = ceil(n / G).
  "nvls_bits"       bitstring runs: paths split as in allreduce; the block
                    gather reduce-adds each sample with multimem.red through an
                    NVLS multicast buffer (MulticastBuffer), so the NVSwitch
                    sums the ranks' contributions into every rank's copy: a
                    fused all-reduce, no collective call.
  "fused_rs"        paths split as in reduce_scatter, but there is no partial
                    output and no collective call: every rank's GEMM epilogue
                    reduce-adds (TMA .add) each output tile straight into the
                    owner rank's row shard over peer memory (CUDA IPC,
                    NVLink on the box) -- the GEMM -> reduce-scatter of
                    SURVEY.md §8(f) row 3 as one kernel.  Full-output
                    tensor-core runs; 2^nA / G a multiple of 256 rows.

The per-rank evaluation is a callable `partial(path_range, row_range, out)`
so the partition and collective logic can be exercised on CPU with gloo
(tests/test_dist_gloo.py); on the GPU it is `Plan.run` (see `run_sharded`).
"""
from __future__ import annotations

from dataclasses import dataclass

MODES = ("allreduce", "reduce_scatter", "rows", "fused_rs", "fused_bits", "nvls_bits")


@dataclass(frozen=True)
class Shard:
    mode: str
    path_range: tuple      # paths this rank evaluates [p0, p1)
    row_range: tuple | None  # rows this rank's kernel writes (None => all rows / bitstrings)
    out_rows: tuple | None   # rows this rank holds after the collective (None => everything)


def path_range_for_rank(n_paths: int, rank: int, world: int):
    """Contiguous range of the linear (mixed-radix, last unit fastest) path
    index: whole subtrees of the path tree when `world` divides the leading
    radices (true for c1..c5 at 1/2/4/8).  Empty (p0 == p1) for some ranks
    when world > n_paths; `sharded_step` then skips the evaluation."""
    return (n_paths * rank // world, n_paths * (rank + 1) // world)


def bits_shard_len(n_samples: int, world: int) -> int:
    """Samples per owner shard of the fused bitstring exchange."""
    return -(-n_samples // world)


def row_range_for_rank(n_a: int, rank: int, world: int):
    rows = 1 << n_a
    return (rows * rank // world, rows * (rank + 1) // world)


def default_mode(full_output: bool, n_paths: int, n_a: int, n_b: int, world: int) -> str:
    """Cheapest exchange for the run: bitstrings and
    small outputs all-reduce; a full output whose partial vectors are large
    relative to the leaves (K small) is row-sharded; otherwise reduce-scatter."""
    if not full_output:
        return "allreduce"
    if world == 1:
        return "rows"
    out_bytes = 8 << (n_a + n_b)
    leaf_bytes = 8 * n_paths * ((1 << n_a) + (1 << n_b))
    if out_bytes > 64 * leaf_bytes or (1 << n_a) < world:
        return "rows" if (1 << n_a) >= world else "allreduce"
    return "reduce_scatter"


def make_shard(mode: str, n_paths: int, n_a: int, rank: int, world: int, full_output: bool) -> Shard:
    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r}")
    if not full_output and mode not in ("allreduce", "fused_bits", "nvls_bits"):
        raise ValueError("bitstring runs use mode='allreduce', 'fused_bits' or 'nvls_bits'")
    if full_output and mode in ("fused_bits", "nvls_bits"):
        raise ValueError(f"{mode} is for bitstring runs")
    if mode in ("reduce_scatter", "rows", "fused_rs") and (1 << n_a) % world:
        raise ValueError("row sharding needs world to divide 2^n_A")
    pr = path_range_for_rank(n_paths, rank, world)
    if mode in ("allreduce", "fused_bits", "nvls_bits"):  # fused_bits: out_rows = the caller's sample slice
        return Shard(mode, pr, None, None)
    rr = row_range_for_rank(n_a, rank, world)
    if mode in ("reduce_scatter", "fused_rs"):
        return Shard(mode, pr, None, rr)
    return Shard(mode, (0, n_paths), rr, rr)


class PeerShards:
    """Every rank's row shard, mapped into this process (fused_rs mode):
    `ptrs[r]` is rank r's shard (CUDA IPC import; this rank's own pointer for
    itself).  The handles travel through torch.distributed (any backend)."""

    def __init__(self, shard_out, group=None):
        import torch.distributed as dist
        from . import hsf as H
        self.local = shard_out
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        mine = H.ipc_export(shard_out) if world > 1 else None
        allh = [None] * world
        if world > 1:
            dist.all_gather_object(allh, mine, group=group)
        self.ptrs, self._opened = [], []
        for r in range(world):
            if r == rank:
                self.ptrs.append(shard_out.data_ptr())
            else:
                p = H.ipc_import(allh[r][0], allh[r][1])
                self.ptrs.append(p)
                self._opened.append((p, allh[r][1]))

    def close(self):
        from . import hsf as H
        for p, off in self._opened:
            H.ipc_release(p, off)
        self._opened = []


class MulticastBuffer:
    """An NVLS multicast buffer of `n` complex64 values on every rank of the
    group (hsf_mcast_*), set up collectively over torch.distributed: rank 0
    creates the multicast object and broadcasts its fabric handle, every rank
    adds its device, binds its memory.  `local` is this rank's copy (a torch
    view of it), `ptrs = [multicast address]` goes to Plan.run(multicast=...)."""

    def __init__(self, n: int, group=None):
        import torch
        import torch.distributed as dist
        from . import hsf as H
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        dev = torch.cuda.current_device()
        nbytes = 8 * n
        if rank == 0:
            self.m = H.Multicast(nbytes, world, dev)
            obj = [self.m.handle]
        else:
            obj = [None]
        if world > 1:
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
            if rank != 0:
                self.m = H.Multicast(nbytes, world, dev, handle=obj[0])
        self.m.add_device()
        if world > 1:
            dist.barrier(group=group)
        lo, mc = self.m.bind()
        if world > 1:
            dist.barrier(group=group)
        self.n = n
        self.mc = mc
        self.local = _tensor_at(lo, n, dev)

    def close(self):
        self.m.close()


def _tensor_at(ptr: int, n: int, dev: int):
    """A complex64 torch tensor over n values at device pointer `ptr` (not owned)."""
    import torch

    class _Arr:
        __cuda_array_interface__ = {"shape": (2 * n,), "typestr": "<f4", "data": (ptr, False), "version": 3}
    return torch.as_tensor(_Arr(), device=f"cuda:{dev}").view(torch.complex64)


def sharded_step(shard: Shard, partial, out, shard_out=None, group=None):
    """One rank's step: evaluate, then the mode's collective.

    out       : full-size output buffer (allreduce / reduce_scatter), the
                row shard itself (rows mode), or a PeerShards (fused_rs)
    shard_out : reduce_scatter destination (rows shard)
    Returns the tensor holding this rank's result."""
    import torch
    import torch.distributed as dist

    if shard.mode in ("fused_rs", "fused_bits", "nvls_bits"):
        # zero the own shard, all ranks' adds land in it, then everyone waits
        sync = torch.cuda.synchronize if out.local.is_cuda else (lambda: None)
        out.local.zero_()
        if dist.is_initialized():
            sync()
            dist.barrier(group=group)
        if shard.path_range[0] < shard.path_range[1]:
            partial(shard.path_range, None, out)
        sync()
        if dist.is_initialized():
            dist.barrier(group=group)
        return out.local
    if shard.path_range[0] < shard.path_range[1]:
        partial(shard.path_range, shard.row_range, out)
    else:  # more ranks than paths: this rank contributes nothing to the sum
        out.zero_()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1 or shard.mode == "rows":
        return out
    if shard.mode == "allreduce":
        dist.all_reduce(torch.view_as_real(out), op=dist.ReduceOp.SUM, group=group)
        return out
    dist.reduce_scatter_tensor(torch.view_as_real(shard_out), torch.view_as_real(out),
                               op=dist.ReduceOp.SUM, group=group)
    return shard_out


def check_plan_hash(plan_hash: int, group=None) -> None:
    """Every rank must evaluate the same plan (the same device programs and
    tables): compare the plans' hashes (hsf_plan_info.plan_hash) across ranks."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    h = torch.tensor([plan_hash & 0x7FFFFFFFFFFFFFFF], dtype=torch.int64, device=dev)
    lo, hi = h.clone(), h.clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    if int(lo.item()) != int(hi.item()):
        raise RuntimeError("plan hash mismatch across ranks (HSF_ERR_PLAN_MISMATCH)")


_LIB_COMMS = {}


def library_comm(group=None):
    """The library's own NCCL communicator for this process group
    (hsf_comm_create), built once: rank 0's unique id travels through
    torch.distributed, then every rank joins."""
    import torch
    import torch.distributed as dist
    from .hsf import Comm
    key = id(group)
    if key not in _LIB_COMMS:
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [Comm.unique_id() if rank == 0 else None]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(obj, src=src, group=group)
        _LIB_COMMS[key] = Comm(obj[0], world, rank, torch.cuda.current_device())
    return _LIB_COMMS[key]


def run_sharded(plan, out, shard: Shard, shard_out=None, bitstrings=None, precision="auto", group=None,
                row_range=None, comm=None, phases=None):
    """GPU entry: `plan.run` (libhsf.so, C ABI) on this rank's range and the
    mode's exchange step.  With `comm` (library_comm()) the all-reduce /
    reduce-scatter runs inside the library, enqueued right after the path-sum
    in the run's CUDA graph; otherwise through torch.distributed.  `row_range`
    overrides the shard's rows (prefix outputs: every rank evaluates the same
    first rows).  Returns the tensor holding this rank's result; with a list
    `phases`, appends the run's per-phase ms (hsf_run_args.phase_ms)."""
    timings = phases is not None
    if comm is not None and shard.mode in ("allreduce", "reduce_scatter") and comm.nranks > 1:
        if shard.path_range[0] >= shard.path_range[1]:
            raise ValueError("the library collective needs a non-empty path range on every rank")
        r = plan.run(out, bitstrings=bitstrings, path_range=shard.path_range, row_range=row_range or shard.row_range,
                     precision=precision, comm=comm, coll=shard.mode, coll_out=shard_out, timings=timings)
        if timings:
            phases.append(r)
        return shard_out if shard.mode == "reduce_scatter" else out

    def partial(path_range, rows, o):
        if isinstance(o, MulticastBuffer):
            r = plan.run(None, bitstrings=bitstrings, path_range=path_range, precision=precision, multicast=o.mc,
                         timings=timings)
        elif isinstance(o, PeerShards):
            r = plan.run(None, bitstrings=bitstrings, path_range=path_range, precision=precision, out_shards=o.ptrs,
                         timings=timings)
        else:
            r = plan.run(o, bitstrings=bitstrings, path_range=path_range, row_range=row_range or rows,
                         precision=precision, timings=timings)
        if timings:
            phases.append(r)
    return sharded_step(shard, partial, out, shard_out, group)
