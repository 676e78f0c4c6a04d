"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 path partition
and its single exchange step (paper_2502_06959_b200/dist.py).

Each rank evaluates its shard with the CPU oracle standing in for `Plan.run`
(the GPU kernels are covered by tests/test_gpu_parity.py, including the
path-range and row-range arguments these shards feed them); the collective
must reassemble exactly the single-process oracle result."""
import os
import socket

import numpy as np
import pytest

from hsf_inputs import make_config
from oracle import hsf_oracle as O
from paper_2502_06959_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_partial(inst, P, bits):
    import torch

    def partial(path_range, row_range, out):
        A, B, c = O.half_states(P, *path_range)
        if bits is not None:
            v = O.recombine_bits(A, B, c, bits, inst.n_low)
        else:
            v = O.recombine_full(A, B, c)
            if row_range is not None:
                v = v[row_range[0] << inst.n_low:row_range[1] << inst.n_low]
        out.copy_(torch.from_numpy(np.ascontiguousarray(v)))
    return partial


class _HostPeers:
    """CPU stand-in for dist.PeerShards: the own row shard; the peer adds the
    GEMM epilogue makes over NVLink are emulated by a reduce-scatter of the
    rank's partial output inside `partial` (the control flow -- zero, barrier,
    evaluate, barrier -- is dist.sharded_step's own)."""

    def __init__(self, local):
        self.local = local


def _fused_partial(inst, P):
    import torch
    import torch.distributed as dist

    def partial(path_range, row_range, peers):
        assert row_range is None  # every rank evaluates all rows of its path range
        A, B, c = O.half_states(P, *path_range)
        v = torch.from_numpy(np.ascontiguousarray(O.recombine_full(A, B, c)))
        dist.reduce_scatter_tensor(torch.view_as_real(peers.local), torch.view_as_real(v), op=dist.ReduceOp.SUM)
    return partial


def _inst(name):
    if name == "single_path":  # no crossing gate: n_p = 1 < world (rank 0's range is empty)
        from types import SimpleNamespace
        bits = np.arange(16, dtype=np.uint64)
        return SimpleNamespace(text="qubits 4\nh 0\nh 2\ncz 0 1\nrx 0x1.8p-1 3\ncz 2 3\n", n=4, n_low=2,
                               blocks=[], bitstrings=bits)
    return make_config(name, twin=True)


def _fused_bits_partial(inst, P):
    import torch
    import torch.distributed as dist

    def partial(path_range, row_range, peers):
        # CPU stand-in for the block gather's reduce-adds into the owners' samples
        A, B, c = O.half_states(P, *path_range)
        v = O.recombine_bits(A, B, c, inst.bitstrings, inst.n_low)
        L = D.bits_shard_len(len(v), dist.get_world_size())
        pad = np.zeros(L * dist.get_world_size(), dtype=complex)
        pad[:len(v)] = v
        dist.reduce_scatter_tensor(torch.view_as_real(peers.local), torch.view_as_real(torch.from_numpy(pad)),
                                   op=dist.ReduceOp.SUM)
    return partial


def _worker(rank, world, port, name, mode, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        inst = _inst(name)
        n, g = O.parse_circuit(inst.text)
        P = O.plan(n, g, inst.n_low, inst.blocks)
        full = inst.bitstrings is None
        n_a = n - inst.n_low
        sh = D.make_shard(mode, P.n_paths, n_a, rank, world, full)
        if full:
            rows = (sh.row_range[1] - sh.row_range[0]) if sh.row_range else (1 << n_a)
            out = torch.zeros(rows << inst.n_low, dtype=torch.complex128)
            shard_out = torch.zeros((1 << n) // world, dtype=torch.complex128) if mode == "reduce_scatter" else None
        else:
            out = torch.zeros(len(inst.bitstrings), dtype=torch.complex128)
            shard_out = None
        if mode == "fused_rs":
            peers = _HostPeers(torch.zeros((1 << n) // world, dtype=torch.complex128))
            res = D.sharded_step(sh, _fused_partial(inst, P), peers)
        elif mode == "fused_bits":
            L = D.bits_shard_len(len(inst.bitstrings), world)
            peers = _HostPeers(torch.zeros(L, dtype=torch.complex128))
            res = D.sharded_step(sh, _fused_bits_partial(inst, P), peers)
            sh = D.Shard(sh.mode, sh.path_range, None, (rank * L, min(len(inst.bitstrings), (rank + 1) * L)))
        else:
            res = D.sharded_step(sh, _oracle_partial(inst, P, inst.bitstrings), out, shard_out)
        # gather every rank's piece on rank 0 in rank order
        pieces = [None] * world
        dist.all_gather_object(pieces, (sh.out_rows, res.numpy()))
        if rank == 0:
            q.put(pieces)
    finally:
        dist.destroy_process_group()


def _run(name, mode, world=2):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get()  # read before join: a large pickled result blocks the pipe
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    return res


def _reference(name):
    inst = _inst(name)
    n, g = O.parse_circuit(inst.text)
    psi = O.schrodinger(n, g)
    return inst, psi if inst.bitstrings is None else psi[inst.bitstrings.astype(np.int64)]


@pytest.mark.parametrize("name,mode", [("c4", "reduce_scatter"), ("c4", "rows"), ("c4", "allreduce"),
                                       ("c4", "fused_rs"), ("c2", "fused_rs"),
                                       ("c1", "allreduce"), ("c5", "allreduce"), ("c3", "allreduce"),
                                       ("single_path", "allreduce"), ("c5", "fused_bits")])
def test_two_rank_shards_reassemble(name, mode):
    inst, ref = _reference(name)
    pieces = _run(name, mode)
    if mode == "allreduce":
        for _, v in pieces:  # every rank holds the whole reduced result
            assert np.abs(v - ref).max() <= 1e-12
    elif mode == "fused_bits":  # rank r owns samples [r L, (r+1) L)
        got = np.concatenate([v for _, v in sorted(pieces, key=lambda x: x[0][0])])[:len(ref)]
        assert np.abs(got - ref).max() <= 1e-12
    else:
        got = np.concatenate([v for _, v in sorted(pieces, key=lambda x: x[0][0])])
        assert [r for r, _ in pieces] == [D.row_range_for_rank(inst.n - inst.n_low, r, 2) for r in range(2)]
        assert np.abs(got - ref).max() <= 1e-12


def test_more_ranks_than_paths():
    # ranks whose range is empty must not evaluate (hsf_run reads 0,0 as "all paths")
    rs = [D.path_range_for_rank(1, r, 2) for r in range(2)]
    assert rs == [(0, 0), (0, 1)]
    calls = []

    class Z:
        def zero_(self):
            calls.append("zero")
    D.sharded_step(D.make_shard("allreduce", 1, 2, 0, 2, False), lambda *a: calls.append("run"), Z())
    assert calls == ["zero"]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_path_ranges_cover_and_are_subtrees(world):
    # c1..c5 radices: the ranges tile [0, n_p) and start on subtree boundaries
    # (world divides the product of the leading radices)
    for name, radices in [("c1", [2] * 4), ("c2", [2] * 12), ("c3", [4] * 4), ("c4", [4] * 3), ("c5", [2] * 8)]:
        n_p = int(np.prod(radices))
        rs = [D.path_range_for_rank(n_p, r, world) for r in range(world)]
        assert rs[0][0] == 0 and rs[-1][1] == n_p
        assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
        sub = n_p // world
        assert all((p1 - p0) == sub and p0 % sub == 0 for p0, p1 in rs)


def test_default_modes():
    # c4 (K = 64, 2^34 outputs): rows; c2 (K = 4096): reduce-scatter; bitstrings: all-reduce
    assert D.default_mode(True, 64, 17, 17, 8) == "rows"
    assert D.default_mode(True, 4096, 12, 12, 8) == "reduce_scatter"
    assert D.default_mode(False, 256, 20, 20, 8) == "allreduce"
    with pytest.raises(ValueError):
        D.make_shard("rows", 16, 6, 0, 2, full_output=False)
    with pytest.raises(ValueError):
        D.make_shard("rows", 16, 1, 0, 4, full_output=True)
