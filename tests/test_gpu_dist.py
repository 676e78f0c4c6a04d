"""GPU coverage of the multi-GPU partition (paper_2502_06959_b200/dist.py) and
the exchange step behind the C ABI (hsf_comm_*, hsf_run_args.coll), against
the CPU oracle.  The pool has one GPU per call, so G-rank runs are emulated in
one process: every rank's shard is evaluated by Plan.run (the CUDA path) on
its own path / row range into its own device buffer, and the mode's exchange
is applied on the device (sum / slice / concatenation) -- the same partition
the NCCL run uses.  The library's communicator runs with one rank (NCCL
refuses two ranks on one GPU): the collective is then the identity, but the
plan-hash check, argument validation and the graph capture of the NCCL call
all run."""
import numpy as np
import pytest

from hsf_inputs import make_config
from oracle import hsf_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as T
    from paper_2502_06959_b200 import build
    build.build()
    assert T.cuda.is_available()
    return T


def _oracle(inst, bits=None):
    n, g = O.parse_circuit(inst.text)
    P = O.plan(n, g, inst.n_low, inst.blocks)
    A, B, c = O.half_states(P)
    return O.recombine_full(A, B, c) if bits is None else O.recombine_bits(A, B, c, bits, inst.n_low)


def _check(got, ref, tol=1e-5, rel=1e-5):
    d = np.abs(got - ref)
    r = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert d.max() <= tol and r <= rel, (d.max(), r)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name,mode", [("c5", "allreduce"), ("c3", "allreduce"), ("c2", "reduce_scatter"),
                                       ("c2", "rows"), ("c4", "rows"), ("c4", "reduce_scatter"),
                                       ("c4", "allreduce"), ("c2", "fused_rs"), ("c5", "fused_bits"),
                                       ("c3", "fused_bits")])
def test_emulated_ranks_every_mode(torch, world, name, mode):
    from paper_2502_06959_b200 import Plan
    from paper_2502_06959_b200 import dist as D
    if mode == "fused_rs":  # shards of >= 256 rows (the GEMM's pair tiles)
        from hsf_inputs.circuits import make_c2
        inst = make_c2(n=20, n_low=10)
    else:
        inst = make_config(name, twin=True)
    full = inst.bitstrings is None
    P = Plan(inst.text, inst.n_low, inst.blocks)
    ref = _oracle(inst, None if full else inst.bitstrings)
    bits = None if full else torch.from_numpy(inst.bitstrings.view(np.int64)).cuda()
    n_a = inst.n - inst.n_low
    parts = []
    shards = None
    if mode == "fused_rs":
        shards = [torch.zeros(((1 << n_a) // world) << inst.n_low, dtype=torch.complex64, device="cuda")
                  for _ in range(world)]
    if mode == "fused_bits":
        L = D.bits_shard_len(len(inst.bitstrings), world)
        shards = [torch.zeros(L, dtype=torch.complex64, device="cuda") for _ in range(world)]
    for r in range(world):
        sh = D.make_shard(mode, P.n_paths, n_a, r, world, full)
        if mode == "fused_rs":  # every rank's epilogue adds into every owner's shard
            P.run(None, path_range=sh.path_range, out_shards=shards)
            continue
        if mode == "fused_bits":  # every rank's block gather adds into every owner's samples
            P.run(None, bitstrings=bits, path_range=sh.path_range, out_shards=shards)
            continue
        rows = (sh.row_range[1] - sh.row_range[0]) if sh.row_range else (1 << n_a)
        o = torch.empty((rows << inst.n_low) if full else len(inst.bitstrings), dtype=torch.complex64, device="cuda")
        P.run(o, bitstrings=bits, path_range=sh.path_range, row_range=sh.row_range)
        parts.append((sh, o))
    torch.cuda.synchronize()
    if mode == "allreduce":
        got = sum(o for _, o in parts)
    elif mode == "reduce_scatter":  # rank r keeps rows [r R/G, (r+1) R/G) of the sum
        tot = sum(o for _, o in parts)
        got = torch.cat([tot.view(world, -1)[r] for r in range(world)])
        assert [sh.out_rows for sh, _ in parts] == [D.row_range_for_rank(n_a, r, world) for r in range(world)]
    elif mode == "rows":
        got = torch.cat([o for _, o in parts])
    else:
        got = torch.cat(shards)[:len(ref)]
    _check(got.cpu().numpy(), ref)


@pytest.mark.parametrize("n_shards", [1, 2, 3, 4])
def test_fused_bits_shards_rejects_and_reduces(torch, n_shards):
    # owner-sharded bitstring output (hsf_run_args.out_shards in bitstring
    # mode): two path halves reduce-added into the same zeroed shards == the
    # oracle's amplitudes, ragged last shard (n not divisible by 3)
    from paper_2502_06959_b200 import Plan
    from paper_2502_06959_b200.hsf import HsfError
    inst = make_config("c5", twin=True)
    P = Plan(inst.text, inst.n_low, inst.blocks)
    ref = _oracle(inst, inst.bitstrings)
    bits = torch.from_numpy(inst.bitstrings.view(np.int64)).cuda()
    L = -(-len(ref) // n_shards)
    shards = [torch.zeros(L, dtype=torch.complex64, device="cuda") for _ in range(n_shards)]
    h = P.n_paths // 2
    for pr in ((0, h), (h, P.n_paths)):
        P.run(None, bitstrings=bits, path_range=pr, out_shards=shards)
    torch.cuda.synchronize()
    _check(torch.cat(shards)[:len(ref)].cpu().numpy(), ref)
    with pytest.raises(HsfError):  # the per-sample gather (too few samples per block) has no sharded epilogue
        P.run(None, bitstrings=bits[:4], out_shards=shards)


@pytest.mark.parametrize("name,coll", [("c5", "allreduce"), ("c3", "allreduce"), ("c2", "allreduce"),
                                       ("c2", "reduce_scatter"), ("c1", "allreduce")])
def test_library_comm_single_rank(torch, name, coll):
    # hsf_comm_create with one rank: plan-hash check, the NCCL call captured in
    # the run's graph after the path-sum (identity at one rank), replayed
    from paper_2502_06959_b200 import Plan
    from paper_2502_06959_b200.hsf import Comm
    inst = make_config(name, twin=True)
    full = inst.bitstrings is None
    P = Plan(inst.text, inst.n_low, inst.blocks, dtype=inst.dtype)
    ref = _oracle(inst, None if full else inst.bitstrings)
    comm = Comm(Comm.unique_id(), 1, 0, torch.cuda.current_device())
    cdt = torch.complex64 if inst.dtype == "c64" else torch.complex128
    bits = None if full else torch.from_numpy(inst.bitstrings.view(np.int64)).cuda()
    out = torch.empty(len(ref), dtype=cdt, device="cuda")
    sh = torch.empty_like(out) if coll == "reduce_scatter" else None
    for _ in range(3):  # capture, then replays
        out.fill_(0)
        P.run(out, bitstrings=bits, comm=comm, coll=coll, coll_out=sh)
    torch.cuda.synchronize()
    got = (sh if sh is not None else out).cpu().numpy()
    tol = 1e-11 if inst.dtype == "c128" else 1e-5
    _check(got, ref, tol, 1e-12 if inst.dtype == "c128" else 1e-5)
    comm.close()


def test_library_comm_argument_errors(torch):
    from paper_2502_06959_b200 import Plan
    from paper_2502_06959_b200.hsf import Comm, HsfError
    inst = make_config("c2", twin=True)
    P = Plan(inst.text, inst.n_low, inst.blocks)
    comm = Comm(Comm.unique_id(), 1, 0)
    out = torch.empty(1 << inst.n, dtype=torch.complex64, device="cuda")
    with pytest.raises(ValueError):
        P.run(out, coll="allreduce")  # no communicator
    with pytest.raises(ValueError):
        P.run(out, comm=comm, coll="reduce_scatter")  # no destination
    with pytest.raises(HsfError):  # host output cannot take the device exchange step
        P.run(np.empty(1 << inst.n, np.complex64), comm=comm, coll="allreduce")
    comm.close()


def test_run_sharded_with_library_comm(torch):
    # dist.run_sharded's library path (one rank: the exchange is inside hsf_run)
    import torch.distributed as dist
    from paper_2502_06959_b200 import Plan
    from paper_2502_06959_b200 import dist as D
    from paper_2502_06959_b200.hsf import Comm
    inst = make_config("c5", twin=True)
    P = Plan(inst.text, inst.n_low, inst.blocks)
    ref = _oracle(inst, inst.bitstrings)
    sh = D.make_shard("allreduce", P.n_paths, inst.n - inst.n_low, 0, 1, False)
    out = torch.empty(len(ref), dtype=torch.complex64, device="cuda")
    bits = torch.from_numpy(inst.bitstrings.view(np.int64)).cuda()
    comm = Comm(Comm.unique_id(), 1, 0)
    ph = []
    res = D.run_sharded(P, out, sh, bitstrings=bits, comm=comm, phases=ph)
    torch.cuda.synchronize()
    assert res is out and len(ph) == 1 and len(ph[0]) == 5
    _check(out.cpu().numpy(), ref)
    assert not dist.is_initialized()
    comm.close()


@pytest.mark.parametrize("name", ["c5", "c3"])
def test_nvls_multicast_bits_single_rank(torch, name):
    # NVLS multicast buffer (hsf_mcast_*, a team of one GPU here): the block
    # gather's multimem.red.add through the multicast address lands in the
    # rank's copy; two path halves accumulate to the oracle's amplitudes, also
    # through dist.run_sharded (mode nvls_bits: zero, evaluate, result = local)
    from paper_2502_06959_b200 import Plan
    from paper_2502_06959_b200 import dist as D
    from paper_2502_06959_b200.hsf import HsfError
    inst = make_config(name, twin=True)
    P = Plan(inst.text, inst.n_low, inst.blocks)
    ref = _oracle(inst, inst.bitstrings)
    bits = torch.from_numpy(inst.bitstrings.view(np.int64)).cuda()
    try:
        mb = D.MulticastBuffer(len(ref))
    except HsfError as e:  # this pool's single-GPU partitions reject every multicast object
        assert e.name == "HSF_ERR_UNSUPPORTED", e
        pytest.skip(str(e))
    h = P.n_paths // 2
    for pr in ((0, h), (h, P.n_paths)):
        P.run(None, bitstrings=bits, path_range=pr, multicast=mb.mc)
    torch.cuda.synchronize()
    _check(mb.local.cpu().numpy(), ref)
    sh = D.make_shard("nvls_bits", P.n_paths, inst.n - inst.n_low, 0, 1, False)
    for _ in range(2):  # graph capture, then replay (zeroed in between by sharded_step)
        res = D.run_sharded(P, mb, sh, bitstrings=bits)
    torch.cuda.synchronize()
    _check(res.cpu().numpy(), ref)
    mb.close()


def test_debug_build_parity(torch):
    # libhsf_debug.so (bounded mbarrier waits that report and trap, the
    # sanitizer substitute) gives the same results: a tcgen05 GEMM run and a
    # bitstring run against the oracle, in a fresh process
    import os
    import subprocess
    import sys
    from paper_2502_06959_b200 import build
    build.build(debug=True)
    code = r"""
import numpy as np, torch
from hsf_inputs import make_config
from oracle import hsf_oracle as O
from paper_2502_06959_b200 import Plan, hsf
assert hsf.LIB_PATH.endswith("libhsf_debug.so")
for name in ("c2", "c5"):
    inst = make_config(name, twin=True)
    n, g = O.parse_circuit(inst.text)
    ref = O.schrodinger(n, g)
    P = Plan(inst.text, inst.n_low, inst.blocks)
    if inst.bitstrings is None:
        out = torch.empty(1 << n, dtype=torch.complex64, device="cuda")
        P.run(out)
    else:
        ref = ref[inst.bitstrings.astype(np.int64)]
        out = torch.empty(len(ref), dtype=torch.complex64, device="cuda")
        P.run(out, bitstrings=torch.from_numpy(inst.bitstrings.view(np.int64)).cuda())
    torch.cuda.synchronize()
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-5, name
print("debug build ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, HSF_DEBUG_LIB="1"), cwd=root,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "debug build ok" in r.stdout, r.stdout + r.stderr
