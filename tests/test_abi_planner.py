"""CPU tests of libhsf.so: the library loads and exports every symbol of
include/hsf.h, and the host planner (hsf_plan: C++ parser, convex schedule,
block assembly, Jacobi SVD, path counts) agrees with what the paper and the
oracle fix.  No GPU compute is called here."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

from hsf_inputs import make_config, random_small_circuit
from hsf_inputs.circuits import make_sbm_qaoa
from oracle import hsf_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def hsf():
    from paper_2502_06959_b200 import build, hsf as H
    build.build()
    return H


def test_header_symbols_exported(hsf):
    hdr = open(os.path.join(ROOT, "include", "hsf.h")).read()
    names = set(re.findall(r"^\w[\w\s\*]*?\b(hsf_\w+)\s*\(", hdr, re.M))
    assert {"hsf_plan", "hsf_run", "hsf_plan_free", "hsf_plan_info_get"} <= names
    lib = ctypes.CDLL(hsf.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(hsf.EXPORTS) == names


def test_version_and_status_strings(hsf):
    assert "sm_100a" in hsf.version()
    L = hsf.lib()
    assert L.hsf_status_str(0) == b"HSF_OK"
    assert L.hsf_status_str(5) == b"HSF_ERR_NONCONVEX_BLOCK"


def _sig(inst, **kw):
    from paper_2502_06959_b200 import Plan
    return Plan(inst.text, inst.n_low, inst.blocks, dtype=inst.dtype, **kw)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_path_counts_and_sigmas_full_configs(hsf, name):
    inst = make_config(name, n_bits=0) if name in ("c3", "c5") else make_config(name)
    P = _sig(inst)
    n, g = O.parse_circuit(inst.text)
    Po = O.plan(n, g, inst.n_low, inst.blocks)
    expect = {"c1": 16, "c2": 4096, "c3": 256, "c4": 64, "c5": 256}[name]
    assert P.n_paths == Po.n_paths == expect
    assert P.ranks == Po.radices
    for s_cpp, u in zip(P.sigmas, Po.units):
        assert np.allclose(s_cpp, u.sigmas, rtol=1e-12, atol=1e-12 * u.sigmas[0])
    expect_t = {"c1": 12, "c2": 144, "c3": 8, "c4": 6, "c5": 48}[name]
    assert abs(P.log2_n_paths_individual - expect_t) < 1e-9


@pytest.mark.parametrize("seed", range(25))
def test_sigmas_random_blocks_match_lapack(hsf, seed):
    inst = random_small_circuit(seed, max_block_qubits=6)
    n, g = O.parse_circuit(inst.text)
    Po = O.plan(n, g, inst.n_low, inst.blocks)
    P = _sig(inst)
    assert P.ranks == Po.radices
    for s_cpp, u in zip(P.sigmas, Po.units):
        assert np.allclose(s_cpp, u.sigmas, rtol=1e-11, atol=1e-12 * u.sigmas[0])
    Pi = _sig(inst, individual=True)
    Poi = O.plan(n, g, inst.n_low, None, "individual")
    assert Pi.ranks == Poi.radices


def test_paper_examples_ranks(hsf):
    from paper_2502_06959_b200 import Plan
    # Example 2: CNOT rank 2; SWAP rank 4; Eq. 11 cascade rank 2
    assert Plan("qubits 2\ncx 1 0\n", 1, [[0]]).ranks == [2]
    assert Plan("qubits 2\nswap 1 0\n", 1, [[0]]).ranks == [4]
    P = Plan("qubits 4\ncx 3 2\ncx 3 1\ncx 3 0\n", 3, [[0, 1, 2]])
    assert P.ranks == [2]
    assert abs(P.log2_n_paths_individual - 3) < 1e-12
    # RZZ(t): sigma = (2|cos t/2|, 2|sin t/2|)
    t = 0.7
    P = Plan(f"qubits 2\nrzz {t.hex()} 1 0\n", 1, [[0]])
    assert np.allclose(P.sigmas[0], [2 * math.cos(t / 2), 2 * math.sin(t / 2)], atol=1e-14)


def test_table2_like_counts(hsf):
    from paper_2502_06959_b200 import Plan
    inst = make_sbm_qaoa(seed=30, sizes=(15, 15), p_inter=0.1)
    P = Plan(inst.text, inst.n_low, inst.blocks)
    n, g = O.parse_circuit(inst.text)
    Po = O.plan(n, g, inst.n_low, inst.blocks)
    assert P.n_paths == Po.n_paths
    assert all(r == 2 for r in P.ranks)


@pytest.mark.parametrize("text,n_low,blocks,status", [
    ("qubits 3\ncx 2 0\nh 0\ncx 2 1\ncx 0 1\n", 1, [[0, 3]], "HSF_ERR_NONCONVEX_BLOCK"),
    ("qubits 2\nfoo 0\n", 1, None, "HSF_ERR_UNSUPPORTED_GATE"),
    ("qubits 2\ncx 0 0\n", 1, None, "HSF_ERR_DUPLICATE_QUBIT"),
    ("qubits 2\ncx 0 2\n", 1, None, "HSF_ERR_DUPLICATE_QUBIT"),
    ("h 0\n", 1, None, "HSF_ERR_PARSE"),
    ("qubits 2\nrx zz 0\n", 1, None, "HSF_ERR_PARSE"),
    ("qubits 2\nh 0\n", 0, None, "HSF_ERR_INVALID_ARG"),
    ("qubits 2\nh 0\n", 2, None, "HSF_ERR_INVALID_ARG"),
])
def test_errors(hsf, text, n_low, blocks, status):
    from paper_2502_06959_b200 import Plan, HsfError
    with pytest.raises(HsfError) as ei:
        Plan(text, n_low, blocks)
    assert ei.value.name == status


def test_path_budget(hsf):
    from paper_2502_06959_b200 import HsfError, Plan
    inst = make_config("c5", n_bits=0)
    with pytest.raises(HsfError) as ei:
        Plan(inst.text, inst.n_low, None, individual=True)  # 2^48 > 2^26
    assert ei.value.name == "HSF_ERR_PATH_BUDGET"


def test_dense_block_too_large(hsf):
    from paper_2502_06959_b200 import HsfError, Plan
    inst = make_config("c3", n_bits=0)
    with pytest.raises(HsfError) as ei:
        Plan(inst.text, inst.n_low, [list(range(0, 200))], max_dense_block_qubits=6)
    assert ei.value.name in ("HSF_ERR_BLOCK_TOO_LARGE", "HSF_ERR_NONCONVEX_BLOCK")


def test_plan_hash_deterministic(hsf):
    from paper_2502_06959_b200 import Plan
    inst = make_config("c4")
    assert Plan(inst.text, inst.n_low, inst.blocks).plan_hash == Plan(inst.text, inst.n_low, inst.blocks).plan_hash
    inst2 = make_config("c4", seed=99)
    assert Plan(inst.text, inst.n_low, inst.blocks).plan_hash != Plan(inst2.text, inst2.n_low, inst2.blocks).plan_hash


def test_workspace_bytes_no_gpu(hsf):
    from paper_2502_06959_b200 import Plan
    inst = make_config("c5", n_bits=0)
    P = Plan(inst.text, inst.n_low, inst.blocks)
    b = P.workspace_bytes(bitstrings_count=1 << 22)
    # both halves' leaves + the transposed copy of the half the block gather
    # does not read in place dominate: 128 x 2^20 complex64 each with the last
    # (diagonal) unit folded, 256 x 2^20 without
    assert 3 * 128 * (1 << 20) * 8 <= b < 3 * 256 * (1 << 20) * 8
    P2 = Plan(inst.text, inst.n_low, inst.blocks, fold_trailing_diag=False)
    assert P2.workspace_bytes(bitstrings_count=1 << 22) >= 3 * 256 * (1 << 20) * 8


def test_run_describe_no_gpu(hsf):
    # hsf_run_describe: the launch sequence and algorithmic work, host only
    from paper_2502_06959_b200 import Plan
    inst = make_config("c5", n_bits=0)
    P = Plan(inst.text, inst.n_low, inst.blocks)
    d = P.describe(1 << 22)
    assert d["core"] == "block_gather" and d["direct_half"] in (0, 1) and d["K"] == 128
    assert d["core_bytes"] == 128 * (1 << 20) * 8 + (1 << 22) * (128 * 8 + 4 + 8 + 8)
    assert d["core_flops_useful"] == 8 * 128 * (1 << 22)
    assert d["sim_bytes"] == P.fold_tree_bytes and d["sim_flops"] == P.fold_tree_flops
    assert d["kernel_launches"] == -1  # never run
    d2 = P.describe(1 << 22, path_range=(3, 9))  # unaligned: the full tree, K = 6 padded to 64
    assert d2["tree_variant"] == (0, 0) and d2["K"] == 6
    assert d2["sim_bytes"][0] == pytest.approx(P.tree_bytes[0] * 6 / 256)
    d3 = P.describe(1 << 10)  # too few samples per block: the per-sample gather
    assert d3["core"] == "gather"
    c2 = make_config("c2")
    Q = Plan(c2.text, c2.n_low, c2.blocks)
    e = Q.describe()
    assert e["core"] == "tc_pair" and e["tc_products"] == 3
    assert e["core_flops_useful"] == 8 * 4096 * 4096 * 4096
    assert e["core_flops_executed"] == 3 * 2 * 4096 * 8192 * 8192
    assert Q.describe(precision="simt")["core"] == "simt"
    assert Q.describe(row_range=(0, 16))["core"] == "tc_swapped"


def test_trailing_fold_detection(hsf):
    # fold needs: last units all-diagonal and no local gate after them
    from paper_2502_06959_b200 import Plan
    for name, units in [("c1", 1), ("c2", 0), ("c3", 0), ("c4", 0), ("c5", 1)]:
        inst = make_config(name, twin=True)
        P = Plan(inst.text, inst.n_low, inst.blocks)
        assert P.fold_units == units, name
        assert Plan(inst.text, inst.n_low, inst.blocks, fold_trailing_diag=False).fold_units == 0
    # three trailing CZ across the cut, nothing after: all three fold
    txt = "qubits 4\nh 0\nh 1\nh 2\nh 3\ncz 1 2\ncz 0 3\ncz 1 3\n"
    P = Plan(txt, 2, [])
    assert P.fold_units == 3 and P.n_paths == 8
    # an H on qubit 2 after cz(1,2) pins the tree to level 1: the two later
    # units still fold; an H on qubit 3 (after every unit) blocks all folding
    assert Plan(txt + "h 2\n", 2, []).fold_units == 2
    assert Plan(txt + "h 3\n", 2, []).fold_units == 0


def test_half_sided_tail_detection(hsf, monkeypatch):
    # full-output runs fold, per half, the trailing units whose factors on that
    # half are diagonal with no gate of that half after them (hoisting moves
    # commuting gates above them)
    from paper_2502_06959_b200 import Plan
    # default: the longest fold whose weight table W[T][2^m] has <= 2^20
    # entries (c2: T = 2^8 of its 2^12 paths), or where the half's gates end
    for name, twin, tail in [("c1", True, (1, 1)), ("c2", True, (8, 0)), ("c2", False, (8, 0)),
                             ("c3", True, (0, 0)), ("c4", True, (0, 0)), ("c5", True, (1, 1))]:
        inst = make_config(name, twin=twin)
        assert Plan(inst.text, inst.n_low, inst.blocks).tail_units == tail, name
    # longest fold the gates allow
    monkeypatch.setenv("HSF_TAIL_PREFIX_BYTES", "0")
    for name, twin, tail in [("c1", True, (1, 1)), ("c2", True, (8, 0)), ("c2", False, (12, 0)),
                             ("c3", True, (0, 0)), ("c4", True, (0, 0)), ("c5", True, (1, 1))]:
        inst = make_config(name, twin=twin)
        P = Plan(inst.text, inst.n_low, inst.blocks)
        assert P.tail_units == tail, name
        assert Plan(inst.text, inst.n_low, inst.blocks, fold_trailing_diag=False).tail_units == (0, 0)
    # c2: every A factor is a 1-qubit phase that commutes with all later A gates,
    # so A's tree is the root alone
    inst = make_config("c2")
    assert Plan(inst.text, inst.n_low, inst.blocks).tail_passes[0] == 1
    txt = "qubits 4\nh 0\nh 1\nh 2\nh 3\ncz 1 2\ncz 0 3\ncz 1 3\n"
    assert Plan(txt, 2, []).tail_units == (3, 3)
    # H on qubit 2 (half A) after unit 0 pins A's tree to level 1; H on qubit 3
    # after every unit blocks A's tail; H on qubit 0 (half B) after unit 1
    # leaves only unit 2 in B's tail
    assert Plan(txt + "h 2\n", 2, []).tail_units == (2, 3)
    assert Plan(txt + "h 3\n", 2, []).tail_units == (0, 3)
    assert Plan(txt + "h 0\n", 2, []).tail_units == (3, 1)


def test_head_scalar_detection(hsf, monkeypatch):
    # leading units whose factors act on computational-basis qubits of a half
    # (only X / diagonal gates before them there) are scalars on that half
    from paper_2502_06959_b200 import Plan
    inst = make_config("c2")  # B's 12 factors precede its QFT on the X-prepared input
    P = Plan(inst.text, inst.n_low, inst.blocks)
    assert P.head_units == (0, 12) and P.tail_passes[1] == 1
    for name in ("c1", "c3", "c4", "c5"):  # H / SU(2) layers first: no head
        inst = make_config(name, twin=True)
        assert Plan(inst.text, inst.n_low, inst.blocks).head_units == (0, 0), name
    # B: cz(1,2) and cp(0,3) see basis qubits 1, 0; h 1 ends it before cz(1,3).
    # A: qubit 3 stays a basis qubit through cz(1,3); h 3 ends it before cz(0,2)
    t = ("qubits 4\nx 1\nx 3\ncz 1 2\ncp 0x1.8p-1 0 3\nh 1\nh 2\ncz 1 3\nh 0\nh 3\ncz 0 2\n"
         "rx 0x1.4p-2 1\n")
    P = Plan(t, 2, [])
    assert P.n_units == 4 and P.head_units == (3, 2) and P.tail_units == (1, 1)
    # a superposition gate before the first unit on its qubit ends the head
    assert Plan("qubits 2\nh 0\ncz 0 1\n", 1, []).head_units == (1, 0)
    assert Plan("qubits 2\nx 0\ncz 0 1\nh 1\n", 1, []).head_units == (1, 1)
    assert Plan(t, 2, [], fold_trailing_diag=False).head_units == (0, 0)
    monkeypatch.setenv("HSF_NO_HEAD_FOLD", "1")
    assert Plan(t, 2, []).head_units == (0, 0)


@pytest.mark.parametrize("seed", range(8))
def test_auto_blocks_match_oracle_finder(hsf, seed):
    # the C++ cascade finder (hsf_plan n_blocks = -1) and the oracle's
    # networkx-based finder agree on the number of units and paths
    from hsf_inputs.circuits import make_sbm_qaoa
    from oracle import hsf_oracle as O
    from paper_2502_06959_b200 import Plan
    sizes = [(6, 6), (7, 8), (15, 15), (16, 17)][seed % 4]
    inst = make_sbm_qaoa(seed=200 + seed, sizes=sizes, p_inter=0.1 + 0.02 * (seed % 4))
    n, g = O.parse_circuit(inst.text)
    blocks, ncasc = O.find_cascades(g, inst.n_low)
    Po = O.plan(n, g, inst.n_low, blocks)
    P = Plan(inst.text, inst.n_low, "auto", log2_path_budget=40)
    assert P.n_units == len(Po.units) == ncasc
    assert P.n_paths == Po.n_paths
    assert P.n_joint_blocks == len(blocks)


def test_partition_mask_validation_and_counts(hsf):
    from paper_2502_06959_b200 import HsfError, Plan
    # GHZ-like chain: cutting between {0,2} and {1,3} crosses 3 CNOTs, the
    # contiguous cut {0,1}|{2,3} only one
    txt = "qubits 4\nh 0\ncx 0 1\ncx 1 2\ncx 2 3\n"
    assert Plan(txt, 2, []).n_units == 1
    assert Plan(txt, [0, 2], []).n_units == 3
    assert Plan(txt, [0, 1], []).plan_hash == Plan(txt, 2, []).plan_hash
    with pytest.raises(HsfError):
        Plan(txt, [0, 9], [])  # qubit beyond the circuit


def test_comm_unique_id_no_gpu(hsf):
    # hsf_comm_unique_id: 128 bytes from NCCL (loaded at run time); no GPU needed
    try:
        uid = hsf.Comm.unique_id()
    except hsf.HsfError as e:  # NCCL not loadable: the library says so, with its own status
        assert e.name == "HSF_ERR_NCCL"
        return
    assert isinstance(uid, bytes) and len(uid) == 128 and uid != bytes(128)
    assert hsf.lib().hsf_status_str(12) == b"HSF_ERR_NCCL" and hsf.lib().hsf_status_str(13) == b"HSF_ERR_PLAN_MISMATCH"


@pytest.mark.parametrize("name", ["c1", "c2", "c5", "q30-1", "q33-3"])
def test_analytic_cascade_sigmas_match_svd(hsf, name):
    # Eq. 11 route: closed-form rank-2 factors of CP / RZZ cascades; the
    # singular values equal the numeric route's (assembly + Jacobi SVD) and
    # LAPACK's on the oracle's block matrices
    from paper_2502_06959_b200 import Plan
    inst = make_config(name)
    blocks = inst.blocks
    if blocks == "auto":
        blocks = O.find_cascades(O.parse_circuit(inst.text)[1], inst.n_low)[0]
    P = Plan(inst.text, inst.n_low, blocks, dtype=inst.dtype)
    Q = Plan(inst.text, inst.n_low, blocks, dtype=inst.dtype, analytic_cascades=False)
    assert P.n_analytic_units == P.n_joint_blocks > 0 and Q.n_analytic_units == 0
    assert P.ranks == Q.ranks and P.n_paths == Q.n_paths
    for a, b in zip(P.sigmas, Q.sigmas):
        assert np.allclose(a, b, rtol=1e-11, atol=0)
    n, g = O.parse_circuit(inst.text)
    OP = O.plan(n, g, inst.n_low, blocks)
    for a, u in zip(P.sigmas, OP.units):
        assert np.allclose(sorted(a), sorted(u.sigmas[:len(a)]), rtol=1e-10)


def test_analytic_cascade_cnot_and_mixed_sides(hsf):
    # CNOT cascade (Eq. 11: P0 (x) I..I + P1 (x) X..X, degenerate sigma), targets
    # on both sides of the cut, control on the low side, and a non-cascade
    # block (falls back to the numeric route)
    from paper_2502_06959_b200 import Plan
    text = ("qubits 6\nh 3\ncx 3 0\ncx 3 1\ncx 3 4\ncx 3 2\ncp 0x1.8p-1 1 5\nrzz 0x1.4p+0 5 1\nrzz 0x1.2p-1 2 1\n"
            "cz 1 4\nh 4\ncx 2 5\n")
    blocks = [[1, 2, 3, 4], [5, 6, 7, 8], [10]]
    P = Plan(text, 3, blocks)
    Q = Plan(text, 3, blocks, analytic_cascades=False)
    assert P.unit_analytic == [True, True, False]  # a single gate keeps the numeric route
    assert P.ranks == Q.ranks == [2, 2, 2]
    for a, b in zip(P.sigmas, Q.sigmas):
        assert np.allclose(a, b, rtol=1e-12, atol=1e-12)
    R = Plan("qubits 4\ncx 2 1\nh 2\ncx 2 0\n", 2, [[0, 1, 2]])  # H on the shared qubit: not a cascade
    assert R.unit_analytic == [False]


def test_tleaf_variant_planned(hsf):
    # bitstring runs: the transposed half's last transition gets a T-leaf pass
    # (2^10-amplitude tiles, R leaves per parent, one 64-thread group per leaf);
    # its generated source is inspectable and self-contained
    from paper_2502_06959_b200 import Plan
    inst = make_config("c5", n_bits=0)
    P = Plan(inst.text, inst.n_low, inst.blocks)
    src = P.pass_source(0, 0, variant=64 + 1)  # folded tree, half A
    assert src and "bar.sync" in src and "cp.async.ca.shared.global" in src and "pb_[sb + " in src and "NTILES" in src
    assert P.pass_source(0, 0, variant=64 + 3) is None  # no such tree variant
    d = P.describe(1 << 22)  # c5 as benched: half B read in place, half A through its T-leaf pass
    assert (d["direct_half"], d["tleaf_half"], d["tleaf_leaves"]) == (1, 0, 8) and d["prep_bytes"] == 0
    assert P.describe(1 << 22, path_range=(2, 10))["tleaf_half"] == -1  # K = 4 padded: no T-leaf
    c3 = make_config("c3", n_bits=0)
    Q = Plan(c3.text, c3.n_low, c3.blocks)
    e = Q.describe(1 << 20)
    assert (e["direct_half"], e["tleaf_half"], e["tleaf_leaves"]) == (0, 1, 4)


def test_smem_tier_choice(hsf):
    # K1 tier limits: 2^13 complex64 always whole-state; 2^14 complex64 whole
    # with smem_tier = 1 (128 KiB per CTA), by the cost model otherwise; 2^15
    # never (256 KiB does not fit in 227 KiB of shared memory)
    from paper_2502_06959_b200 import Plan
    for m, tier, want in [(13, 0, True), (14, 1, True), (15, 1, False)]:
        inst = make_config("c5", n=2 * m, n_low=m, layers=4, fanout=4, n_bits=0)
        P = Plan(inst.text, inst.n_low, inst.blocks, smem_tier=tier)
        assert P.whole_state == (want, want), (m, tier, P.whole_state)
    inst = make_config("c5", n=26, n_low=13, layers=4, fanout=4, n_bits=0)
    assert Plan(inst.text, inst.n_low, inst.blocks, dtype="c128", smem_tier=1).whole_state == (True, True)
    assert Plan(inst.text, inst.n_low, inst.blocks, tile_qubits=11).whole_state == (False, False)


@pytest.mark.parametrize("na,nb,depth", [(2, 2, 4), (3, 3, 8), (4, 4, 8), (5, 5, 6), (5, 3, 7)])
def test_sequential_route_sigmas(hsf, na, nb, depth):
    # sequential (MPO-style) factors of a dense block: same rank and singular
    # values as the assembly + SVD route and as LAPACK on the oracle's block
    # matrix, without assembling the block
    import time
    from hsf_inputs import make_brick_block
    from paper_2502_06959_b200 import Plan
    inst = make_brick_block(na, nb, depth)
    t0 = time.perf_counter()
    P = Plan(inst.text, inst.n_low, inst.blocks, block_route=2)
    t_seq = time.perf_counter() - t0
    assert P.unit_sequential == [True] and P.unit_analytic == [False]
    n, g = O.parse_circuit(inst.text)
    OP = O.plan(n, g, inst.n_low, inst.blocks)
    assert P.ranks == [OP.units[0].rank]
    assert np.allclose(P.sigmas[0], OP.units[0].sigmas[:len(P.sigmas[0])], rtol=1e-10, atol=1e-12)
    if na + nb <= 8:  # the assembly route is fast enough to compare beside it
        Q = Plan(inst.text, inst.n_low, inst.blocks, block_route=1)
        assert Q.unit_sequential == [False] and P.ranks == Q.ranks
        assert np.allclose(P.sigmas[0], Q.sigmas[0], rtol=1e-11, atol=1e-12)
    assert t_seq < 2.0, t_seq  # (assembly + Jacobi SVD of the 5 + 5 block: ~12 s)


@pytest.mark.parametrize("seed", range(12))
def test_sequential_route_random_blocks(hsf, seed):
    # random blocks with dense 1..3-qubit gates (crossing 3-qubit gates have
    # 1 + 2 or 2 + 1 sides): both routes give the same ranks and sigma
    from paper_2502_06959_b200 import Plan
    inst = random_small_circuit(seed)
    P = Plan(inst.text, inst.n_low, inst.blocks, block_route=2, analytic_cascades=False)
    Q = Plan(inst.text, inst.n_low, inst.blocks, block_route=1, analytic_cascades=False)
    assert P.ranks == Q.ranks
    for a, b in zip(P.sigmas, Q.sigmas):
        assert np.allclose(a, b, rtol=1e-11, atol=1e-12)
    n, g = O.parse_circuit(inst.text)
    OP = O.plan(n, g, inst.n_low, inst.blocks)
    for a, u in zip(P.sigmas, OP.units):
        assert np.allclose(a, u.sigmas[:len(a)], rtol=1e-10, atol=1e-12)


def test_block_route_option_checked(hsf):
    from paper_2502_06959_b200 import Plan
    inst = make_config("c3", twin=True)
    with pytest.raises(hsf.HsfError):
        Plan(inst.text, inst.n_low, inst.blocks, block_route=3)
    # auto: the c3 windows (2 + 2) keep the assembly route
    assert Plan(inst.text, inst.n_low, inst.blocks).unit_sequential == [False] * len(inst.blocks)
