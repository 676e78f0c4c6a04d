"""Pins for the CPU oracle (oracle/hsf_oracle.py) against what the paper and the
mathematics fix: paper worked examples, closed forms, brute force, invariants.
None of these compare the oracle with itself."""
import math
import os

import numpy as np
import pytest

from hsf_inputs import make_config, random_small_circuit
from hsf_inputs.circuits import make_sbm_qaoa
from oracle import hsf_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _circ(text):
    return O.parse_circuit(text)


# ------------------------------------------------------------------ gates
@pytest.mark.parametrize("name,params,k", [("h", (), 1), ("x", (), 1), ("z", (), 1), ("rx", (0.3,), 1),
                                           ("rz", (1.1,), 1), ("cz", (), 2), ("cx", (), 2), ("swap", (), 2),
                                           ("cp", (0.7,), 2), ("rzz", (2.2,), 2)])
def test_library_gates_unitary(name, params, k):
    U = O.gate_matrix(name, params, k)
    assert np.allclose(U.conj().T @ U, np.eye(1 << k), atol=1e-12)


def test_cnot_is_paper_bipartite_form():
    # PAPER.md Example 2: CNOT = P0 (x) I + P1 (x) X, written out by hand
    expect = np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], dtype=complex)
    assert np.array_equal(O.gate_matrix("cx", (), 2), expect)


def test_rzz_is_exponential_of_zz():
    # RZZ(t) = exp(-i t/2 Z(x)Z): compare with a Taylor series of the 4x4 generator
    t = 0.913
    Z = np.diag([1, -1]).astype(complex)
    G = -0.5j * t * np.kron(Z, Z)
    E, term = np.eye(4, dtype=complex), np.eye(4, dtype=complex)
    for j in range(1, 40):
        term = term @ G / j
        E = E + term
    assert np.allclose(O.gate_matrix("rzz", (t,), 2), E, atol=1e-14)


def test_rx_is_exponential_of_x():
    t = 1.37
    X = np.array([[0, 1], [1, 0]], dtype=complex)
    G = -0.5j * t * X
    E, term = np.eye(2, dtype=complex), np.eye(2, dtype=complex)
    for j in range(1, 40):
        term = term @ G / j
        E = E + term
    assert np.allclose(O.gate_matrix("rx", (t,), 1), E, atol=1e-14)


def test_z_h_relations():
    # Z written out by hand; Z = H X H and X = H Z H (the Hadamard conjugation)
    Z = np.array([[1, 0], [0, -1]], dtype=complex)
    H, X = O.gate_matrix("h", (), 1), O.gate_matrix("x", (), 1)
    assert np.allclose(O.gate_matrix("z", (), 1), Z, atol=0)
    assert np.allclose(H @ X @ H, Z, atol=1e-15) and np.allclose(H @ Z @ H, X, atol=1e-15)


def test_rz_is_exponential_of_z():
    # RZ(t) = exp(-i t/2 Z) (the RZZ / RX convention), Taylor series of the generator
    t = -2.71
    G = -0.5j * t * np.diag([1, -1]).astype(complex)
    E, term = np.eye(2, dtype=complex), np.eye(2, dtype=complex)
    for j in range(1, 40):
        term = term @ G / j
        E = E + term
    assert np.allclose(O.gate_matrix("rz", (t,), 1), E, atol=1e-14)


def test_cz_cp_phase_on_11():
    # CZ |11> = -|11>, identity on the other basis states; CZ = (I (x) H) CNOT (I (x) H);
    # CP(t) multiplies |11> by e^{it} (control and target symmetric), CP(pi) = CZ
    CZ = O.gate_matrix("cz", (), 2)
    for j in range(4):
        e = np.zeros(4, dtype=complex)
        e[j] = 1
        assert np.array_equal(CZ @ e, -e if j == 3 else e)
    IH = np.kron(np.eye(2), O.gate_matrix("h", (), 1))
    assert np.allclose(IH @ O.gate_matrix("cx", (), 2) @ IH, CZ, atol=1e-15)
    t = 0.4321
    CP = O.gate_matrix("cp", (t,), 2)
    assert np.allclose(CP @ np.array([0, 0, 0, 1]), [0, 0, 0, np.exp(1j * t)], atol=1e-15)
    assert np.allclose(CP[:3, :3], np.eye(3), atol=0)
    assert np.allclose(O.gate_matrix("cp", (math.pi,), 2), CZ, atol=1e-15)
    n, g = _circ("qubits 2\ncp %s 0 1\n" % float(t).hex())
    n2, g2 = _circ("qubits 2\ncp %s 1 0\n" % float(t).hex())
    psi0 = np.full(4, 0.5, dtype=complex)
    assert np.allclose(O.apply_gate(psi0, 2, g[0].U, g[0].qubits), O.apply_gate(psi0, 2, g2[0].U, g2[0].qubits))


def test_swap_exchanges_qubits():
    # SWAP (a (x) b) = b (x) a; SWAP = CNOT(0,1) CNOT(1,0) CNOT(0,1)
    rng = np.random.default_rng(3)
    a = rng.standard_normal(2) + 1j * rng.standard_normal(2)
    b = rng.standard_normal(2) + 1j * rng.standard_normal(2)
    S = O.gate_matrix("swap", (), 2)
    assert np.allclose(S @ np.kron(a, b), np.kron(b, a), atol=1e-15)
    CX = O.gate_matrix("cx", (), 2)
    P = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=complex)  # relabel qubits
    assert np.allclose(CX @ (P @ CX @ P) @ CX, S, atol=1e-15)


# ------------------------------------------------------------ Schroedinger
def test_bell_state_paper_example1():
    text = open(os.path.join(GOLD, "bell.txt")).read()
    circ = "\n".join(l for l in text.splitlines() if not l.startswith("#"))
    n, g = _circ(circ)
    psi = O.schrodinger(n, g)
    expect = np.array([1, 0, 0, 1]) / math.sqrt(2)
    assert np.allclose(psi, expect, atol=1e-15)


@pytest.mark.parametrize("n,n_low", [(4, 2), (7, 3), (10, 5)])
def test_ghz_across_cut(n, n_low):
    text = f"qubits {n}\nh 0\n" + "".join(f"cx {q} {q + 1}\n" for q in range(n - 1))
    n, g = _circ(text)
    expect = np.zeros(1 << n, dtype=complex)
    expect[0] = expect[-1] = 1 / math.sqrt(2)
    assert np.allclose(O.schrodinger(n, g), expect, atol=1e-14)
    assert np.allclose(O.hsf(n, g, n_low), expect, atol=1e-14)
    # individual cut: a single crossing CNOT, rank 2
    P = O.plan(n, g, n_low, None, "individual")
    assert P.radices == [2]


def _rev(i, n):
    return int(format(i, "0%db" % n)[::-1], 2)


@pytest.mark.parametrize("n", [6, 8, 12])
def test_qft_closed_form(n):
    # QFT without final swaps of |x>: psi[i] = 2^{-n/2} exp(2 pi i x rev_n(i) / 2^n)
    inst = make_config("c2", twin=True, n=n, n_low=n // 2, seed=11 + n)
    nn, g = _circ(inst.text)
    x = inst.meta["x"]
    cf = np.array([np.exp(2j * np.pi * x * _rev(i, n) / 2 ** n) for i in range(1 << n)]) / 2 ** (n / 2)
    assert np.abs(O.schrodinger(nn, g) - cf).max() < 1e-13
    assert np.abs(O.hsf(nn, g, inst.n_low, inst.blocks) - cf).max() < 1e-13
    P = O.plan(nn, g, inst.n_low, inst.blocks)
    assert P.radices == [2] * (n - n // 2)  # each ladder tail is one rank-2 block


@pytest.mark.parametrize("seed", range(6))
def test_schrodinger_vs_bruteforce_unitary(seed):
    inst = random_small_circuit(seed, n=int(3 + seed % 4), n_gates=14)
    n, g = _circ(inst.text)
    U = O.unitary_bruteforce(n, g)
    assert np.allclose(U.conj().T @ U, np.eye(1 << n), atol=1e-12)
    for init in (0, (1 << n) - 1, 5 % (1 << n)):
        assert np.allclose(O.schrodinger(n, g, init), U[:, init], atol=1e-12)


# ---------------------------------------------------------- Schmidt step
def _single_unit(text, n_low):
    n, g = _circ(text)
    P = O.plan(n, g, n_low, [list(range(len(g)))])
    assert len(P.units) == 1
    return P.units[0], g


def test_schmidt_ranks_individual_gates():
    assert _single_unit("qubits 2\ncx 1 0\n", 1)[0].rank == 2
    assert _single_unit("qubits 2\ncz 1 0\n", 1)[0].rank == 2
    assert _single_unit("qubits 2\nswap 1 0\n", 1)[0].rank == 4  # P:131 (SWAP r = 4)
    assert _single_unit(f"qubits 2\nrzz {0.0.hex()} 1 0\n", 1)[0].rank == 1
    assert _single_unit(f"qubits 2\nrzz {0.7.hex()} 1 0\n", 1)[0].rank == 2


def test_rzz_singular_values_closed_form():
    # RZZ(t) = cos(t/2) I(x)I - i sin(t/2) Z(x)Z; unit-Frobenius factors give
    # sigma = (2|cos t/2|, 2|sin t/2|); unitary-scale coefficients = (|cos|, |sin|)
    t = 0.7
    u, _ = _single_unit(f"qubits 2\nrzz {t.hex()} 1 0\n", 1)
    assert np.allclose(sorted(u.sigmas), sorted([2 * abs(math.cos(t / 2)), 2 * abs(math.sin(t / 2))]), atol=1e-14)
    assert np.allclose(sorted(np.abs(u.c)), sorted([abs(math.cos(t / 2)), abs(math.sin(t / 2))]), atol=1e-14)


def test_product_operator_rank_one():
    txt = "qubits 2\nh 1\nrx %s 0\n" % (0.4).hex()
    n, g = _circ(txt)
    P = O.plan(n, g, 1, [[0, 1]])
    assert P.units[0].rank == 1


def test_cnot_cascade_eq11():
    # Example 4 / Eq. 11: 3-CNOT cascade from control q3 (side a)
    # onto q2,q1,q0 (side b): C = P0(x)I(x)I(x)I + P1(x)X(x)X(x)X, rank 2 (vs 2^3).
    u, g = _single_unit("qubits 4\ncx 3 2\ncx 3 1\ncx 3 0\n", 3)
    assert u.rank == 2
    # the X factors span {P0, P1}; the Y factors span {I, XXX}
    P0 = np.diag([1, 0]).astype(complex)
    P1 = np.diag([0, 1]).astype(complex)
    X1 = np.array([[0, 1], [1, 0]], dtype=complex)
    XXX = np.kron(np.kron(X1, X1), X1)
    basis_a = np.stack([P0.ravel(), P1.ravel()], 1)
    basis_b = np.stack([np.eye(8).ravel(), XXX.ravel()], 1)
    for Xm in u.X:
        coef, *_ = np.linalg.lstsq(basis_a, Xm.ravel(), rcond=None)
        assert np.allclose(basis_a @ coef, Xm.ravel(), atol=1e-12)
    for Ym in u.Y:
        coef, *_ = np.linalg.lstsq(basis_b, Ym.ravel(), rcond=None)
        assert np.allclose(basis_b @ coef, Ym.ravel(), atol=1e-12)
    expect = np.kron(P0, np.eye(8)) + np.kron(P1, XXX)
    assert np.allclose(O.unit_reconstruction(u), expect, atol=1e-12)
    # individually cut: 2^3 paths
    n, gg = _circ("qubits 4\ncx 3 2\ncx 3 1\ncx 3 0\n")
    assert O.plan(n, gg, 3, None, "individual").n_paths == 8


@pytest.mark.parametrize("depth", [1, 2, 4, 8])
def test_joint_rank_saturates_at_16(depth):
    # Example 3 / Eq. 10: a 2+2 block has rank <= 2^(2*2)
    rng = np.random.default_rng(depth)
    lines = ["qubits 4"]
    for _ in range(depth):
        for q in range(4):
            v = rng.standard_normal(4)
            a, b, c, d = v / np.linalg.norm(v)
            lines.append("u 1 %d %s" % (q, " ".join(x.hex() for x in [a, b, c, d, -c, d, a, -b])))
        lines.append("cx 1 2")
        lines.append("cz 0 3")
        lines.append("swap 1 3")
    n, g = _circ("\n".join(lines) + "\n")
    P = O.plan(n, g, 2, [list(range(len(g)))])
    Pi = O.plan(n, g, 2, None, "individual")
    assert P.units[0].rank <= 16
    assert Pi.n_paths == (2 * 2 * 4) ** depth
    if depth >= 2:
        assert P.n_paths < Pi.n_paths


@pytest.mark.parametrize("seed", range(8))
def test_reconstruction_random_blocks(seed):
    inst = random_small_circuit(seed, max_block_qubits=6)
    n, g = _circ(inst.text)
    P = O.plan(n, g, inst.n_low, inst.blocks)
    for u in P.units:
        ref = O.unit_matrix(g, u)
        assert np.linalg.norm(O.unit_reconstruction(u) - ref) <= 1e-12 * np.linalg.norm(ref)
        # Eq. 10 rank bound
        assert u.rank <= min(4 ** len(u.Sa), 4 ** len(u.Sb))
        # unitary block -> sum |c_m|^2 = 1 with unitary-scale factors
        assert abs(np.sum(np.abs(u.c) ** 2) - 1) < 1e-12


def test_nonconvex_block_rejected():
    n, g = _circ("qubits 3\ncx 2 0\nh 0\ncx 2 1\ncx 0 1\n")
    # {g0, g3} with g1 (h 0) between them on qubit 0 and g3 after g1: cycle
    with pytest.raises(O.NonConvexBlock):
        O.plan(n, g, 1, [[0, 3]])


# ------------------------------------------------------------- path sums
@pytest.mark.parametrize("seed", range(30))
def test_joint_equals_individual_equals_schrodinger_random(seed):
    inst = random_small_circuit(seed, n_gates=8 + seed % 17)
    n, g = _circ(inst.text)
    ref = O.schrodinger(n, g)
    P = O.plan(n, g, inst.n_low, inst.blocks)
    if P.n_paths > 1024:
        inst = random_small_circuit(seed, n_gates=8)
        n, g = _circ(inst.text)
        ref = O.schrodinger(n, g)
    joint = O.hsf(n, g, inst.n_low, inst.blocks)
    assert np.abs(joint - ref).max() < 1e-12
    Pi = O.plan(n, g, inst.n_low, None, "individual")
    if Pi.n_paths <= 512:
        ind = O.hsf(n, g, inst.n_low, None, "individual")
        assert np.abs(ind - ref).max() < 1e-12


@pytest.mark.parametrize("name", ["c1", "c3", "c4", "c5"])
def test_configs_twins_match_schrodinger(name):
    inst = make_config(name, twin=True)
    n, g = _circ(inst.text)
    ref = O.schrodinger(n, g)
    P = O.plan(n, g, inst.n_low, inst.blocks)
    A, B, c = O.half_states(P)
    full = O.recombine_full(A, B, c)
    assert np.abs(full - ref).max() < 1e-13
    assert abs(O.gram_norm2(A, B, c) - 1) < 1e-12
    if inst.bitstrings is not None:
        amps = O.recombine_bits(A, B, c, inst.bitstrings, inst.n_low)
        assert np.abs(amps - ref[inst.bitstrings.astype(np.int64)]).max() < 1e-13


def test_c1_full_size_paths():
    inst = make_config("c1")
    n, g = _circ(inst.text)
    P = O.plan(n, g, inst.n_low, inst.blocks)
    Pi = O.plan(n, g, inst.n_low, None, "individual")
    assert (P.n_paths, Pi.n_paths) == (16, 4096)  # BJ configs[0]: <=16 vs 2^12
    ref = O.schrodinger(n, g)
    assert np.abs(O.hsf(n, g, inst.n_low, inst.blocks) - ref).max() < 1e-13


def test_path_counts_full_configs():
    # BJ: c2 2^12 joint; c3 4^4; c4 4^3; c5 2^8 joint vs 2^48 individual
    expect = {"c2": (4096, None), "c3": (256, 256), "c4": (64, 64), "c5": (256, 2 ** 48)}
    for name, (pj, pt) in expect.items():
        inst = make_config(name, n_bits=0) if name in ("c3", "c5") else make_config(name)
        n, g = _circ(inst.text)
        P = O.plan(n, g, inst.n_low, inst.blocks)
        assert P.n_paths == pj, name
        if pt is not None:
            # individual ranks: every crossing gate here has rank 2
            ncross = sum(1 for x in g if O.classify(x.qubits, inst.n_low) == "cross")
            assert 2 ** ncross == pt, name


def test_no_crossing_gates_is_kron():
    rng = np.random.default_rng(3)
    lines = ["qubits 6"]
    for q in range(6):
        v = rng.standard_normal(4)
        a, b, c, d = v / np.linalg.norm(v)
        lines.append("u 1 %d %s" % (q, " ".join(x.hex() for x in [a, b, c, d, -c, d, a, -b])))
    lines += ["cx 0 1", "cz 4 5", "cx 3 4"]
    n, g = _circ("\n".join(lines) + "\n")
    P = O.plan(n, g, 3)
    assert P.n_paths == 1
    A, B, c = O.half_states(P)
    assert np.allclose(O.recombine_full(A, B, c), np.kron(A[:, 0], B[:, 0]), atol=1e-15)
    assert np.abs(O.recombine_full(A, B, c) - O.schrodinger(n, g)).max() < 1e-14


def test_path_ranges_sum_to_whole():
    # partition of the path index (per-GPU ranges) sums to the 1-way result
    inst = make_config("c5", twin=True)
    n, g = _circ(inst.text)
    P = O.plan(n, g, inst.n_low, inst.blocks)
    ref = O.recombine_full(*O.half_states(P))
    for G in (2, 4, 8):
        tot = 0
        for r in range(G):
            p0, p1 = r * P.n_paths // G, (r + 1) * P.n_paths // G
            tot = tot + O.recombine_full(*O.half_states(P, p0, p1))
        assert np.abs(tot - ref).max() < 1e-14


# ------------------------------------------------- paper tables (path counts)
def _table2():
    rows = []
    for line in open(os.path.join(GOLD, "table2_paths.txt")):
        if line.startswith("#") or not line.strip():
            continue
        name, lt, lj, blocks, sep, sepc = line.split()
        rows.append((name, int(lt), int(lj), int(blocks), int(sep), int(sepc)))
    return rows


@pytest.mark.parametrize("row", _table2(), ids=lambda r: r[0])
def test_table2_path_counts(row):
    # Build crossing structure with the paper's counts: `blocks` RZZ cascades
    # holding (sep_cuts - sep) crossing gates plus `sep` separate crossing RZZs.
    # The oracle must reproduce Table I's path counts n_p^j and n_p^t.
    name, lt, lj, blocks, sep, sepc = row
    assert lt == sepc
    in_blocks = sepc - sep
    sizes = [in_blocks // blocks + (1 if i < in_blocks % blocks else 0) for i in range(blocks)]
    nb = 16
    lines, blk = [f"qubits {nb + blocks + sep}"], []
    gi, t = 0, 0
    for i, s in enumerate(sizes):
        ids = []
        for _ in range(s):
            lines.append(f"rzz {0.37.hex()} {t % nb} {nb + i}")
            ids.append(gi)
            gi += 1
            t += 1
        blk.append(ids)
    for j in range(sep):
        lines.append(f"rzz {0.61.hex()} {t % nb} {nb + blocks + j}")
        gi += 1
        t += 1
    n, g = _circ("\n".join(lines) + "\n")
    P = O.plan(n, g, nb, blk)
    Pi = O.plan(n, g, nb, None, "individual")
    assert P.n_paths == 2 ** lj
    assert Pi.n_paths == 2 ** lt


def test_sbm_qaoa_blocks_are_rank2_cascades():
    inst = make_sbm_qaoa(seed=31, sizes=(6, 6), p_inter=0.3)
    n, g = _circ(inst.text)
    P = O.plan(n, g, inst.n_low, inst.blocks)
    for u in P.units:
        assert u.rank == 2
    assert abs(np.linalg.norm(O.hsf(n, g, inst.n_low, inst.blocks)) - 1) < 1e-12
    assert np.abs(O.hsf(n, g, inst.n_low, inst.blocks) - O.schrodinger(n, g)).max() < 1e-13


# ------------------------------------------------- commutation + block finder
def test_interleaved_commuting_block_is_convex():
    # RZZ(1,2) and RZZ(1,3) share qubit 1 with RZZ(0,1) between them: all are
    # diagonal, so the block {g0, g2} is convex after commuting
    txt = ("qubits 4\nh 0\nh 1\nh 2\nh 3\n" + f"rzz {0.3.hex()} 1 2\nrzz {0.5.hex()} 0 1\nrzz {0.7.hex()} 1 3\n"
           + "rx 0.4 0\nrx 0.4 1\nrx 0.4 2\nrx 0.4 3\n").replace("rx 0.4", "rx " + 0.4.hex())
    n, g = _circ(txt)
    P = O.plan(n, g, 2, [[4, 6]])
    assert [u.rank for u in P.units] == [2]  # the cascade centred on qubit 1
    assert np.abs(O.hsf(n, g, 2, [[4, 6]]) - O.schrodinger(n, g)).max() < 1e-14
    # a non-diagonal gate on the shared qubit between them breaks convexity
    n2, g2 = _circ(txt.replace(f"rzz {0.5.hex()} 0 1", "h 1"))
    with pytest.raises(O.NonConvexBlock):
        O.plan(n2, g2, 2, [[4, 6]])


def _brute_min_cover(edge_list):
    verts = sorted({v for e in edge_list for v in e})
    for k in range(len(verts) + 1):
        import itertools
        for cov in itertools.combinations(verts, k):
            c = set(cov)
            if all(a in c or b in c for a, b in edge_list):
                return k
    return len(verts)


@pytest.mark.parametrize("seed", range(12))
def test_find_cascades_minimum_cover_bruteforce(seed):
    # the finder's cascade count is a minimum vertex cover (Koenig), checked
    # by exhaustive search on small random crossing graphs; the planned joint
    # HSF with its blocks reproduces the Schroedinger state
    rng = np.random.default_rng([seed, 11])
    nb, na = 4, 4
    lines = [f"qubits {nb + na}"] + [f"h {q}" for q in range(nb + na)]
    edges = set()
    for _ in range(int(rng.integers(3, 10))):
        b, a = int(rng.integers(nb)), int(nb + rng.integers(na))
        edges.add((b, a))
        lines.append(f"rzz {float(rng.uniform(0, 3)).hex()} {b} {a}")
    lines += [f"rx {0.3.hex()} {q}" for q in range(nb + na)]
    n, g = _circ("\n".join(lines) + "\n")
    blocks, ncasc = O.find_cascades(g, nb)
    assert ncasc == _brute_min_cover(sorted(edges))
    P = O.plan(n, g, nb, blocks)
    assert all(u.rank <= 2 for u in P.units)
    assert P.n_paths == 2 ** ncasc
    assert np.abs(O.hsf(n, g, nb, blocks) - O.schrodinger(n, g)).max() < 1e-13


@pytest.mark.parametrize("row", _table2(), ids=lambda r: r[0])
def test_table2_counts_from_block_finder(row):
    # Table I/II structure (blocks + separate RZZ cuts) rebuilt as a circuit
    # with the gates in file order scattered: the automatic finder recovers
    # n_p^j = 2^(blocks + sep)
    name, lt, lj, blocks, sep, sepc = row
    in_blocks = sepc - sep
    sizes = [in_blocks // blocks + (1 if i < in_blocks % blocks else 0) for i in range(blocks)]
    nb = 40
    gl, t = [], 0
    for i, sz in enumerate(sizes):
        for _ in range(sz):
            gl.append((t, nb + i))
            t += 1
    for j in range(sep):
        gl.append((t, nb + blocks + j))
        t += 1
    rng = np.random.default_rng(len(gl))
    rng.shuffle(gl)
    lines = [f"qubits {nb + blocks + sep}"] + [f"rzz {0.37.hex()} {b} {a}" for b, a in gl]
    n, g = _circ("\n".join(lines) + "\n")
    found, ncasc = O.find_cascades(g, nb)
    assert ncasc == lj
    assert len(found) == blocks


@pytest.mark.parametrize("procs", [1, 3])
def test_parallel_driver_matches_direct(procs):
    # oracle/parallel.py: forked workers running simulate_path on path chunks,
    # sampled rows only -> recombine_bits; must equal the direct naive HSF
    from oracle import parallel as OP
    inst = make_config("c5", twin=True)
    n, g = O.parse_circuit(inst.text)
    P = O.plan(n, g, inst.n_low, inst.blocks)
    bits = np.concatenate([inst.bitstrings[:500], inst.bitstrings[:50]])
    ref = O.hsf(n, g, inst.n_low, inst.blocks, bits=bits)
    got = OP.bits_amplitudes(P, bits, inst.n_low, procs=procs)
    assert np.abs(got - ref).max() <= 1e-14
    A, B, c = OP.half_state_rows(P, [0, 3], [1], 2, 7, procs=procs)
    A2, B2, c2 = O.half_states(P, 2, 7)
    assert np.array_equal(A, A2[[0, 3]]) and np.array_equal(B, B2[[1]]) and np.array_equal(c, c2)
