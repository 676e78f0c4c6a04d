"""CPU oracle for joint-cut Hybrid Schroedinger-Feynman (HSF) simulation.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this module.
The product path (`paper_2502_06959_b200`, `libhsf.so`) never imports, links
or calls it; the two share no code (only the circuit-file format written by
`hsf_inputs`).

Plain, slow, obviously-correct complex128 NumPy, in the order and notation of
arXiv 2502.06959 (PAPER.md; line numbers "P:n"):

  * Schroedinger-style simulation: consecutive gate matrix-vector products on
    the 2^n statevector (Example 1 P:53-63).
  * HSF: horizontal partition into halves a (high qubits) and b (low qubits),
    every crossing gate / jointly-cut block replaced by its Schmidt
    decomposition A = sum_m sigma_m X_m (x) Y_m (Eq. 4); each choice
    of one term per cut unit is a "path"; n_p = prod r_i; the result is
    the sum over paths of the Kronecker products of the two half-states
    (P:109).
  * Joint cutting: gates of a block are multiplied first, then the block is
    Schmidt-decomposed by reshaping / matricising (Eq. 5-6,
    P:163-172), an SVD (Eq. 7) and absorbing U, V* into the factors
    (Eq. 8-9).

Readings where the paper is silent: qubit 0 = LSB;
half A = high qubits [n_low, n) = the paper's partition a; first-listed gate
qubit = MSB of the gate-local index; block-local index LSB = smallest support
qubit; singular values <= 1e-12 * sigma_0 dropped; factors rescaled to unitary
scale (X * sqrt(2^|S_a|), Y * sqrt(2^|S_b|), c = sigma / sqrt(2^|S|)).

Parity status: every function below is pinned by tests/test_oracle.py against
closed forms, paper examples, brute force or invariants.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

SVD_REL_TOL = 1e-12


# ----------------------------------------------------------------- gate library
def gate_matrix(name: str, params, k: int, payload=None) -> np.ndarray:
    """Dense 2^k x 2^k matrix; first-listed qubit = most significant local bit."""
    if name == "h":
        return np.array([[1, 1], [1, -1]], dtype=complex) / math.sqrt(2.0)
    if name == "x":
        return np.array([[0, 1], [1, 0]], dtype=complex)
    if name == "z":
        return np.array([[1, 0], [0, -1]], dtype=complex)
    if name == "rx":
        t = params[0]
        c, s = math.cos(t / 2), math.sin(t / 2)
        return np.array([[c, -1j * s], [-1j * s, c]], dtype=complex)
    if name == "rz":
        t = params[0]
        return np.diag([np.exp(-0.5j * t), np.exp(0.5j * t)])
    if name == "cz":
        return np.diag([1, 1, 1, -1]).astype(complex)
    if name == "cx":
        # PAPER.md Example 2: CNOT = P0 (x) I + P1 (x) X, control first
        P0 = np.array([[1, 0], [0, 0]], dtype=complex)
        P1 = np.array([[0, 0], [0, 1]], dtype=complex)
        return np.kron(P0, np.eye(2)) + np.kron(P1, gate_matrix("x", (), 1))
    if name == "swap":
        m = np.zeros((4, 4), dtype=complex)
        m[0, 0] = m[3, 3] = m[1, 2] = m[2, 1] = 1
        return m
    if name == "cp":
        return np.diag([1, 1, 1, np.exp(1j * params[0])])
    if name == "rzz":
        # RZZ(theta) = exp(-i theta/2 Z (x) Z)
        t = params[0]
        a, b = np.exp(-0.5j * t), np.exp(0.5j * t)
        return np.diag([a, b, b, a])
    if name == "u":
        d = 1 << k
        v = np.asarray(payload, dtype=float).reshape(d, d, 2)
        return v[..., 0] + 1j * v[..., 1]
    raise ValueError(f"unsupported gate {name!r}")


@dataclass
class Gate:
    name: str
    params: tuple
    qubits: tuple  # first-listed = MSB of U's index
    U: np.ndarray

    @property
    def diagonal(self) -> bool:
        return bool(np.all(self.U == np.diag(np.diag(self.U))))


_ARITY = {"h": (0, 1), "x": (0, 1), "z": (0, 1), "rx": (1, 1), "rz": (1, 1), "cz": (0, 2), "cx": (0, 2),
          "swap": (0, 2), "cp": (1, 2), "rzz": (1, 2)}


def parse_circuit(text: str):
    """Circuit file -> (n, [Gate]).  Format: hsf_inputs/circuits.py docstring."""
    n = None
    gates = []
    for lineno, raw in enumerate(text.splitlines(), 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        tok = line.split()
        if tok[0] == "qubits":
            n = int(tok[1])
            continue
        if n is None:
            raise ValueError(f"line {lineno}: gate before 'qubits'")
        name = tok[0]
        if name == "u":
            k = int(tok[1])
            qs = tuple(int(t) for t in tok[2:2 + k])
            payload = [float.fromhex(t) for t in tok[2 + k:]]
            if len(payload) != 2 * (1 << (2 * k)):
                raise ValueError(f"line {lineno}: bad payload length")
            params = ()
        else:
            npar, nq = _ARITY[name]
            params = tuple(float.fromhex(t) for t in tok[1:1 + npar])
            qs = tuple(int(t) for t in tok[1 + npar:1 + npar + nq])
            payload = None
            k = nq
        if len(set(qs)) != len(qs) or any(not (0 <= q < n) for q in qs):
            raise ValueError(f"line {lineno}: bad qubits {qs}")
        gates.append(Gate(name, params, qs, gate_matrix(name, params, k, payload)))
    return n, gates


# ------------------------------------------------------- Schroedinger-style sim
def apply_gate(psi: np.ndarray, m: int, U: np.ndarray, qubits) -> np.ndarray:
    """psi' = U_embedded psi on an m-qubit vector.  psi is viewed as a
    (2,)*m tensor whose axis t holds qubit m-1-t; first-listed qubit of U is
    its most significant index."""
    k = len(qubits)
    t = psi.reshape((2,) * m)
    axes = [m - 1 - q for q in qubits]
    Ut = U.reshape((2,) * (2 * k))
    out = np.tensordot(Ut, t, axes=(list(range(k, 2 * k)), axes))
    # tensordot puts the k new axes first; move them back to `axes`
    out = np.moveaxis(out, list(range(k)), axes)
    return out.reshape(-1)


def schrodinger(n: int, gates, init_index: int = 0) -> np.ndarray:
    """Full statevector U_circuit |init>  (Sec. II-A, Example 1)."""
    psi = np.zeros(1 << n, dtype=complex)
    psi[init_index] = 1.0
    for g in gates:
        psi = apply_gate(psi, n, g.U, g.qubits)
    return psi


def unitary_bruteforce(n: int, gates) -> np.ndarray:
    """Full 2^n x 2^n circuit unitary built column by column from the gate
    definitions with explicit bit manipulation (independent of apply_gate)."""
    N = 1 << n
    total = np.eye(N, dtype=complex)
    for g in gates:
        k = len(g.qubits)
        E = np.zeros((N, N), dtype=complex)
        for j in range(N):
            jl = 0
            for q in g.qubits:  # first-listed = MSB
                jl = (jl << 1) | ((j >> q) & 1)
            for il in range(1 << k):
                i = j
                for pos, q in enumerate(g.qubits):
                    bit = (il >> (k - 1 - pos)) & 1
                    i = (i & ~(1 << q)) | (bit << q)
                E[i, j] += g.U[il, jl]
        total = E @ total
    return total


# ------------------------------------------------------------------ HSF planner
def classify(qubits, n_low: int) -> str:
    """LocalLow / LocalHigh / Crossing."""
    lo = [q < n_low for q in qubits]
    if all(lo):
        return "low"
    if not any(lo):
        return "high"
    return "cross"


@dataclass
class Unit:
    gate_ids: list
    support: list  # sorted ascending
    Sa: list  # high-side support (global qubit ids)
    Sb: list  # low-side support
    sigmas: np.ndarray
    c: np.ndarray  # rank r, complex coefficient per term
    X: list  # r matrices on Sa (local index LSB = smallest qubit)
    Y: list  # r matrices on Sb
    diagonal_route: bool

    @property
    def rank(self) -> int:
        return len(self.c)


class NonConvexBlock(ValueError):
    pass


def _is_diagonal(U) -> bool:
    return bool(np.count_nonzero(U - np.diag(np.diag(U))) == 0)


def _schedule(gates, n_low, units_gate_ids):
    """Contract each unit in the gate-dependency DAG and Kahn-sort (ties:
    smallest gate id).  Returns [("gate", gid) | ("unit", uid)]; raises
    NonConvexBlock on a cycle.

    Dependencies follow commutation: an op depends on every earlier op on a
    shared qubit unless both are diagonal (diagonal operators commute), so a
    block of mutually commuting diagonal gates (the paper's RZZ cascades, which
    "mutually commute, which gives a lot of freedom to reorder the gates such
    that grouping ... can be performed") is convex however the
    commuting gates are interleaved in the file."""
    owner = {}
    for u, ids in enumerate(units_gate_ids):
        for gi in ids:
            owner[gi] = ("unit", u)
    nodes = {}
    for gi in range(len(gates)):
        key = owner.get(gi, ("gate", gi))
        nodes.setdefault(key, []).append(gi)
    succ = {k: set() for k in nodes}
    indeg = {k: 0 for k in nodes}
    last_nd = {}   # qubit -> node of the last non-diagonal gate
    diags = {}     # qubit -> nodes of diagonal gates since then
    for gi, g in enumerate(gates):
        key = owner.get(gi, ("gate", gi))
        diag = _is_diagonal(g.U)
        deps = set()
        for q in g.qubits:
            if q in last_nd:
                deps.add(last_nd[q])
            if not diag:
                deps.update(diags.get(q, ()))
        for d in deps:
            if d != key and key not in succ[d]:
                succ[d].add(key)
                indeg[key] += 1
        for q in g.qubits:
            if diag:
                diags.setdefault(q, set()).add(key)
            else:
                last_nd[q] = key
                diags[q] = set()
    import heapq
    heap = [(min(nodes[k]), k) for k in nodes if indeg[k] == 0]
    heapq.heapify(heap)
    order = []
    while heap:
        _, k = heapq.heappop(heap)
        order.append(k)
        for s in succ[k]:
            indeg[s] -= 1
            if indeg[s] == 0:
                heapq.heappush(heap, (min(nodes[s]), s))
    if len(order) != len(nodes):
        raise NonConvexBlock("block is not convex in the wire DAG")
    return order


def _embed(U, gate_qubits, support):
    """Embed a gate into the block-local space (bit t <-> support[t])."""
    kS = len(support)
    pos = [support.index(q) for q in gate_qubits]
    k = len(gate_qubits)
    N = 1 << kS
    E = np.zeros((N, N), dtype=complex)
    for j in range(N):
        jl = 0
        for p in pos:
            jl = (jl << 1) | ((j >> p) & 1)
        for il in range(1 << k):
            i = j
            for t, p in enumerate(pos):
                bit = (il >> (k - 1 - t)) & 1
                i = (i & ~(1 << p)) | (bit << p)
            E[i, j] += U[il, jl]
    return E


def schmidt_unit(gates, gate_ids, n_low, rel_tol=SVD_REL_TOL) -> Unit:
    """Joint cut of one block: assemble, reshape (Eq. 5-6), SVD (Eq. 7), absorb
    U and V* into X_m, Y_m (Eq. 8-9), drop sigma_m <= rel_tol*sigma_0, rescale."""
    support = sorted({q for gi in gate_ids for q in gates[gi].qubits})
    Sb = [q for q in support if q < n_low]
    Sa = [q for q in support if q >= n_low]
    nb, na = len(Sb), len(Sa)
    members = [gates[gi] for gi in gate_ids]
    diag = all(g.diagonal for g in members)
    if diag:
        # diagonal route: u(i) = prod of member diagonal entries; the SVD of the
        # 2^nb x 2^na matrix M[i^b, i^a] is the operator-Schmidt decomposition of
        # a diagonal operator with diagonal factors.
        N = 1 << len(support)
        d = np.ones(N, dtype=complex)
        for g in members:
            dg = np.diag(g.U)
            pos = [support.index(q) for q in g.qubits]
            for i in range(N):
                il = 0
                for p in pos:
                    il = (il << 1) | ((i >> p) & 1)
                d[i] *= dg[il]
        M = np.zeros((1 << nb, 1 << na), dtype=complex)
        for i in range(N):
            M[i & ((1 << nb) - 1), i >> nb] = d[i]
        Uu, s, Vh = np.linalg.svd(M)
        keep = s > rel_tol * s[0]
        X = [np.diag(Vh[m, :]) for m in range(len(s)) if keep[m]]
        Y = [np.diag(Uu[:, m]) for m in range(len(s)) if keep[m]]
    else:
        US = np.eye(1 << len(support), dtype=complex)
        for g in members:  # circuit order: later gates multiply from the left
            US = _embed(g.U, g.qubits, support) @ US
        # A~[(i^b, j^b), (i^a, j^a)] = U_S[(i^a, i^b), (j^a, j^b)]   (Eq. 6)
        T = US.reshape(1 << na, 1 << nb, 1 << na, 1 << nb)  # [i^a, i^b, j^a, j^b]
        At = T.transpose(1, 3, 0, 2).reshape(1 << (2 * nb), 1 << (2 * na))
        Uu, s, Vh = np.linalg.svd(At, full_matrices=False)  # Eq. 7
        keep = s > rel_tol * s[0]
        # Eq. 8-9: X_m = sum V*_{m,(i^a,j^a)} |i^a><j^a|, Y_m = sum U_{(i^b,j^b),m} |i^b><j^b|
        X = [Vh[m, :].reshape(1 << na, 1 << na) for m in range(len(s)) if keep[m]]
        Y = [Uu[:, m].reshape(1 << nb, 1 << nb) for m in range(len(s)) if keep[m]]
    s = s[keep]
    sa, sb = math.sqrt(1 << na), math.sqrt(1 << nb)
    X = [x * sa for x in X]
    Y = [y * sb for y in Y]
    c = s / (sa * sb)
    return Unit(list(gate_ids), support, Sa, Sb, s, c.astype(complex), X, Y, diag)


@dataclass
class Plan:
    n: int
    n_low: int
    gates: list
    units: list
    order: list  # schedule

    @property
    def n_a(self):
        return self.n - self.n_low

    @property
    def radices(self):
        return [u.rank for u in self.units]

    @property
    def n_paths(self) -> int:
        return int(np.prod(self.radices, dtype=object)) if self.units else 1


def plan(n, gates, n_low, blocks=None, mode="joint") -> Plan:
    """Classify, form units: joint mode -> user blocks + singleton
    crossing gates; individual mode -> every crossing gate alone."""
    if not (1 <= n_low < n):
        raise ValueError("cut must leave both halves non-empty")
    blocks = blocks or []
    units_ids = []
    in_block = set()
    if mode == "joint":
        for b in blocks:
            units_ids.append(sorted(b))
            in_block.update(b)
    for gi, g in enumerate(gates):
        if gi not in in_block and classify(g.qubits, n_low) == "cross":
            units_ids.append([gi])
    order = _schedule(gates, n_low, units_ids)
    # units numbered in schedule order
    sched_units = [k[1] for k in order if k[0] == "unit"]
    units = [schmidt_unit(gates, units_ids[u], n_low) for u in sched_units]
    remap = {u: i for i, u in enumerate(sched_units)}
    order = [("unit", remap[k[1]]) if k[0] == "unit" else k for k in order]
    return Plan(n, n_low, gates, units, order)


def find_cascades(gates, n_low):
    """Automatic joint blocks: cascades of commuting diagonal
    two-qubit crossing gates sharing one qubit, as few as possible.

    Each such gate is an edge between its low and high qubit, each tagged with
    its epoch (count of earlier non-diagonal gates on that qubit); a minimum
    vertex cover of this bipartite multigraph (networkx Hopcroft-Karp matching
    + Koenig's theorem, a library primitive) is a smallest set of cascade
    centres.  Returns (blocks with >= 2 gates, number of cascades)."""
    import networkx as nx
    from networkx.algorithms import bipartite
    epoch = {}
    G = nx.Graph()
    edges = []
    for gi, g in enumerate(gates):
        if len(g.qubits) == 2 and _is_diagonal(g.U):
            b, a = sorted(g.qubits)
            if b < n_low <= a:
                lb, ra = ("L", b, epoch.get(b, 0)), ("R", a, epoch.get(a, 0))
                G.add_node(lb, bipartite=0)
                G.add_node(ra, bipartite=1)
                G.add_edge(lb, ra)
                edges.append((gi, lb, ra))
        if not _is_diagonal(g.U):
            for q in g.qubits:
                epoch[q] = epoch.get(q, 0) + 1
    if not edges:
        return [], 0
    left = {v for v in G if v[0] == "L"}
    matching = bipartite.hopcroft_karp_matching(G, top_nodes=left)
    cover = bipartite.to_vertex_cover(G, matching, top_nodes=left)
    groups = {}
    for gi, lb, ra in edges:
        key = lb if lb in cover else ra
        groups.setdefault(key, []).append(gi)
    blocks = sorted(sorted(v) for v in groups.values() if len(v) >= 2)
    return blocks, len(cover)


# ----------------------------------------------------------------- path engine
def path_digits(p: int, radices) -> list:
    """Mixed radix, last unit fastest."""
    d = [0] * len(radices)
    for u in range(len(radices) - 1, -1, -1):
        d[u] = p % radices[u]
        p //= radices[u]
    return d


def simulate_path(P: Plan, p: int):
    """One Feynman path: both half-circuits from |0...0>, each unit applying
    its chosen Schmidt term.  Returns (psi_A, psi_B, c_p)."""
    nb, na = P.n_low, P.n_a
    dig = path_digits(p, P.radices)
    a = np.zeros(1 << na, dtype=complex)
    a[0] = 1
    b = np.zeros(1 << nb, dtype=complex)
    b[0] = 1
    c = 1.0 + 0j
    for kind, idx in P.order:
        if kind == "gate":
            g = P.gates[idx]
            cls = classify(g.qubits, nb)
            if cls == "low":
                b = apply_gate(b, nb, g.U, g.qubits)
            elif cls == "high":
                a = apply_gate(a, na, g.U, tuple(q - nb for q in g.qubits))
            else:
                raise AssertionError("crossing gate outside a unit")
        else:
            u = P.units[idx]
            m = dig[idx]
            # local matrices have LSB = smallest support qubit -> list qubits MSB first
            b = apply_gate(b, nb, u.Y[m], tuple(reversed(u.Sb)))
            a = apply_gate(a, na, u.X[m], tuple(q - nb for q in reversed(u.Sa)))
            c *= u.c[m]
    return a, b, c


def half_states(P: Plan, p0: int = 0, p1: int | None = None):
    """Psi_A (2^nA x K), Psi_B (2^nB x K), c (K) for paths [p0, p1)."""
    p1 = P.n_paths if p1 is None else p1
    K = p1 - p0
    A = np.zeros((1 << P.n_a, K), dtype=complex)
    B = np.zeros((1 << P.n_low, K), dtype=complex)
    c = np.zeros(K, dtype=complex)
    for j, p in enumerate(range(p0, p1)):
        A[:, j], B[:, j], c[j] = simulate_path(P, p)
    return A, B, c


def recombine_full(A, B, c) -> np.ndarray:
    """psi[i_A * 2^nB + i_B] = sum_p c_p A[i_A,p] B[i_B,p]  (Kronecker sum)."""
    return ((A * c[None, :]) @ B.T).reshape(-1)


def recombine_bits(A, B, c, bits, n_low) -> np.ndarray:
    """Amplitudes for a bitstring set (bit q = qubit q), in input order."""
    bits = np.asarray(bits, dtype=np.uint64)
    ia = (bits >> np.uint64(n_low)).astype(np.int64)
    ib = (bits & np.uint64((1 << n_low) - 1)).astype(np.int64)
    out = np.empty(len(bits), dtype=complex)
    Ac = A * c[None, :]
    for s0 in range(0, len(bits), 1 << 14):
        s1 = min(len(bits), s0 + (1 << 14))
        out[s0:s1] = np.einsum("sk,sk->s", Ac[ia[s0:s1]], B[ib[s0:s1]])
    return out


def hsf(n, gates, n_low, blocks=None, mode="joint", bits=None, p0=0, p1=None):
    """Naive HSF: plan, every path from scratch, Kronecker recombination."""
    P = plan(n, gates, n_low, blocks, mode)
    A, B, c = half_states(P, p0, p1)
    if bits is None:
        return recombine_full(A, B, c)
    return recombine_bits(A, B, c, bits, n_low)


def gram_norm2(A, B, c) -> float:
    """||psi||^2 = sum_{p,q} c_p conj(c_q) <A_q|A_p> <B_q|B_p>, without forming psi."""
    GA = A.conj().T @ A
    GB = B.conj().T @ B
    return float(np.real(np.sum(np.conj(c)[:, None] * c[None, :] * GA * GB)))


def unit_reconstruction(u: Unit) -> np.ndarray:
    """sum_m c_m X_m (x) Y_m in block-local index order (high side = MSB part)."""
    tot = 0
    for m in range(u.rank):
        tot = tot + u.c[m] * np.kron(u.X[m], u.Y[m])
    return tot


def unit_matrix(gates, u: Unit) -> np.ndarray:
    """Dense block matrix in block-local order (LSB = smallest support qubit),
    rebuilt from scratch by products of embedded member gates."""
    US = np.eye(1 << len(u.support), dtype=complex)
    for gi in u.gate_ids:
        US = _embed(gates[gi].U, gates[gi].qubits, u.support) @ US
    return US
