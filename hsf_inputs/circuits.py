"""Seeded circuit generators for the five BASELINE.json configs (c1..c5), their
small "twins", a paper-shaped SBM-QAOA family, and random small circuits.

Circuit text format (one item per line; shared by the oracle and the C ABI):

    qubits <n>
    h q | x q | z q
    cz a b | cx a b | swap a b            (cx: first-listed qubit = control)
    cp <theta> a b | rzz <theta> a b | rx <theta> q | rz <theta> q
    u <k> q_1 .. q_k <2*4^k reals>        (row-major, re/im interleaved,
                                           first-listed qubit = most significant
                                           bit of the gate-local index)

Every real is written with ``float.hex`` so both sides read bit-identical
values.  Qubit 0 is the least significant bit of a basis index (PAPER.md
Sec. II-A, i=(i_{n-1},...,i_0)).  The cut is given out of band as ``n_low``:
half B = qubits [0, n_low), half A = [n_low, n).

Draw order: ``numpy.random.default_rng(seed)``
in gate-emission order; bitstrings from ``default_rng([seed, 1])``.
Nothing here evaluates a gate or a state.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Instance:
    name: str
    n: int
    n_low: int
    gates: list  # (name, params tuple, qubits tuple, payload list-of-reals or None)
    blocks: list  # list of lists of gate indices (joint-cut grouping)
    bitstrings: np.ndarray | None = None  # uint64, bit q = qubit q; None => full output
    dtype: str = "c64"
    meta: dict = field(default_factory=dict)

    @property
    def text(self) -> str:
        return serialize(self.n, self.gates)


def _hx(v: float) -> str:
    return float(v).hex()


def serialize(n: int, gates) -> str:
    lines = [f"qubits {n}"]
    for name, params, qubits, payload in gates:
        if name == "u":
            k = len(qubits)
            lines.append(
                "u %d %s %s" % (k, " ".join(str(q) for q in qubits), " ".join(_hx(x) for x in payload))
            )
        else:
            ps = " ".join(_hx(p) for p in params)
            qs = " ".join(str(q) for q in qubits)
            lines.append(f"{name} {ps} {qs}".replace("  ", " ").strip())
    return "\n".join(lines) + "\n"


def _haar_su2(rng) -> list:
    """Haar SU(2): normalised 4-Gaussian (a,b,c,d) -> [[a+ib, c+id], [-c+id, a-ib]]."""
    v = rng.standard_normal(4)
    a, b, c, d = v / np.linalg.norm(v)
    # row-major, re/im interleaved
    return [a, b, c, d, -c, d, a, -b]


def _u1(q, rng):
    return ("u", (), (q,), _haar_su2(rng))


def _bitstrings(seed, n, count):
    rng = np.random.default_rng([seed, 1])
    if n >= 64:
        raise ValueError("n < 64 required")
    return rng.integers(0, 1 << n, size=count, dtype=np.uint64)


def _convex_closure(gates, seeds):
    """Gates lying on a wire-DAG path between two members of `seeds`."""
    order = len(gates)
    succ = [set() for _ in range(order)]
    last = {}
    for i, (_, _, qs, _) in enumerate(gates):
        for q in qs:
            if q in last:
                succ[last[q]].add(i)
            last[q] = i
    seeds = set(seeds)
    lo, hi = min(seeds), max(seeds)

    def reach_from(starts):
        seen = set(starts)
        stack = list(starts)
        while stack:
            g = stack.pop()
            for s in succ[g]:
                if s <= hi and s not in seen:
                    seen.add(s)
                    stack.append(s)
        return seen

    down = reach_from(seeds)
    # reverse reachability
    pred = [set() for _ in range(order)]
    for i in range(order):
        for s in succ[i]:
            pred[s].add(i)
    up = set(seeds)
    stack = list(seeds)
    while stack:
        g = stack.pop()
        for p in pred[g]:
            if p >= lo and p not in up:
                up.add(p)
                stack.append(p)
    return sorted(down & up)


# --------------------------------------------------------------------------- c1
def make_c1(seed: int = 1, n: int = 12, n_low: int = 6, layers: int = 4, n_targets: int = 3) -> Instance:
    """BJ configs[0]: H on all, then `layers` x [Haar SU(2) on all -> CZ on
    even-odd pairs inside each half -> block of CP(theta) sharing control
    n_low-1 with targets n_low..n_low+n_targets-1].  complex128, full output."""
    rng = np.random.default_rng(seed)
    g = [("h", (), (q,), None) for q in range(n)]
    blocks = []
    for _ in range(layers):
        for q in range(n):
            g.append(_u1(q, rng))
        for a in range(0, n - 1, 2):
            if (a < n_low) == (a + 1 < n_low):
                g.append(("cz", (), (a, a + 1), None))
        blk = []
        for t in range(n_low, n_low + n_targets):
            blk.append(len(g))
            g.append(("cp", (rng.uniform(0, 2 * math.pi),), (n_low - 1, t), None))
        blocks.append(blk)
    return Instance("c1", n, n_low, g, blocks, None, "c128", {"seed": seed})


# --------------------------------------------------------------------------- c2
def make_c2(seed: int = 2, n: int = 24, n_low: int = 12) -> Instance:
    """BJ configs[1]: QFT (no final swaps) on a seeded random basis state x.
    For j = n-1..0: H(j); CP(pi/2^(j-k))(j,k), k = j-1..0.  Block per ladder
    j >= n_low: its crossing tail {CP(j,k): k < n_low}.  complex64, full output."""
    rng = np.random.default_rng(seed)
    x = int(rng.integers(0, 1 << n))
    g = [("x", (), (q,), None) for q in range(n) if (x >> q) & 1]
    blocks = []
    for j in range(n - 1, -1, -1):
        g.append(("h", (), (j,), None))
        blk = []
        for k in range(j - 1, -1, -1):
            if j >= n_low and k < n_low:
                blk.append(len(g))
            g.append(("cp", (math.pi / (1 << (j - k)),), (j, k), None))
        if blk:
            blocks.append(blk)
    return Instance("c2", n, n_low, g, blocks, None, "c64", {"seed": seed, "x": x})


# --------------------------------------------------------------------------- c3
def make_c3(seed: int = 3, n: int = 30, n_low: int = 15, depth: int = 16, n_bits: int = 1 << 20,
            window: int = 4) -> Instance:
    """BJ configs[2]: brickwork, layer L = Haar SU(2) on all, then CZ(a,a+1)
    for a = L mod 2, step 2.  The crossing CZ(n_low-1, n_low) gates are grouped
    pairwise (each pair within `window` layers) into blocks = convex closure of
    the pair.  complex64, amplitudes of `n_bits` iid uniform bitstrings."""
    rng = np.random.default_rng(seed)
    g = []
    crossing = []
    for L in range(depth):
        for q in range(n):
            g.append(_u1(q, rng))
        for a in range(L % 2, n - 1, 2):
            if a == n_low - 1:
                crossing.append((L, len(g)))
            g.append(("cz", (), (a, a + 1), None))
    blocks = []
    # group crossing gates whose layers fall in the same window of `window` layers
    groups = {}
    for L, gi in crossing:
        groups.setdefault(L // window, []).append(gi)
    for _, seeds in sorted(groups.items()):
        blocks.append(_convex_closure(g, seeds))
    bits = _bitstrings(seed, n, n_bits) if n_bits else None
    return Instance("c3", n, n_low, g, blocks, bits, "c64", {"seed": seed})


# --------------------------------------------------------------------------- c4
def make_c4(seed: int = 4, n: int = 34, n_low: int = 17, p: int = 3) -> Instance:
    """BJ configs[3]: QAOA-style p-layer ring.  H on all; per layer RZZ(gamma_l)
    on every ring edge (crossing edges (n_low-1,n_low) and (n-1,0) emitted last,
    adjacent) then RX(beta_l) on all; gamma, beta ~ U[0, pi).  One block per
    layer = its two crossing RZZ.  complex64, full output."""
    rng = np.random.default_rng(seed)
    g = [("h", (), (q,), None) for q in range(n)]
    blocks = []
    for _ in range(p):
        gamma = rng.uniform(0, math.pi)
        beta = rng.uniform(0, math.pi)
        for i in range(n - 1):
            if i != n_low - 1:
                g.append(("rzz", (gamma,), (i, i + 1), None))
        blk = [len(g), len(g) + 1]
        g.append(("rzz", (gamma,), (n_low - 1, n_low), None))
        g.append(("rzz", (gamma,), (n - 1, 0), None))
        blocks.append(blk)
        for q in range(n):
            g.append(("rx", (beta,), (q,), None))
    return Instance("c4", n, n_low, g, blocks, None, "c64", {"seed": seed})


# --------------------------------------------------------------------------- c5
def make_c5(seed: int = 5, n: int = 40, n_low: int = 20, layers: int = 8, fanout: int = 6,
            n_bits: int = 1 << 22) -> Instance:
    """BJ configs[4]: per layer Haar SU(2) on all, then one CP(theta) fan-out
    block: a uniform control in half A drives CP to `fanout` distinct uniform
    targets in half B.  complex64, amplitudes of `n_bits` iid bitstrings."""
    rng = np.random.default_rng(seed)
    g = []
    blocks = []
    for _ in range(layers):
        for q in range(n):
            g.append(_u1(q, rng))
        ctrl = int(rng.integers(n_low, n))
        targets = rng.choice(n_low, size=fanout, replace=False)
        blk = []
        for t in targets:
            blk.append(len(g))
            g.append(("cp", (rng.uniform(0, 2 * math.pi),), (ctrl, int(t)), None))
        blocks.append(blk)
    bits = _bitstrings(seed, n, n_bits) if n_bits else None
    return Instance("c5", n, n_low, g, blocks, bits, "c64", {"seed": seed})


# ------------------------------------------------------- paper-shaped SBM QAOA
def make_sbm_qaoa(seed: int = 30, sizes=(15, 15), p_intra: float = 0.8, p_inter: float = 0.1,
                  n_bits: int = 0) -> Instance:
    """Single-layer QAOA MaxCut on a two-community stochastic-block-model graph
    (Sec. V, Table II shapes).  Problem layer RZZ(gamma) per edge,
    mixer RX(beta); crossing edges are emitted grouped by their high-side
    vertex so each group is a commuting RZZ cascade -> one joint block (rank 2).
    A synthetic stand-in: the paper's instances and seeds are unpublished."""
    rng = np.random.default_rng(seed)
    nb, na = sizes
    n = nb + na
    gamma = rng.uniform(0, math.pi)
    beta = rng.uniform(0, math.pi)
    intra, inter = [], {}
    for i in range(n):
        for j in range(i + 1, n):
            same = (i < nb) == (j < nb)
            if rng.uniform() < (p_intra if same else p_inter):
                if same:
                    intra.append((i, j))
                else:
                    inter.setdefault(j, []).append(i)  # j in A (high), i in B
    g = [("h", (), (q,), None) for q in range(n)]
    for (i, j) in intra:
        g.append(("rzz", (gamma,), (i, j), None))
    blocks = []
    for a in sorted(inter):
        blk = []
        for b in inter[a]:
            blk.append(len(g))
            g.append(("rzz", (gamma,), (b, a), None))
        if len(blk) > 1:
            blocks.append(blk)
    for q in range(n):
        g.append(("rx", (beta,), (q,), None))
    bits = _bitstrings(seed, n, n_bits) if n_bits else None
    return Instance(f"sbm{n}", n, nb, g, blocks, bits, "c64", {"seed": seed})


# ------------------------------------------- Table II-shaped QAOA (NEXT row 1)
# PAPER.md Table II: single-layer QAOA MaxCut on two-community
# stochastic-block-model graphs, p_intra 0.8, cut after the first partition,
# output = the first 10^6 amplitudes.  Synthetic stand-ins:
# same shapes, our seeds (the paper's graphs are unpublished).  Blocks are
# found by the planner ("auto").
TABLE2 = {
    "q30-1": ((15, 15), 0.10), "q30-2": ((15, 15), 0.15), "q30-3": ((15, 15), 0.17),
    "q31-1": ((15, 16), 0.10), "q31-2": ((15, 16), 0.15), "q31-3": ((15, 16), 0.17),
    "q32-1": ((16, 16), 0.10), "q32-2": ((16, 16), 0.11), "q32-3": ((16, 16), 0.12),
    "q33-1": ((16, 17), 0.10), "q33-2": ((16, 17), 0.11), "q33-3": ((16, 17), 0.12),
}


def make_table2(name: str, seed: int | None = None, prefix: int = 10 ** 6) -> Instance:
    sizes, p_inter = TABLE2[name]
    idx = sorted(TABLE2).index(name)
    inst = make_sbm_qaoa(seed=3000 + idx if seed is None else seed, sizes=sizes, p_intra=0.8, p_inter=p_inter)
    inst.name = name
    inst.blocks = "auto"
    inst.meta.update({"prefix": prefix, "sizes": sizes, "p_inter": p_inter, "p_intra": 0.8})
    return inst


# ------------------------------------------------------- one large dense block
def make_brick_block(na: int, nb: int, depth: int, seed: int = 0, n: int = 16, n_low: int = 8,
                     n_bits: int = 0) -> Instance:
    """One joint block of `depth` brickwork layers (Haar SU(2) on every block
    qubit, then CZ on alternating neighbour pairs) on the nb + na qubits around
    the cut [n_low - nb, n_low + na), after a Haar layer on all n qubits and
    before another: the large dense blocks the paper's cost remark is about
    (P:192-194), for the sequential factor route."""
    rng = np.random.default_rng([seed, 11])
    qs = list(range(n_low - nb, n_low + na))
    g = [_u1(q, rng) for q in range(n)]
    blk = []
    for L in range(depth):
        for q in qs:
            blk.append(len(g))
            g.append(_u1(q, rng))
        for a in range(L % 2, len(qs) - 1, 2):
            blk.append(len(g))
            g.append(("cz", (), (qs[a], qs[a + 1]), None))
    g += [_u1(q, rng) for q in range(n)]
    bits = _bitstrings(seed, n, n_bits) if n_bits else None
    return Instance("brick%d+%d" % (nb, na), n, n_low, g, [blk], bits, "c64", {"seed": seed, "depth": depth})


# ---------------------------------------------------------- random small sweeps
_NAMED_1Q = ("h", "x", "z", "rx", "rz")
_NAMED_2Q = ("cz", "cx", "swap", "cp", "rzz")


def random_small_circuit(seed: int, n: int | None = None, n_gates: int | None = None,
                         max_block_qubits: int = 6, with_u: bool = True) -> Instance:
    """Random circuit over the whole gate library plus dense 1..3-qubit `u`
    gates, a random contiguous cut, and random joint blocks formed from runs of
    consecutive gates (consecutive runs are always convex in the wire DAG)."""
    rng = np.random.default_rng([seed, 7])
    n = n if n is not None else int(rng.integers(4, 11))
    n_low = int(rng.integers(1, n))
    n_gates = n_gates if n_gates is not None else int(rng.integers(8, 40))
    g = []
    for _ in range(n_gates):
        r = rng.uniform()
        if r < 0.35:
            name = _NAMED_1Q[int(rng.integers(len(_NAMED_1Q)))]
            q = int(rng.integers(n))
            params = (rng.uniform(0, 2 * math.pi),) if name in ("rx", "rz") else ()
            g.append((name, params, (q,), None))
        elif r < 0.8 or not with_u:
            name = _NAMED_2Q[int(rng.integers(len(_NAMED_2Q)))]
            a, b = (int(x) for x in rng.choice(n, size=2, replace=False))
            params = (rng.uniform(0, 2 * math.pi),) if name in ("cp", "rzz") else ()
            g.append((name, params, (a, b), None))
        else:
            k = int(rng.integers(1, min(3, n) + 1))
            qs = tuple(int(x) for x in rng.choice(n, size=k, replace=False))
            # random (generally non-unitary is allowed by the method, but keep
            # it unitary so the norm invariant holds): QR of a Gaussian
            d = 1 << k
            z = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
            q_, r_ = np.linalg.qr(z)
            q_ = q_ * (np.diag(r_) / np.abs(np.diag(r_)))
            payload = []
            for row in q_:
                for v in row:
                    payload += [float(v.real), float(v.imag)]
            g.append(("u", (), qs, payload))
    # blocks: random runs of consecutive gates containing a crossing gate
    def crossing(i):
        qs = g[i][2]
        return any(q < n_low for q in qs) and any(q >= n_low for q in qs)

    blocks = []
    i = 0
    while i < len(g):
        if crossing(i) and rng.uniform() < 0.7:
            j = i
            supp = set(g[i][2])
            while j + 1 < len(g) and rng.uniform() < 0.6:
                s2 = supp | set(g[j + 1][2])
                if len(s2) > max_block_qubits:
                    break
                supp = s2
                j += 1
            blocks.append(list(range(i, j + 1)))
            i = j + 1
        else:
            i += 1
    return Instance(f"rand{seed}", n, n_low, g, blocks, None, "c128", {"seed": seed})


def random_folding_circuit(seed: int, n: int | None = None, n_gates: int | None = None) -> Instance:
    """Random circuit shaped to exercise the half-sided folds: X gates on
    random qubits, then diagonal crossing gates (cz / cp / rzz, the head: they
    see computational-basis qubits), then a random body (random_small_circuit's
    library), then diagonal crossing gates again (the tail) and possibly a few
    trailing 1-qubit gates.  Blocks: none (every crossing gate its own unit)."""
    rng = np.random.default_rng([seed, 11])
    n = n if n is not None else int(rng.integers(4, 10))
    n_low = int(rng.integers(1, n))
    body = random_small_circuit(seed + 1000, n=n, n_gates=n_gates if n_gates is not None else int(rng.integers(4, 16)))
    g = []
    for q in range(n):
        if rng.uniform() < 0.5:
            g.append(("x", (), (q,), None))

    def diag_cross():
        a = int(rng.integers(0, n_low))
        b = int(rng.integers(n_low, n))
        name = ("cz", "cp", "rzz")[int(rng.integers(3))]
        params = (rng.uniform(0, 2 * math.pi),) if name in ("cp", "rzz") else ()
        return (name, params, (a, b) if rng.uniform() < 0.5 else (b, a), None)

    for _ in range(int(rng.integers(1, 4))):
        g.append(diag_cross())
    g += [x for x in body.gates if x[0] != "u" or len(x[2]) == 1]
    for _ in range(int(rng.integers(1, 4))):
        g.append(diag_cross())
    for _ in range(int(rng.integers(0, 3))):
        q = int(rng.integers(n))
        g.append(("h", (), (q,), None))
    return Instance(f"fold{seed}", n, n_low, g, [], None, "c64", {"seed": seed})


# ------------------------------------------------------------------- registry
CONFIGS = {
    "c1": make_c1,
    "c2": make_c2,
    "c3": make_c3,
    "c4": make_c4,
    "c5": make_c5,
}

# small twins: same generator, oracle-friendly sizes
TWINS = {
    "c1": dict(n=12, n_low=6),
    "c2": dict(n=16, n_low=8),
    "c3": dict(n=12, n_low=6, depth=16, n_bits=4096),
    "c4": dict(n=12, n_low=6, p=3),
    "c5": dict(n=12, n_low=6, layers=8, fanout=3, n_bits=4096),
}


def make_config(name: str, seed: int | None = None, twin: bool = False, **kw) -> Instance:
    if name in TABLE2:
        if twin:  # oracle-sized stand-in of the same family
            inst = make_sbm_qaoa(seed=3100 + sorted(TABLE2).index(name) if seed is None else seed, sizes=(6, 6),
                                 p_intra=0.8, p_inter=0.3)
            inst.name, inst.blocks = name + "t", "auto"
            inst.meta["prefix"] = 1000
            return inst
        return make_table2(name, seed, **kw)
    fn = CONFIGS[name]
    args = dict(TWINS[name]) if twin else {}
    args.update(kw)
    if seed is not None:
        args["seed"] = seed
    inst = fn(**args)
    if twin:
        inst.name = name + "t"
    return inst
