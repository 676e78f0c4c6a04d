"""Process-parallel driver of the CPU oracle (TEST INFRASTRUCTURE ONLY; same
import rules as hsf_oracle.py).

It adds no arithmetic: each worker runs `hsf_oracle.simulate_path` for a
chunk of paths (one Feynman path = the two half-circuits from |0..0>)
and returns only the half-state entries the caller asks for, so full-size
bitstring configurations (2^20-amplitude halves) can be checked on a sample of
outputs without holding every path's half-states.  The Kronecker sum over
paths is then `hsf_oracle.recombine_bits` on those rows (SURVEY.md §8(d):
"multiprocessing.Pool over path chunks").
"""
from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

from . import hsf_oracle as O

_P = None  # the plan, inherited by forked workers


def _one_thread():
    """Workers run single-threaded BLAS: `procs` processes are the parallelism."""
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:  # pragma: no cover - threadpoolctl missing
        pass


def _chunk(args):
    p0, p1, rows_a, rows_b = args
    ka = np.empty((len(rows_a), p1 - p0), dtype=complex)
    kb = np.empty((len(rows_b), p1 - p0), dtype=complex)
    c = np.empty(p1 - p0, dtype=complex)
    for j, p in enumerate(range(p0, p1)):
        a, b, c[j] = O.simulate_path(_P, p)
        ka[:, j] = a[rows_a]
        kb[:, j] = b[rows_b]
    return p0, ka, kb, c


def n_procs() -> int:
    return max(1, len(os.sched_getaffinity(0)))


def half_state_rows(P, rows_a, rows_b, p0=0, p1=None, procs=None, chunk=None):
    """Psi_A[rows_a, p], Psi_B[rows_b, p], c_p for paths [p0, p1), paths
    evaluated in `procs` forked worker processes."""
    global _P
    p1 = P.n_paths if p1 is None else p1
    procs = procs or n_procs()
    chunk = chunk or max(1, -(-(p1 - p0) // (4 * procs)))
    rows_a = np.asarray(rows_a, dtype=np.int64)
    rows_b = np.asarray(rows_b, dtype=np.int64)
    jobs = [(q, min(p1, q + chunk), rows_a, rows_b) for q in range(p0, p1, chunk)]
    _P = P
    A = np.empty((len(rows_a), p1 - p0), dtype=complex)
    B = np.empty((len(rows_b), p1 - p0), dtype=complex)
    c = np.empty(p1 - p0, dtype=complex)
    try:
        if procs == 1:
            res = map(_chunk, jobs)
        else:
            pool = mp.get_context("fork").Pool(procs, initializer=_one_thread)
            res = pool.imap_unordered(_chunk, jobs)
        for q, ka, kb, cc in res:
            A[:, q - p0:q - p0 + ka.shape[1]] = ka
            B[:, q - p0:q - p0 + kb.shape[1]] = kb
            c[q - p0:q - p0 + len(cc)] = cc
        if procs != 1:
            pool.close()
            pool.join()
    finally:
        _P = None
    return A, B, c


def bits_amplitudes(P, bits, n_low, p0=0, p1=None, procs=None):
    """The oracle's amplitudes of a bitstring sample over paths [p0, p1):
    `recombine_bits` on the rows the sample touches."""
    bits = np.asarray(bits, dtype=np.uint64)
    ia = (bits >> np.uint64(n_low)).astype(np.int64)
    ib = (bits & np.uint64((1 << n_low) - 1)).astype(np.int64)
    ua, inv_a = np.unique(ia, return_inverse=True)
    ub, inv_b = np.unique(ib, return_inverse=True)
    A, B, c = half_state_rows(P, ua, ub, p0, p1, procs)
    # re-index: the compacted rows play the role of the full half-states
    compact = (inv_a.astype(np.uint64) << np.uint64(n_low)) | inv_b.astype(np.uint64)
    if len(ub) > (1 << n_low):
        raise AssertionError("row compaction overflow")
    return O.recombine_bits(A, B, c, compact, n_low)
