"""TEST INFRASTRUCTURE ONLY -- exhaustive posterior enumeration for small codes.

Ground truth for the cycle-free exactness suite (the checker, never the
product).  Restates the reference's test oracles
(/root/reference/pkg/tests/oracles.py:116-173) in numpy:

    all_patterns        oracles.py:116-118   every Pauli pattern of n qubits (4^n)
    pattern_weights     oracles.py:121-124   i.i.d. depolarizing prior with eps0
    pattern_syndromes   oracles.py:127-132   symplectic syndromes of all patterns
    posterior_marginals oracles.py:135-146   per-qubit posterior over {I, X, Z, Y}
    map_decisions       oracles.py:149-152   per-qubit MAP Pauli, ties to the lower code
    brute_vn_message    oracles.py:155-173   exact qubit->check LLR on a tree

Pauli codes follow pauli.py:28-31 (I=0, X=1, Z=2, Y=3; bit 0 = x, bit 1 = z);
rows are [(column, symbol)] as in SparseCheckMatrix.rows.  Pinned against the
reference's own functions in tests/test_oracle_pins.py.
"""
from __future__ import annotations

import itertools

import numpy as np


def trace_inner(a: int, b: int) -> int:
    """1 iff Paulis a and b anticommute (pauli.py trace_inner)."""
    return ((a & 1) & (b >> 1)) ^ ((a >> 1) & (b & 1))


def dense_planes(n, rows):
    """(hx, hz) uint8 (m, n): x and z bits of every row's symbols."""
    hx = np.zeros((len(rows), n), dtype=np.uint8)
    hz = np.zeros((len(rows), n), dtype=np.uint8)
    for i, row in enumerate(rows):
        for j, s in row:
            hx[i, j] = s & 1
            hz[i, j] = s >> 1
    return hx, hz


def all_patterns(n: int) -> np.ndarray:
    return np.array(list(itertools.product(range(4), repeat=n)), dtype=np.uint8)


def pattern_weights(patterns: np.ndarray, eps0: float) -> np.ndarray:
    wt = (patterns != 0).sum(axis=1)
    n = patterns.shape[1]
    return (1.0 - eps0) ** (n - wt) * (eps0 / 3.0) ** wt


def pattern_syndromes(n, rows, patterns: np.ndarray) -> np.ndarray:
    hx, hz = dense_planes(n, rows)
    ex, ez = (patterns & 1).astype(np.int64), (patterns >> 1).astype(np.int64)
    return ((ez @ hx.T.astype(np.int64) + ex @ hz.T.astype(np.int64)) % 2).astype(np.uint8)


def posterior_marginals(n, rows, s, eps0: float) -> np.ndarray:
    patterns = all_patterns(n)
    match = (pattern_syndromes(n, rows, patterns) == np.asarray(s, dtype=np.uint8)).all(axis=1)
    pats = patterns[match]
    w = pattern_weights(pats, eps0)
    marg = np.zeros((n, 4))
    for j in range(n):
        np.add.at(marg[j], pats[:, j], w)
    return marg / w.sum()


def map_decisions(n, rows, s, eps0: float) -> np.ndarray:
    return np.argmax(posterior_marginals(n, rows, s, eps0), axis=1).astype(np.uint8)


def brute_vn_message(n, rows, s, eps0: float, check: int, qubit: int, _cache=None) -> float:
    """Exact qubit-to-check LLR of edge (check, qubit) on a cycle-free code:
    log P(error commutes with the edge symbol) - log P(anticommutes), under
    the prior conditioned on every OTHER check's syndrome bit."""
    sym = dict(rows[check])[qubit]
    if _cache is None:
        patterns = all_patterns(n)
        syndromes = pattern_syndromes(n, rows, patterns)
    else:
        patterns, syndromes = _cache
    others = [i for i in range(len(rows)) if i != check]
    s = np.asarray(s, dtype=np.uint8)
    match = (syndromes[:, others] == s[others]).all(axis=1)
    pats = patterns[match]
    w = pattern_weights(pats, eps0)
    anti = np.array([trace_inner(e, sym) for e in range(4)])[pats[:, qubit]]
    return float(np.log(w[anti == 0].sum()) - np.log(w[anti == 1].sum()))


def brute_vn_messages(n, rows, s, eps0: float, edges) -> np.ndarray:
    """brute_vn_message for every (check, qubit, _) of ``edges`` (canonical
    order), sharing one pattern enumeration."""
    patterns = all_patterns(n)
    cache = (patterns, pattern_syndromes(n, rows, patterns))
    return np.array([brute_vn_message(n, rows, s, eps0, i, j, cache) for i, j, _ in edges])
