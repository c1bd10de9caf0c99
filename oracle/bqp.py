"""Second-order moment relaxation of a binary quadratic program (oracle).

PAPER.md:455-477 (§6.1, Eq. BQP and Eq. 6.3): v(x) = [1, x_1..x_q, x_1x_2, x_1x_3, ..,
x_{q-1}x_q]; one linear constraint per square-free monomial of degree <= 4
(P:476); the dual of the SOS relaxation is (DSDP) with C = 0.

Ordering (reading R18): basis and constraint monomials in graded-lex order
of sorted index tuples; this is the contract for bit-exact index-map parity.
"""
from __future__ import annotations

import itertools

import numpy as np


def basis_monomials(d: int):
    """Monomials of v(x) as sorted index tuples, graded-lex."""
    out = [()]
    out += [(i,) for i in range(d)]
    out += list(itertools.combinations(range(d), 2))
    return out


def constraint_monomials(d: int):
    """All square-free monomials of degree <= 4, graded-lex."""
    out = []
    for k in range(5):
        out += list(itertools.combinations(range(d), k))
    return out


def relax(Q: np.ndarray, c: np.ndarray):
    """Return (amap, cnt, b) of the dense second-order relaxation.

    amap[i, j] = id of the reduced product v_i(x) * v_j(x) mod (x_k^2 - 1), i.e. the
    symmetric difference of the two index sets. A_a is the 0/1 indicator
    of {(i, j) : amap[i, j] = a} over ordered positions, so <A_a, X> counts
    off-diagonal entries twice and (AA*)_aa = cnt_a.
    b_a = coefficient of monomial a in x^T Q x + c^T x reduced mod the ideal:
    b_{1} = sum_i Q_ii, b_{x_i} = c_i, b_{x_i x_j} = 2 Q_ij (i < j), 0 for degree 3-4.
    """
    d = Q.shape[0]
    basis = basis_monomials(d)
    cons = constraint_monomials(d)
    ids = {mono: k for k, mono in enumerate(cons)}
    n, m = len(basis), len(cons)
    amap = np.empty((n, n), dtype=np.int32)
    sets = [frozenset(t) for t in basis]
    for i in range(n):
        for j in range(n):
            amap[i, j] = ids[tuple(sorted(sets[i] ^ sets[j]))]
    cnt = np.bincount(amap.ravel(), minlength=m).astype(np.int64)
    b = np.zeros(m)
    b[ids[()]] = np.trace(Q)
    for i in range(d):
        b[ids[(i,)]] = c[i]
    for i, j in itertools.combinations(range(d), 2):
        b[ids[(i, j)]] = 2.0 * Q[i, j]
    return amap, cnt, b


def moment_vector(x: np.ndarray, d: int) -> np.ndarray:
    """mu(x)_a = prod_{i in a} x_i for every constraint monomial a (graded-lex)."""
    return np.array([np.prod(x[list(a)]) if a else 1.0 for a in constraint_monomials(d)])


def basis_vector(x: np.ndarray, d: int) -> np.ndarray:
    """v(x)."""
    return np.array([np.prod(x[list(a)]) if a else 1.0 for a in basis_monomials(d)])


def bqp_value(Q: np.ndarray, c: np.ndarray, x: np.ndarray) -> float:
    return float(x @ Q @ x + c @ x)


def brute_force(Q: np.ndarray, c: np.ndarray):
    """min over x in {-1,1}^d of x^T Q x + c^T x by exhaustive enumeration."""
    d = Q.shape[0]
    if d > 24:
        raise ValueError("brute force limited to d <= 24")
    best, arg = np.inf, None
    for bits in range(1 << d):
        x = np.array([1.0 if (bits >> k) & 1 else -1.0 for k in range(d)])
        v = bqp_value(Q, c, x)
        if v < best:
            best, arg = v, x
    return best, arg
