"""Pins for oracle/bqp.py and oracle/operators.py (DESIGN.md "Oracle pins" P1-P3).

Every check compares the oracle against something other than itself: closed-form
counts, an independent bitmask construction of the index map, the polynomial
identity b^T mu(x) = x^T Q x + c^T x on {-1,1}^d, exhaustive Gram matrices.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

from inputs import bqp_instance
from oracle import bqp
from oracle import operators as ops

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_spec_examples.json")))


def _n(d):
    return 1 + d + d * (d - 1) // 2


def _m(d):
    return sum(math.comb(d, k) for k in range(5))


@pytest.mark.parametrize("d,n,m", GOLD["relaxation_sizes"]["cases"])
def test_golden_sizes(d, n, m):
    assert _n(d) == n and _m(d) == m
    if d <= 40:
        assert len(bqp.basis_monomials(d)) == n
        assert len(bqp.constraint_monomials(d)) == m


@pytest.mark.parametrize("d", list(range(2, 13)))
def test_counts_closed_form(d):
    Q, c = bqp_instance(d, 0)
    amap, cnt, b = bqp.relax(Q, c)
    assert amap.shape == (_n(d), _n(d))
    assert cnt.size == _m(d) == b.size
    assert int(cnt.sum()) == _n(d) ** 2


def _bitmask_map(d):
    """Independent construction: monomials as bitmasks, product = XOR, ids by
    (popcount, lexicographic index tuple)."""
    basis = [0] + [1 << i for i in range(d)] + [(1 << i) | (1 << j) for i in range(d) for j in range(i + 1, d)]
    cons = [mk for mk in range(1 << d) if bin(mk).count("1") <= 4]
    cons.sort(key=lambda mk: (bin(mk).count("1"), [i for i in range(d) if mk >> i & 1]))
    ids = {mk: k for k, mk in enumerate(cons)}
    n = len(basis)
    return np.array([[ids[basis[i] ^ basis[j]] for j in range(n)] for i in range(n)], dtype=np.int32)


@pytest.mark.parametrize("d", [2, 3, 5, 8, 10, 12])
def test_index_map_matches_bitmask_construction(d):
    Q, c = bqp_instance(d, 1)
    amap, cnt, b = bqp.relax(Q, c)
    np.testing.assert_array_equal(amap, _bitmask_map(d))


@pytest.mark.parametrize("d", [3, 5, 10])
def test_class_sizes(d):
    """cnt = n for the constant monomial (the diagonal), 2d for degree 1 and 2,
    6 for degree 3 and 4 (counted by hand, P1)."""
    Q, c = bqp_instance(d, 0)
    amap, cnt, b = bqp.relax(Q, c)
    n = _n(d)
    mons = bqp.constraint_monomials(d)
    for a, mono in enumerate(mons):
        expect = {0: n, 1: 2 * d, 2: 2 * d, 3: 6, 4: 6}[len(mono)]
        assert cnt[a] == expect, (mono, cnt[a], expect)
    assert np.all(np.diag(amap) == 0)
    np.testing.assert_array_equal(amap, amap.T)


@pytest.mark.parametrize("d", [4, 10])
def test_b_reproduces_polynomial_on_hypercube(d):
    """b^T mu(x) = x^T Q x + c^T x for all x in {-1,1}^d (reduction mod x_i^2 - 1)."""
    Q, c = bqp_instance(d, 2)
    amap, cnt, b = bqp.relax(Q, c)
    for bits in range(1 << d):
        x = np.array([1.0 if bits >> k & 1 else -1.0 for k in range(d)])
        assert abs(b @ bqp.moment_vector(x, d) - bqp.bqp_value(Q, c, x)) < 1e-12


def test_b_with_nonzero_diagonal():
    rng = np.random.default_rng(5)
    d = 5
    Q = rng.standard_normal((d, d)); Q = Q + Q.T
    c = rng.standard_normal(d)
    amap, cnt, b = bqp.relax(Q, c)
    for bits in range(1 << d):
        x = np.array([1.0 if bits >> k & 1 else -1.0 for k in range(d)])
        assert abs(b @ bqp.moment_vector(x, d) - bqp.bqp_value(Q, c, x)) < 1e-12


@pytest.mark.parametrize("d", [3, 6])
def test_moment_matrix_feasible(d):
    """A(v(x) v(x)^T) = cnt o mu(x): y(S) = mu(x) for the rank-one moment matrix."""
    Q, c = bqp_instance(d, 0)
    amap, cnt, b = bqp.relax(Q, c)
    m = cnt.size
    for bits in [0, 5, (1 << d) - 1]:
        x = np.array([1.0 if bits >> k & 1 else -1.0 for k in range(d)])
        v = bqp.basis_vector(x, d)
        S = np.outer(v, v)
        np.testing.assert_allclose(ops.A(amap, S, m), cnt * bqp.moment_vector(x, d), atol=1e-12)
        assert np.allclose(np.diag(S), 1.0)
        np.testing.assert_allclose(ops.At(amap, bqp.moment_vector(x, d)), S, atol=0)


@pytest.mark.parametrize("d", [2, 4])
def test_AAt_diagonal_exhaustive(d):
    """(AA*)_ab = <A_a, A_b> computed from explicit indicator matrices."""
    Q, c = bqp_instance(d, 0)
    amap, cnt, b = bqp.relax(Q, c)
    m = cnt.size
    mats = [(amap == a).astype(float) for a in range(m)]
    G = np.array([[np.sum(mats[a] * mats[bb]) for bb in range(m)] for a in range(m)])
    np.testing.assert_allclose(G, np.diag(ops.AAt(amap, m)))


def test_adjointness_and_D():
    d = 6
    Q, c = bqp_instance(d, 0)
    amap, cnt, b = bqp.relax(Q, c)
    m = cnt.size
    rng = np.random.default_rng(0)
    X = rng.standard_normal(amap.shape); X = X + X.T
    y = rng.standard_normal(m)
    assert abs(np.sum(ops.At(amap, y) * X) - y @ ops.A(amap, X, m)) < 1e-10 * np.abs(X).sum()
    D = ops.D_matrix(amap, cnt, b)
    np.testing.assert_allclose(ops.A(amap, D, m), b, atol=1e-12)
    # y-update orthogonality: <A*(y) - (S+C), A*(v)> = 0 for random v
    S = X
    yy = ops.y_update(amap, cnt, S, None)
    for _ in range(3):
        v = rng.standard_normal(m)
        assert abs(np.sum((ops.At(amap, yy) - S) * ops.At(amap, v))) < 1e-10 * np.abs(S).sum()
    # gram_solve round trip
    np.testing.assert_allclose(ops.gram_solve(cnt, ops.A(amap, ops.At(amap, y), m)), y, rtol=1e-13)


def test_spec_operator_examples():
    # A = identity on a 2x2 block -> trace; A_1 = E12 + E21 -> 2 X_12
    X = np.array([[1.0, 2.0], [2.0, 3.0]])
    amap = np.array([[0, 1], [1, 0]], dtype=np.int32)  # a=0: diagonal, a=1: off-diagonal pair
    out = ops.A(amap, X, 2)
    assert out[0] == 4.0 and out[1] == 4.0
    with pytest.raises(ValueError):
        ops.check_assumption2(np.array([2, 0]))


def test_brute_force_golden():
    t = GOLD["toy_bqp"]
    assert bqp.brute_force(np.array(t["Q"], float), np.array(t["c"], float))[0] == t["min"]
    q = GOLD["all_ones_c"]["q"]
    val, x = bqp.brute_force(np.zeros((q, q)), np.ones(q))
    assert val == GOLD["all_ones_c"]["min"] and np.all(x == -1)


def test_bqp_generator_distribution():
    Q, c = bqp_instance(40, 0)
    np.testing.assert_array_equal(Q, Q.T)
    assert np.all(np.diag(Q) == 0)
    assert np.abs(Q).max() <= 1 and np.abs(c).max() <= 1
    Qs, _ = bqp_instance(150, 0, "er05")
    frac = np.count_nonzero(np.triu(Qs, 1)) / (150 * 149 / 2)
    assert 0.04 < frac < 0.06
