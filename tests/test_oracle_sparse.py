"""Pins for oracle/sparse_bqp.py (multi-block clique-chain relaxation, SURVEY §8(f) f2;
PAPER.md:555-602, remark P:434-436).

Pinned against: closed-form sizes; the dense relaxation (t = 1 is the dense problem of
oracle/bqp.py, itself pinned); the moment identity b^T mu(x) = objective on all of {-1,1}^d;
the semantics of the index map (A*(mu(x)) = v(x_k) v(x_k)^T on every block); adjointness;
Taylor slopes of the block ALM derivatives; the y-elimination against an explicit
least-squares minimisation of L_sigma; brute force (lower bound, tightness certificate)."""
import itertools
import math

import numpy as np
import pytest

from inputs import bqp_instance, chain_bqp_instance, initial_factor, random_matrix, random_unit_factor
from oracle import admm, bqp
from oracle import operators as ops
from oracle import sparse_bqp as sb
from oracle import subproblem as sp


def _slope(ts, errs):
    return np.polyfit(np.log(ts), np.log(errs), 1)[0]


@pytest.mark.parametrize("q,t", [(4, 1), (4, 3), (5, 4), (6, 2), (20, 3)])
def test_sizes_closed_form(q, t):
    Qs, cs = chain_bqp_instance(q, t, 0)
    amaps, cnt, b, mons = sb.relax_chain(Qs, cs)
    nb = 1 + q + q * (q - 1) // 2
    assert amaps.shape == (t, nb, nb)
    # union of the cliques' monomials: consecutive cliques share 2 variables (4 monomials incl. 1)
    assert cnt.size == t * sum(math.comb(q, k) for k in range(5)) - 4 * (t - 1)
    assert cnt.sum() == t * nb * nb and np.all(cnt >= 1)  # Assumption 2
    assert cnt[0] == t * nb  # the constant monomial: every diagonal entry of every block
    for k in range(t):
        assert np.array_equal(amaps[k], amaps[k].T)
        assert np.all(np.diag(amaps[k]) == 0)


def test_single_block_is_the_dense_relaxation():
    """t = 1: the clique is all d = q variables, so the relaxation is the dense one."""
    q = 7
    Qs, cs = chain_bqp_instance(q, 1, 3)
    amaps, cnt, b, _ = sb.relax_chain(Qs, cs)
    amap, cnt_d, b_d = bqp.relax(Qs[0], cs[0])
    assert np.array_equal(amaps[0], amap) and np.array_equal(cnt, cnt_d)
    np.testing.assert_array_equal(b, b_d)


@pytest.mark.parametrize("q,t", [(4, 3), (5, 2)])
def test_moment_identity_and_index_map_semantics(q, t):
    """b^T mu(x) = sum_k x_k^T Q_k x_k + c_k^T x_k on all of {-1,1}^d, and A*(mu(x)) restricted to
    block k is v(x_k) v(x_k)^T (the index map is the monomial product mod x^2 = 1)."""
    Qs, cs = chain_bqp_instance(q, t, 1)
    amaps, cnt, b, mons = sb.relax_chain(Qs, cs)
    d = (q - 2) * t + 2
    nb = amaps.shape[1]
    for bits in itertools.product((-1.0, 1.0), repeat=d):
        x = np.array(bits)
        mu = sb.chain_moment_vector(x, mons)
        assert abs(b @ mu - sb.chain_value(Qs, cs, x)) <= 1e-12 * (1 + abs(b @ mu))
        V = sb.chain_block_factor(x, q, t)
        Sb = sb.block_gram(V, V, t)
        np.testing.assert_array_equal(sb.At_blocks(amaps, mu), Sb)
    assert V.shape[0] == t * nb


def test_adjointness_and_gram():
    Qs, cs = chain_bqp_instance(4, 3, 2)
    amaps, cnt, b, _ = sb.relax_chain(Qs, cs)
    t, nb, m = amaps.shape[0], amaps.shape[1], cnt.size
    rng = np.random.default_rng(5)
    X = rng.standard_normal((t, nb, nb))
    y = rng.standard_normal(m)
    assert abs(sb.A_blocks(amaps, X, m) @ y - np.sum(X * sb.At_blocks(amaps, y))) <= 1e-10
    # AA* = Diag(cnt), column by column on a few ids
    for a in (0, 1, m // 2, m - 1):
        e = np.zeros(m)
        e[a] = 1.0
        np.testing.assert_array_equal(sb.A_blocks(amaps, sb.At_blocks(amaps, e), m), cnt * e)


def _block_state(q=4, t=3, seed=0, sigma=2.0, p=3):
    Qs, cs = chain_bqp_instance(q, t, seed)
    amaps, cnt, b, _ = sb.relax_chain(Qs, cs)
    t, nb, m = amaps.shape[0], amaps.shape[1], cnt.size
    rng = np.random.default_rng([seed, 9])
    Xt = rng.standard_normal((t, nb, nb)) * 0.3
    Xt = Xt + np.transpose(Xt, (0, 2, 1))
    Xt = Xt - sb.At_blocks(amaps, sb.A_blocks(amaps, Xt, m) / cnt)  # A(X~) = 0 (Lemma 3.1)
    D = sb.At_blocks(amaps, b / cnt)
    N = t * nb
    Y = random_unit_factor(N, p, seed + 11)
    U = sp.project(Y, random_matrix(N, p, seed + 12))
    return amaps, cnt, b, Xt, D, Xt + D, sigma, Y, U


def test_single_block_alm_matches_dense_alm():
    Q, c = bqp_instance(6, 4)
    amap, cnt, b = bqp.relax(Q, c)
    n = amap.shape[0]
    T = ops.D_matrix(amap, cnt, b) + 0.1 * np.eye(n)
    Y = random_unit_factor(n, 4, 1)
    U = sp.project(Y, random_matrix(n, 4, 2))
    o = sp.alm_eval(T, amap, cnt, None, 1.7, Y, U)
    ob = sb.block_alm_eval(T[None], amap[None], cnt, 1.7, Y, U)
    assert abs(o["f"] - ob["f"]) <= 1e-12 * abs(o["f"])
    for key in ("R", "H", "rho"):
        np.testing.assert_allclose(ob[key], o[key], rtol=0, atol=1e-12 * np.abs(o[key]).max())


@pytest.mark.parametrize("seed", [0, 1])
def test_block_alm_taylor_slopes_and_tangency(seed):
    amaps, cnt, b, Xt, D, T, sigma, Y, U = _block_state(seed=seed)
    prob = sb.BlockALMProblem(T, amaps, cnt, sigma)
    f0, g0, ctx = prob.costgrad(Y)
    H = prob.hess(ctx, U)
    assert np.abs(sp.rowdot(g0, Y)).max() <= 1e-10 * np.abs(g0).max()
    assert np.abs(sp.rowdot(H, Y)).max() <= 1e-10 * np.abs(H).max()
    ts1 = np.array([1e-3, 3e-4, 1e-4, 3e-5])
    e1 = [abs(prob.costgrad(sp.retract(Y, s * U))[0] - f0 - s * sp.inner(g0, U)) for s in ts1]
    assert abs(_slope(ts1, e1) - 2.0) < 0.1, e1
    ts2 = np.array([3e-3, 1e-3, 3e-4, 1e-4])
    e2 = [abs(prob.costgrad(sp.retract(Y, s * U))[0] - f0 - s * sp.inner(g0, U) - 0.5 * s * s * sp.inner(U, H))
          for s in ts2]
    assert abs(_slope(ts2, e2) - 3.0) < 0.2, e2
    # self-adjoint Hessian
    V = sp.project(Y, random_matrix(Y.shape[0], Y.shape[1], 77))
    HV = prob.hess(ctx, V)
    assert abs(sp.inner(HV, U) - sp.inner(H, V)) <= 1e-10 * (abs(sp.inner(H, V)) + 1)


def test_block_alm_is_the_y_eliminated_lagrangian():
    """(sigma/2) f^ - ||T||^2/(2 sigma) = min_y L_sigma(S, y, X~) (Lemma 3.1) with the
    minimum found by a generic least-squares solve over y (not the cnt division), blocks summed."""
    amaps, cnt, b, Xt, D, T, sigma, Y, U = _block_state(seed=3, sigma=1.3)
    t, nb, m = amaps.shape[0], amaps.shape[1], cnt.size
    S = sb.block_gram(Y, Y, t)
    # L(y) = <D, S> - <X~, A*(y) - S> + sigma/2 ||A*(y) - S||^2 over the blocks; A* as a matrix
    Amat = np.zeros((t * nb * nb, m))
    Amat[np.arange(t * nb * nb), amaps.ravel()] = 1.0
    s, xt = S.ravel(), Xt.ravel()
    # minimiser: sigma A^T (A y - s) - A^T x~ = 0  <=>  least squares of A y ~ s + x~/sigma
    ymin = np.linalg.lstsq(Amat, s + xt / sigma, rcond=None)[0]
    R = Amat @ ymin - s
    Lmin = float(D.ravel() @ s - xt @ R + 0.5 * sigma * R @ R)
    f = sb.block_alm_eval(T, amaps, cnt, sigma, Y)["f"]
    assert abs(0.5 * sigma * f - np.sum(T * T) / (2 * sigma) - Lmin) <= 1e-9 * (1 + abs(Lmin))


def test_block_escape_directions():
    """t = 1: the dense escape rule (oracle/admm.escape_directions). t > 1: column c carries the
    c-th most negative eigenvector of every block with one (reading R39), each a unit eigenvector
    of its block with negative curvature, so <[0,V], 4 X [0,V]> < 0 (Thm 4.5)."""
    rng = np.random.default_rng(8)
    nb = 6
    A = rng.standard_normal((nb, nb))
    B = (A + A.T) / 2
    lam, V = np.linalg.eigh(B)
    for emax in (1, 3, 5):
        np.testing.assert_allclose(sb.block_escape_directions([lam], [V], 1e-9, emax),
                                   admm.escape_directions(lam, V, 1e-9, emax), atol=1e-12)
    blocks = []
    for k in range(3):
        A = rng.standard_normal((nb, nb))
        blocks.append((A + A.T) / 2 + (k - 1) * 1.5 * np.eye(nb))  # different numbers of negative eigenvalues
    lams, Vs = zip(*[np.linalg.eigh(Bk) for Bk in blocks])
    negs = [int(np.sum(l < -1e-9 * (1 + max(float(x[-1]) for x in lams)))) for l in lams]
    E = sb.block_escape_directions(list(lams), list(Vs), 1e-9, 4)
    assert E.shape[1] == min(4, max(negs))
    for k in range(3):
        Ek = E[k * nb:(k + 1) * nb]
        for c in range(E.shape[1]):
            v = Ek[:, c]
            if c < negs[k]:
                assert abs(np.linalg.norm(v) - 1) < 1e-12
                np.testing.assert_allclose(blocks[k] @ v, lams[k][c] * v, atol=1e-10)
                assert v[np.argmax(np.abs(v))] > 0
            else:
                assert not v.any()
    Xd = np.zeros((3 * nb, 3 * nb))
    for k in range(3):
        Xd[k * nb:(k + 1) * nb, k * nb:(k + 1) * nb] = blocks[k]
    assert np.trace(E.T @ Xd @ E) < 0


def _chain_solve(q, t, seed, p0=2):
    Qs, cs = chain_bqp_instance(q, t, seed)
    amaps, cnt, b, mons = sb.relax_chain(Qs, cs)
    N = amaps.shape[0] * amaps.shape[1]
    prm = admm.Params(p0=p0)
    out = sb.solve_blocks(amaps, cnt, b, prm, initial_factor(N, p0, seed))
    return Qs, cs, amaps, cnt, b, mons, out


def test_single_block_solve_equals_dense_solve():
    """t = 1: Algorithm 2 over blocks and the dense Algorithm 2 run the same iteration."""
    q = 6
    Qs, cs, amaps, cnt, b, mons, out = _chain_solve(q, 1, 0)
    n = amaps.shape[1]
    ref = admm.solve(amaps[0], cnt, b, None, admm.Params(p0=2), initial_factor(n, 2, 0))
    assert out["status"] == ref["status"] == "converged"
    assert out["outer_iters"] == ref["outer_iters"]
    assert abs(out["dual_obj"] - ref["dual_obj"]) <= 1e-9 * (1 + abs(ref["dual_obj"]))


@pytest.mark.parametrize("q,t,seed", [(4, 3, 0), (5, 3, 1), (6, 2, 2)])
def test_chain_solve_lower_bound_and_certificate(q, t, seed):
    Qs, cs, amaps, cnt, b, mons, out = _chain_solve(q, t, seed)
    assert out["status"] == "converged" and out["eta_max"] <= 1e-8
    bf, xbf = sb.chain_brute_force(Qs, cs)
    assert out["dual_obj"] <= bf + 1e-6  # the relaxation is a lower bound
    res = sb.block_residues(amaps, cnt, b, out["y"], out["Y"], out["T"])  # recomputed
    assert res["eta_max"] <= 1e-8
    assert abs(out["y"][0] - 1.0) <= 1e-8  # y_1 = 1 <=> every diagonal of every block is 1
    # rank-one blocks: round x from the degree-1 moments and certify tightness
    x = np.sign(out["y"][1:1 + (q - 2) * t + 2])
    if abs(sb.chain_value(Qs, cs, x) - out["dual_obj"]) <= 1e-6 * (1 + abs(bf)):
        assert abs(bf - out["dual_obj"]) <= 1e-6 * (1 + abs(bf))
