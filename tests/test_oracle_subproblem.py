"""Pins for oracle/subproblem.py (DESIGN.md "Oracle pins" P4-P7).

Finite-difference Taylor slopes, self-adjointness, the literal paper formulas
Eq. 4.6 / Eq. 4.7 / L_sigma on the paper scale, the saddle-escape
identity and the nearest-correlation-matrix special case (P7)."""
import json
import os

import numpy as np
import pytest

from inputs import bqp_instance, random_matrix, random_symmetric, random_unit_factor
from oracle import bqp
from oracle import operators as ops
from oracle import subproblem as sp

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_spec_examples.json")))


def _slope(ts, errs):
    return np.polyfit(np.log(ts), np.log(errs), 1)[0]


def _bqp_state(d=4, seed=0, sigma=2.0, lemma31=True):
    """A BQP operator plus a state T with A(T) = b (Lemma 3.1) or arbitrary."""
    Q, c = bqp_instance(d, seed)
    amap, cnt, b = bqp.relax(Q, c)
    n, m = amap.shape[0], cnt.size
    D = ops.D_matrix(amap, cnt, b)
    Xt = random_symmetric(n, seed + 1, 0.3)
    if lemma31:  # remove the A-range part so that A(X~) = 0
        Xt = Xt - ops.At(amap, ops.A(amap, Xt, m) / cnt)
    return amap, cnt, b, D, Xt, Xt + D, sigma


def test_projector_examples_and_idempotency():
    g = GOLD["projector_example"]
    Y = np.array(g["Y"], float); U = np.array(g["U"], float)
    np.testing.assert_array_equal(sp.project(Y, U), U)
    Y = random_unit_factor(30, 5, 0)
    U = random_matrix(30, 5, 1)
    P1 = sp.project(Y, U)
    assert np.abs(sp.project(Y, P1) - P1).max() <= 1e-14
    assert np.abs(sp.rowdot(P1, Y)).max() <= 1e-14
    u = random_matrix(30, 1, 2)[:, 0]
    assert np.abs(sp.project(Y, u[:, None] * Y)).max() <= 1e-14  # normal space annihilated


def test_retraction_examples():
    g = GOLD["retraction_example"]
    np.testing.assert_allclose(sp.retract(np.array(g["Y"], float), np.array(g["U"], float)), g["out"], rtol=1e-15)
    Y = random_unit_factor(10, 3, 0)
    np.testing.assert_array_equal(sp.retract(Y, np.zeros_like(Y)), Y / np.linalg.norm(Y, axis=1, keepdims=True))
    with pytest.raises(FloatingPointError):
        sp.retract(Y, -Y)
    # first-order agreement ||R(tU) - (Y + tU)|| = O(t^2)
    U = sp.project(Y, random_matrix(10, 3, 1))
    ts = np.array([1e-2, 1e-3, 1e-4])
    errs = [np.linalg.norm(sp.retract(Y, t * U) - (Y + t * U)) for t in ts]
    assert abs(_slope(ts, errs) - 2.0) < 0.1


def test_fixed_special_case_and_invariance():
    # sigma=1, X~=y=C=D=0 => Psi = 1/2 ||S||^2: on the f scale M = 0 => f = ||S||^2
    Y = random_unit_factor(20, 4, 3)
    S = Y @ Y.T
    assert abs(sp.fixed_eval(np.zeros((20, 20)), Y)["f"] - np.sum(S * S)) <= 1e-12 * np.sum(S * S)
    M = random_symmetric(20, 4)
    O, _ = np.linalg.qr(random_matrix(4, 4, 5))
    a, b = sp.fixed_eval(M, Y), sp.fixed_eval(M, Y @ O)
    assert abs(a["f"] - b["f"]) <= 1e-12 * abs(a["f"])
    assert abs(np.linalg.norm(a["R"]) - np.linalg.norm(b["R"])) <= 1e-10 * np.linalg.norm(a["R"])


def _fd_checks(costgrad, hess, Y, U):
    f0, g0 = costgrad(Y)
    assert np.abs(sp.rowdot(g0, Y)).max() <= 1e-10 * max(1.0, np.abs(g0).max())
    H = hess(Y, U)
    assert np.abs(sp.rowdot(H, Y)).max() <= 1e-10 * max(1.0, np.abs(H).max())
    ts1 = np.array([1e-3, 3e-4, 1e-4, 3e-5])
    e1 = [abs(costgrad(sp.retract(Y, t * U))[0] - f0 - t * sp.inner(g0, U)) for t in ts1]
    assert abs(_slope(ts1, e1) - 2.0) < 0.1, e1
    ts2 = np.array([3e-3, 1e-3, 3e-4, 1e-4])
    e2 = [abs(costgrad(sp.retract(Y, t * U))[0] - f0 - t * sp.inner(g0, U) - 0.5 * t * t * sp.inner(U, H))
          for t in ts2]
    assert abs(_slope(ts2, e2) - 3.0) < 0.2, e2  # row normalisation is a 2nd-order retraction


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_fixed_gradient_hessian_fd(seed):
    n, p = 25, 4
    M = random_symmetric(n, seed, 0.5)
    Y = random_unit_factor(n, p, seed)
    U = sp.project(Y, random_matrix(n, p, seed + 10))
    _fd_checks(lambda Y: (sp.fixed_eval(M, Y)["f"], sp.fixed_eval(M, Y)["R"]),
               lambda Y, U: sp.fixed_eval(M, Y, U)["H"], Y, U)


@pytest.mark.parametrize("seed", [0, 1])
def test_alm_gradient_hessian_fd(seed):
    amap, cnt, b, D, Xt, T, sigma = _bqp_state(4, seed)
    n = amap.shape[0]
    Y = random_unit_factor(n, 3, seed)
    U = sp.project(Y, random_matrix(n, 3, seed + 20))
    ev = lambda Y, U=None: sp.alm_eval(T, amap, cnt, None, sigma, Y, U)
    _fd_checks(lambda Y: (ev(Y)["f"], ev(Y)["R"]), lambda Y, U: ev(Y, U)["H"], Y, U)


def test_hessian_self_adjoint():
    amap, cnt, b, D, Xt, T, sigma = _bqp_state(4, 3)
    n = amap.shape[0]
    Y = random_unit_factor(n, 3, 7)
    U = sp.project(Y, random_matrix(n, 3, 8))
    V = sp.project(Y, random_matrix(n, 3, 9))
    HU = sp.alm_eval(T, amap, cnt, None, sigma, Y, U)["H"]
    HV = sp.alm_eval(T, amap, cnt, None, sigma, Y, V)["H"]
    a, bb = sp.inner(V, HU), sp.inner(U, HV)
    assert abs(a - bb) <= 1e-10 * max(abs(a), 1.0)
    M = random_symmetric(n, 1)
    HU = sp.fixed_eval(M, Y, U)["H"]; HV = sp.fixed_eval(M, Y, V)["H"]
    assert abs(sp.inner(V, HU) - sp.inner(U, HV)) <= 1e-10 * max(abs(sp.inner(V, HU)), 1.0)


def test_alm_matches_paper_eq46_eq47_and_Lsigma():
    """The f^-scale gradient/HVP equal (2/sigma) x the literal Eq. 4.6/4.7 with
    grad Phi at y(S), and (sigma/2) f^ - ||T||^2/(2 sigma) = L_sigma(S, y(S), X~)
    whenever A(X~) = 0 (Lemma 3.1)."""
    amap, cnt, b, D, Xt, T, sigma = _bqp_state(4, 5, sigma=3.0)
    n, m = amap.shape[0], cnt.size
    Y = random_unit_factor(n, 3, 11)
    U = sp.project(Y, random_matrix(n, 3, 12))
    out = sp.alm_eval(T, amap, cnt, None, sigma, Y, U)
    S = Y @ Y.T
    yS = ops.y_update(amap, cnt, S, None)
    G = sp.grad_Phi(S, yS, Xt, D, None, amap, sigma)
    np.testing.assert_allclose(out["R"], (2.0 / sigma) * sp.paper_grad(G, Y), atol=1e-11)
    np.testing.assert_allclose(out["H"], (2.0 / sigma) * sp.paper_hess(G, Y, U, amap, cnt, sigma), atol=1e-11)
    L = sp.L_sigma(S, yS, Xt, D, None, amap, sigma)
    assert abs(0.5 * sigma * out["f"] - np.sum(T * T) / (2 * sigma) - L) <= 1e-10 * (1 + abs(L))
    # y(S) minimises L_sigma over y (Lemma 3.1 / closed form)
    for s in range(3):
        yy = yS + 1e-3 * random_matrix(m, 1, 30 + s)[:, 0]
        assert sp.L_sigma(S, yy, Xt, D, None, amap, sigma) > L


def test_fixed_matches_paper_eq46_and_Lsigma():
    """Fixed-M: grad matches Eq. 4.6 and (sigma/2) f differs from L_sigma(S, y, X~)
    by a Y-independent constant."""
    amap, cnt, b, D, Xt, T, sigma = _bqp_state(4, 6, sigma=1.5, lemma31=False)
    n, m = amap.shape[0], cnt.size
    y = random_matrix(m, 1, 40)[:, 0]
    M = ops.At(amap, y) - T / sigma
    Ys = [random_unit_factor(n, 3, 50 + s) for s in range(3)]
    diffs = []
    for Y in Ys:
        S = Y @ Y.T
        out = sp.fixed_eval(M, Y)
        diffs.append(0.5 * sigma * out["f"] - sp.L_sigma(S, y, Xt, D, None, amap, sigma))
        G = sp.grad_Phi(S, y, Xt, D, None, amap, sigma)
        np.testing.assert_allclose(out["R"], (2.0 / sigma) * sp.paper_grad(G, Y), atol=1e-11)
        U = sp.project(Y, random_matrix(n, 3, 60))
        H = sp.fixed_eval(M, Y, U)["H"]
        np.testing.assert_allclose(H, (2.0 / sigma) * sp.paper_hess(G, Y, U, amap, cnt, sigma, False), atol=1e-11)
    assert np.ptp(diffs) <= 1e-9 * (1 + abs(diffs[0]))


def test_saddle_escape_identity():
    """At ([Y, 0], [0, V]) the Hessian equals 4 X_f U with
    X_f = (S - M) - Diag(diag((S - M) S)) (P:293-297 on the f scale)."""
    n, p, dl = 20, 3, 2
    M = random_symmetric(n, 9)
    Y = random_unit_factor(n, p, 9)
    S = Y @ Y.T
    Xf = (S - M) - np.diag(np.diag((S - M) @ S))
    V = np.linalg.qr(random_matrix(n, dl, 10))[0]
    Yp = np.hstack([Y, np.zeros((n, dl))])
    U = np.hstack([np.zeros((n, p)), V])
    out = sp.fixed_eval(M, Yp, U)
    np.testing.assert_allclose(out["H"], 4.0 * Xf @ U, atol=1e-12)
    assert abs(sp.inner(U, out["R"])) <= 1e-12


def _ncm_higham(M, iters=4000):
    """Nearest correlation matrix by alternating projections with Dykstra's
    correction (Higham 2002): a textbook routine independent of the oracle."""
    Yk = M.copy()
    dS = np.zeros_like(M)
    for _ in range(iters):
        R = Yk - dS
        w, V = np.linalg.eigh(R)
        X = (V * np.maximum(w, 0)) @ V.T
        dS = X - R
        Yk = X.copy()
        np.fill_diagonal(Yk, 1.0)
    return Yk


def test_fixed_subproblem_is_nearest_correlation_matrix():
    """Under fixed-M, min over the oblique manifold of ||YY^T - M||^2 with p = n is
    the nearest-correlation-matrix problem (P7); RTR must reach its optimal value."""
    from oracle.rtr import RTRParams, rtr

    n = 12
    M = random_symmetric(n, 21, 0.6) + np.eye(n)
    S_ncm = _ncm_higham(M)
    f_ncm = np.sum((S_ncm - M) ** 2)
    prob = sp.FixedMProblem(M)
    Y, info = rtr(prob, random_unit_factor(n, n, 3), RTRParams(n, n), 1e-10)
    assert abs(info["f"] - f_ncm) <= 1e-7 * (1 + f_ncm)


def test_alm_cost_forms_agree():
    """The accurate evaluation of f^ equals its defining expression
    ||S + C + T/sigma||^2 - sum_a A(S+C)_a^2/cnt_a (up to rounding of the latter)."""
    amap, cnt, b, D, Xt, T, sigma = _bqp_state(5, 4, sigma=7.0, lemma31=False)
    n, m = amap.shape[0], cnt.size
    C = random_symmetric(n, 77, 0.1)
    for s in range(3):
        Y = random_unit_factor(n, 4, 80 + s)
        S = Y @ Y.T
        a = ops.A(amap, S + C, m)
        ref = np.sum((S + C + T / sigma) ** 2) - np.sum(a * a / cnt)
        assert abs(sp.alm_cost(T, amap, cnt, C, sigma, Y) - ref) <= 1e-12 * np.sum((S + C + T / sigma) ** 2)
        f, _, _ = sp.ALMProblem(T, amap, cnt, C, sigma).costgrad(Y)
        assert f == sp.alm_cost(T, amap, cnt, C, sigma, Y) or abs(f - ref) <= 1e-12 * abs(ref)


# ---- pins of the row-sampled / blocked / RTR-callable copies ------------
@pytest.mark.parametrize("p", [1, 16, 64])
def test_fixed_rows_match_fixed_eval(p):
    """fixed_rows (the checker of the n = 16384 / 32768 GPU tests and of the bench's
    cpu_baseline) equals the FD-pinned fixed_eval row by row (E, rho, R, H)."""
    n = 200
    M = random_symmetric(n, 31 + p, 1.0 / np.sqrt(n))
    Y = random_unit_factor(n, p, 32)
    U = sp.project(Y, random_matrix(n, p, 33))
    full = sp.fixed_eval(M, Y, U)
    rows = np.array([0, 1, 7, 64, 127, 128, 150, 199])
    part = sp.fixed_rows(M[rows], rows, Y, U)
    for key in ("E", "R", "H"):
        scale = max(1.0, np.abs(full[key]).max())
        assert np.abs(part[key] - full[key][rows]).max() <= 1e-13 * scale, key
    assert np.abs(part["rho"] - full["rho"][rows]).max() <= 1e-13 * max(1.0, np.abs(full["rho"]).max())


@pytest.mark.parametrize("block", [1, 37, 64, 1024])
def test_fixed_cost_blocked_matches_fixed_cost(block):
    n, p = 150, 8
    M = random_symmetric(n, 41, 0.2)
    Y = random_unit_factor(n, p, 42)
    ref = sp.fixed_eval(M, Y)["f"]
    f = sp.fixed_cost_blocked(lambda i0, i1: M[i0:i1], Y, block)
    assert abs(f - ref) <= 1e-13 * ref
    assert abs(sp.fixed_cost(M, Y) - ref) <= 1e-13 * ref


@pytest.mark.parametrize("with_C", [False, True])
def test_alm_problem_matches_alm_eval(with_C):
    """ALMProblem.costgrad / .hess (the copies RTR drives) equal the FD-pinned alm_eval:
    f, R (costgrad) and H (hess at the cached point)."""
    amap, cnt, b, D, Xt, T, sigma = _bqp_state(5, 9, sigma=2.5, lemma31=not with_C)
    n = amap.shape[0]
    C = random_symmetric(n, 91, 0.05) if with_C else None
    prob = sp.ALMProblem(T, amap, cnt, C, sigma)
    for s in range(2):
        Y = random_unit_factor(n, 4, 92 + s)
        U = sp.project(Y, random_matrix(n, 4, 94 + s))
        ref = sp.alm_eval(T, amap, cnt, C, sigma, Y, U)
        f, R, ctx = prob.costgrad(Y)
        H = prob.hess(ctx, U)
        assert abs(f - ref["f"]) <= 1e-13 * max(1.0, abs(ref["f"]))
        assert np.abs(R - ref["R"]).max() <= 1e-12 * max(1.0, np.abs(ref["E"]).max())
        assert np.abs(H - ref["H"]).max() <= 1e-12 * max(1.0, np.abs(ref["H"]).max())
    assert prob.n_costgrad == 2 and prob.n_hvp == 2


def test_alm_problem_taylor_slopes():
    """ALMProblem itself passes the Taylor-slope checks (slope 2 for the gradient, 3 with the
    Hessian term) with a nonzero C, independently of alm_eval."""
    amap, cnt, b, D, Xt, T, sigma = _bqp_state(4, 12, sigma=1.7, lemma31=False)
    n = amap.shape[0]
    C = random_symmetric(n, 120, 0.05)
    prob = sp.ALMProblem(T, amap, cnt, C, sigma)
    Y = random_unit_factor(n, 3, 121)
    U = sp.project(Y, random_matrix(n, 3, 122))

    def cg(Yx):
        f, R, _ = prob.costgrad(Yx)
        return f, R

    def hs(Yx, Ux):
        _, _, ctx = prob.costgrad(Yx)
        return prob.hess(ctx, Ux)

    _fd_checks(cg, hs, Y, U)
