"""Pins for oracle/admm.py (DESIGN.md "Oracle pins" P8-P14): sigma rule branches,
residue special cases, escape (Thm 4.5), rank reduction, Lemma 3.1 invariant and the
final result against brute force / weak duality."""
import json
import os

import numpy as np
import pytest

from inputs import bqp_instance, initial_factor, random_matrix, random_symmetric, random_unit_factor
from oracle import admm, bqp
from oracle import operators as ops
from oracle import subproblem as sp

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_spec_examples.json")))


def test_sigma_rule_branches():
    prm = admm.Params(sigma_min=1e-3, sigma_max=1e7, gamma=2.0, tau1=0.1, tau2=1.0)
    # ratio = R/(1+|b|); b_norm = 1 => ratio = R/2
    assert admm.sigma_update(4.0, 2 * 0.05, 1.0, 1.0, prm) == 2.0           # ratio .05 < .1 g
    assert admm.sigma_update(2e-3, 2 * 0.05, 1.0, 1.0, prm) == 1e-3         # clipped at sigma_min
    assert admm.sigma_update(4.0, 2 * 2.0, 1.0, 1.0, prm) == 8.0            # ratio 2 > 1 g
    assert admm.sigma_update(6e6, 2 * 2.0, 1.0, 1.0, prm) == 1e7            # clipped at sigma_max
    assert admm.sigma_update(4.0, 2 * 0.5, 1.0, 1.0, prm) == 4.0            # in between
    assert admm.sigma_update(4.0, 2 * 0.1, 1.0, 1.0, prm) == 4.0            # boundary tau1 (not <)
    assert admm.sigma_update(4.0, 2 * 1.0, 1.0, 1.0, prm) == 4.0            # boundary tau2 (not >)


def test_eta_d_golden():
    g = GOLD["eta_d_diag"]
    lam = np.linalg.eigvalsh(np.array(g["X"], float))
    assert admm.eta_d_of(lam[0], lam[-1]) == pytest.approx(g["eta_d"], rel=1e-15)
    assert admm.eta_d_of(0.0, 0.0) == 0.0


def test_escape_direction_theorem():
    """Thm 4.5: U = [0, V] satisfies <U, grad> = 0 and
    <U, Hess U> = 4 sum v^T X_f v < 0 at [Y, 0] (f scale)."""
    n, p = 24, 3
    M = random_symmetric(n, 1)
    Y = random_unit_factor(n, p, 2)
    S = Y @ Y.T
    Xf = (S - M) - np.diag(np.diag((S - M) @ S))
    lam, V = np.linalg.eigh(Xf)
    Vs = admm.escape_directions(lam, V, 1e-9, 3)
    assert Vs is not None and Vs.shape[1] == min(3, int(np.sum(lam < -1e-9 * (1 + abs(lam[-1])))))
    Yp = np.hstack([Y, np.zeros((n, Vs.shape[1]))])
    U = np.hstack([np.zeros((n, p)), Vs])
    out = sp.fixed_eval(M, Yp, U)
    assert abs(sp.inner(U, out["R"])) <= 1e-12
    curv = sp.inner(U, out["H"])
    assert curv < 0
    assert abs(curv - 4.0 * np.trace(Vs.T @ Xf @ Vs)) <= 1e-10 * abs(curv)
    # PSD X -> no direction; spec example X = Diag(1,-2,3) -> e_2
    assert admm.escape_directions(np.array([0.0, 1.0]), np.eye(2), 1e-9, 3) is None
    lam, V = np.linalg.eigh(np.diag([1.0, -2.0, 3.0]))
    Vs = admm.escape_directions(lam, V, 1e-9, 3)
    np.testing.assert_array_equal(Vs[:, 0], [0.0, 1.0, 0.0])


def test_rank_reduction_keeps_S():
    n = 30
    Y = random_unit_factor(n, 3, 4)
    Yp = np.hstack([Y @ np.linalg.qr(random_matrix(3, 3, 5))[0], np.zeros((n, 2))])  # rank 3, p = 5
    Yr = admm.rank_reduce(Yp, 1e-6)
    assert Yr.shape[1] == 3
    assert np.abs(Yr @ Yr.T - Y @ Y.T).max() <= 1e-12
    assert admm.rank_reduce(Y, 1e-6) is Y


def _solve(d, seed, **kw):
    Q, c = bqp_instance(d, seed)
    amap, cnt, b = bqp.relax(Q, c)
    prm = admm.Params(**kw)
    Y0 = initial_factor(amap.shape[0], prm.p0, seed)
    return Q, c, amap, cnt, b, prm, Y0


def test_toy_q2():
    g = GOLD["toy_bqp"]
    Q, c = np.array(g["Q"], float), np.array(g["c"], float)
    amap, cnt, b = bqp.relax(Q, c)
    out = admm.solve(amap, cnt, b, None, admm.Params(p0=2), initial_factor(4, 2, 0))
    assert out["status"] == "converged"
    assert abs(out["dual_obj"] - g["min"]) <= 1e-6


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_d10_solve_brute_force_and_invariants(seed):
    Q, c, amap, cnt, b, prm, Y0 = _solve(10, seed, p0=2)
    m = cnt.size
    lemma = []

    def cb(k, st):  # Lemma 3.1: A(X~^k) = 0 <=> A(T^k) = b at every k
        T = st["T"]
        lemma.append(np.linalg.norm(ops.A(amap, T, m) - b) / (1 + np.linalg.norm(T - ops.D_matrix(amap, cnt, b))))

    out = admm.solve(amap, cnt, b, None, prm, Y0, callback=cb)
    assert out["status"] == "converged" and out["eta_max"] <= 1e-8
    assert max(lemma) <= 1e-8
    bf, xbf = bqp.brute_force(Q, c)
    # lower-bound property (weak duality) and tightness via the rank-one certificate
    assert out["dual_obj"] <= bf + 1e-6
    Y = out["Y"]
    assert np.abs(np.linalg.norm(Y, axis=1) - 1).max() <= 1e-12
    ev = np.linalg.eigvalsh(Y.T @ Y)
    if ev.size == 1 or ev[-2] <= 1e-8 * ev[-1]:  # numerically rank one: round and certify
        x = np.sign(Y[1:11] @ Y[0])
        assert abs(bqp.bqp_value(Q, c, x) - out["dual_obj"]) <= 1e-6 * (1 + abs(bf))
    # recompute the residues from scratch on the returned tuple
    res = admm.residues(amap, cnt, b, None, out["y"], out["Y"], out["T"])
    assert res["eta_max"] <= 1e-8
    # y_1 = 1 <=> diag(S) = 1
    assert abs(out["y"][0] - 1.0) <= 1e-8


def test_p_update_escape_xor_reduce():
    """Readings R15/R34: an outer iteration either pads Y with its escape columns (p_{k+1} =
    p_k + delta_k exactly) or, when X has no escape directions, compresses Y (p_{k+1} <= p_k)."""
    for d, seed in ((10, 0), (12, 1)):
        Q, c, amap, cnt, b, prm, Y0 = _solve(d, seed, p0=2)
        tr = admm.solve(amap, cnt, b, None, prm, Y0)["trace"]
        assert any(r["escape_delta"] > 0 for r in tr)
        for r0, r1 in zip(tr, tr[1:]):
            if r0["escape_delta"] > 0:
                assert r1["p"] == r0["p"] + r0["escape_delta"]
            else:
                assert r1["p"] <= r0["p"]


def test_residue_diving_behaviour():
    """Residue diving (Fig. 3): the last outer iteration drops
    log10 eta_max by >= 4 decades on at least 2 of 3 q = 10 instances (measured with the
    readings R30-R34: 7.9, 5.8 and 3.5 decades for seeds 0, 1, 2)."""
    dives = 0
    for seed in range(3):
        Q, c, amap, cnt, b, prm, Y0 = _solve(10, seed, p0=2)
        tr = admm.solve(amap, cnt, b, None, prm, Y0)["trace"]
        drop = np.log10(tr[-2]["eta_max"]) - np.log10(tr[-1]["eta_max"]) if len(tr) >= 2 else 0.0
        dives += drop >= 4
    assert dives >= 2


def test_determinism():
    Q, c, amap, cnt, b, prm, Y0 = _solve(6, 3, p0=2)
    a = admm.solve(amap, cnt, b, None, prm, Y0)["trace"]
    bb = admm.solve(amap, cnt, b, None, prm, Y0)["trace"]
    strip = lambda tr: [{k: v for k, v in r.items() if k != "time_s"} for r in tr]
    assert strip(a) == strip(bb)


@pytest.mark.parametrize("d,seed", [(5, 0), (7, 1), (8, 2), (12, 3)])
def test_lower_bound_property(d, seed):
    Q, c, amap, cnt, b, prm, Y0 = _solve(d, seed, p0=2)
    out = admm.solve(amap, cnt, b, None, prm, Y0)
    assert out["status"] == "converged"
    assert out["dual_obj"] <= bqp.brute_force(Q, c)[0] + 1e-6


def test_preconditioned_tcg_operator_and_solve():
    """Reading R35: the Gram preconditioner Prec(R) = P_Y(R W) is self-adjoint and positive
    definite on the tangent space, reduces to W = I for an orthonormal-column Y at mu = 0 limit,
    and the preconditioned RTR reaches the same certified optimum (eta_max <= 1e-8, objective
    equal to the unpreconditioned solve's and below the brute-force minimum)."""
    from oracle.rtr import gram_preconditioner

    n, p = 30, 5
    Y = random_unit_factor(n, p, 3)
    P = gram_preconditioner(Y, 0.1)
    U = sp.project(Y, random_matrix(n, p, 4))
    V = sp.project(Y, random_matrix(n, p, 5))
    assert abs(sp.inner(V, P(U)) - sp.inner(U, P(V))) <= 1e-12 * abs(sp.inner(V, P(U)))
    assert sp.inner(U, P(U)) > 0 and np.abs(sp.rowdot(P(U), Y)).max() <= 1e-14
    assert gram_preconditioner(Y, 0.0) is None
    for seed in (0, 1):
        Q, c, amap, cnt, b, prm, Y0 = _solve(10, seed, p0=2, precond_mu=0.05)
        out = admm.solve(amap, cnt, b, None, prm, Y0)
        ref = admm.solve(amap, cnt, b, None, admm.Params(p0=2), Y0)
        assert out["status"] == "converged" and out["eta_max"] <= 1e-8
        assert abs(out["dual_obj"] - ref["dual_obj"]) <= 1e-6 * (1 + abs(ref["dual_obj"]))
        assert out["dual_obj"] <= bqp.brute_force(Q, c)[0] + 1e-6


def test_sigma_boost_reading_r41():
    """Reading R41: with sigma_boost > 0 the penalty is raised whenever eta_d <= sigma_boost * eta_p
    (whatever Eq. 5.1 says); the solve still reaches the brute-force-certified optimum of the tight d = 10
    instance, and the sigma trajectory differs from the plain Eq. 5.1 one."""
    Q, c, amap, cnt, b, prm, Y0 = _solve(10, 2, p0=2)
    plain = admm.solve(amap, cnt, b, None, prm, Y0)
    prm_b = admm.Params(p0=2, sigma_boost=0.5)
    boosted = admm.solve(amap, cnt, b, None, prm_b, Y0)
    assert boosted["status"] == "converged" and boosted["eta_max"] <= 1e-8
    assert abs(boosted["dual_obj"] - plain["dual_obj"]) <= 1e-6 * (1 + abs(plain["dual_obj"]))
    for r0, r1 in zip(boosted["trace"], boosted["trace"][1:]):
        if r0["eta_d"] <= 0.5 * r0["eta_p"]:
            assert r1["sigma"] == min(prm_b.gamma * r0["sigma"], prm_b.sigma_max)
    assert [r["sigma"] for r in boosted["trace"]] != [r["sigma"] for r in plain["trace"]][:len(boosted["trace"])]
