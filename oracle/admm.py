"""ManiDSDP, Algorithm 2, oracle.

State is kept as T = X~ + D (reading R3): A(X~) = 0 <=> A(T) = b (Lemma 3.1).
Per outer iteration k:
  3. solve (Sub-k) inexactly by RTR, warm direction U
  4. S = Y Y^T
  5. y = (AA*)^{-1} A(S + C)
  6. X~ <- X~ - sigma (A*(y) - S - C)   i.e.  T <- T - sigma R
  7. z = diag((X~ + D) S) = rowdot(T Y, Y)
  8. X = X~ + D - Diag(z) = T - Diag(z)
  9. escape direction from the negative eigenvectors of X        (Thm 4.5)
 10. p update (rank reduction / growth)                          (reading R15)
 11. sigma update, Eq. 5.1
KKT residues with the eta_g reading R7.
Parity: the final objective and residues are pinned (weak duality, brute force,
certificates); the trajectory (Y^k, p^k, escapes, iteration counts) is "parity
unpinned" (P17).
"""
from __future__ import annotations

import math
import time

import numpy as np

from . import operators as ops
from .rtr import RTRParams, rtr
from .subproblem import ALMProblem, FixedMProblem, rowdot

TRACE_COLUMNS = ("iter", "eta_p", "eta_d", "eta_g", "eta_max", "primal_obj", "dual_obj", "sigma",
                 "p", "inner_iters", "cg_iters", "escape_delta", "time_s")


class Params:
    """Alg. 2 inputs and the unspecified constants (readings R9-R16)."""

    def __init__(self, **kw):
        self.sigma0 = 1.0
        self.sigma_min = 1e-3
        self.sigma_max = 1e7
        self.gamma = 2.0
        self.tau1 = 0.1
        self.tau2 = 1.0
        self.tol = 1e-8
        self.eig_neg_tol = 1e-9
        self.rank_tol = 1e-4
        self.p0 = 2
        self.max_outer = 300
        self.max_rtr = 500
        self.escape_max = 8
        self.mode = "alm"
        self.eps_scale = 1e-2
        self.eps_floor = 1e-12
        self.rho_reg = 1e3
        self.stall_rtr = 10
        self.max_tcg = 100
        self.precond_mu = -1.0  # reading R35: Gram right-preconditioner of the truncated CG (0 = off,
                                # < 0 = auto: mu = 0.1 for 2048 <= n < 8192, off otherwise)
        self.stall_factor = 100.0  # reading R30: the stagnation exit applies within this x the tolerance
        self.escape_gate = 0.0  # reading R36: escape / rank change only after an inner solve within
                                # escape_gate x its tolerance (0 = always)
        self.hold_max = 0  # reading R40: at most this many consecutive multiplier holds (0 = never)
        self.hold_tau = 0.0  # reading R40: hold while eta_d(X^{k+1}) > hold_tau min(1, eta_p) (Thm 5.3's
                             # lambda_min(X^{k+1}) >= -tau_k, enforced by escapes)
        self.sigma_boost = 0.0  # reading R41: when eta_d <= sigma_boost * eta_p, sigma_{k+1} = min(gamma sigma_k,
                                # sigma_max) whatever Eq. 5.1 says (Alg. 1 step 8 "certain policy"); 0 = off
        for k, v in kw.items():
            if not hasattr(self, k):
                raise TypeError(f"unknown parameter {k}")
            setattr(self, k, v)


def eta_d_of(lam_min: float, lam_max: float) -> float:
    """eta_d = max(0, -lambda_min(X)) / (1 + |lambda_max(X)|)."""
    return max(0.0, -lam_min) / (1.0 + abs(lam_max))


def residues(amap, cnt, b, C, y, Y, T):
    """eta_p, eta_d, eta_g and the objectives of a tuple (y, S = YY^T, X = T - Diag z).

    eta_p = ||A*(y) - S - C|| / (1 + ||C||)
    eta_d = max(0, -lambda_min(X)) / (1 + |lambda_max(X)|)
    eta_g = |b^T y - pobj| / (1 + |b^T y| + |pobj|),  pobj = <C, X + Diag z> + 1^T z
                                                             (P:451 read as R7)
    """
    S = Y @ Y.T
    SC = S if C is None else S + C
    R = ops.At(amap, y) - SC
    z = rowdot(T @ Y, Y)
    X = T - np.diag(z)
    lam, V = np.linalg.eigh(X)
    nC = 0.0 if C is None else float(np.linalg.norm(C))
    eta_p = float(np.linalg.norm(R)) / (1.0 + nC)
    eta_d = eta_d_of(lam[0], lam[-1])
    dobj = float(b @ y)
    pobj = (0.0 if C is None else float(np.sum(C * T))) + float(np.sum(z))
    eta_g = abs(dobj - pobj) / (1.0 + abs(dobj) + abs(pobj))
    return {"eta_p": eta_p, "eta_d": eta_d, "eta_g": eta_g, "eta_max": max(eta_p, eta_d, eta_g),
            "dual_obj": dobj, "primal_obj": pobj, "z": z, "X": X, "lam": lam, "V": V, "R": R}


def escape_directions(lam, V, eig_neg_tol, escape_max):
    """Eigenvectors of X with lambda < -eig_neg_tol (1 + |lambda_max|), most negative
    first, at most escape_max; sign fixed so the largest-|.| entry is positive
    (Thm 4.5; readings R14, R25)."""
    thresh = -eig_neg_tol * (1.0 + abs(lam[-1]))
    idx = [i for i in range(lam.size) if lam[i] < thresh][:escape_max]
    if not idx:
        return None
    Vs = V[:, idx].copy()
    for j in range(Vs.shape[1]):
        k = int(np.argmax(np.abs(Vs[:, j])))
        if Vs[k, j] < 0:
            Vs[:, j] = -Vs[:, j]
    return Vs


def rank_reduce(Y, rank_tol):
    """Compress Y to its numerical rank r (singular values >= rank_tol * largest),
    Y <- Y W_r, rows renormalised (reading R15). Keeps p >= 1."""
    G = Y.T @ Y
    ev, W = np.linalg.eigh(G)  # ascending
    keep = ev > (rank_tol ** 2) * ev[-1]
    r = max(1, int(np.sum(keep)))
    if r >= Y.shape[1]:
        return Y
    Yr = Y @ W[:, -r:]
    return Yr / np.linalg.norm(Yr, axis=1, keepdims=True)


def sigma_update(sigma, R_norm, b_norm, grad_norm, prm: Params):
    """Eq. 5.1; grad_norm = ||grad Psi_k(Y^{k+1})|| on the paper scale."""
    ratio = R_norm / (1.0 + b_norm)
    if ratio < prm.tau1 * grad_norm:
        return max(sigma / prm.gamma, prm.sigma_min)
    if ratio > prm.tau2 * grad_norm:
        return min(prm.gamma * sigma, prm.sigma_max)
    return sigma


def solve(amap, cnt, b, C, prm: Params, Y0: np.ndarray, verbose=False, callback=None):
    """Algorithm 2. Returns a dict with y, Y, z, X (via T), residues, trace, status."""
    t0 = time.perf_counter()
    n = amap.shape[0]
    m = cnt.size
    ops.check_assumption2(cnt)
    D = ops.D_matrix(amap, cnt, b)
    T = D.copy()  # X~^0 = 0
    y = np.zeros(m)  # y^0 = 0
    sigma = prm.sigma0
    Y = Y0.copy()
    U = None
    eta_prev = 1.0
    b_norm = float(np.linalg.norm(b))
    trace = []
    status = "not_converged"
    res = None
    totals = {"rtr": 0, "tcg": 0, "costgrad": 0, "hvp": 0, "p_max": Y.shape[1]}
    holds = 0
    for k in range(prm.max_outer):
        p = Y.shape[1]
        if prm.mode == "alm":
            prob = ALMProblem(T, amap, cnt, C, sigma)
        else:
            M = ops.At(amap, y) - T / sigma
            if C is not None:
                M = M - C
            prob = FixedMProblem(M)
        eps_k = max(0.1 * min(1.0, eta_prev) * prm.eps_scale, prm.eps_floor)  # ||XY|| scale
        grad_tol = 4.0 * eps_k / sigma  # f scale: ||XY|| = sigma/4 ||R||
        Y, info = rtr(prob, Y, RTRParams(n, p, max_iter=prm.max_rtr, rho_reg=prm.rho_reg,
                                        max_tcg=prm.max_tcg if prm.max_tcg > 0 else None,
                                        precond_mu=(prm.precond_mu if prm.precond_mu >= 0 else
                                                    (0.1 if 2048 <= n < 8192 else 0.0))), grad_tol, warm_U=U,
                      stall=prm.stall_rtr, stall_factor=prm.stall_factor)
        totals["rtr"] += info["iters"]
        totals["tcg"] += info["tcg"]
        totals["costgrad"] += prob.n_costgrad
        totals["hvp"] += prob.n_hvp
        grad_paper = 0.5 * sigma * info["gnorm"]
        S = Y @ Y.T
        y = ops.y_update(amap, cnt, S, C)
        SC = S if C is None else S + C
        Rp = ops.At(amap, y) - SC
        T_prev = T
        T = T - sigma * Rp
        res = residues(amap, cnt, b, C, y, Y, T)
        if callback is not None:
            callback(k + 1, {"T": T, "y": y, "Y": Y, "sigma": sigma, "res": res})
        delta = 0
        row = {"iter": k + 1, **{c: res[c] for c in ("eta_p", "eta_d", "eta_g", "eta_max",
                                                       "primal_obj", "dual_obj")},
               "sigma": sigma, "p": p, "inner_iters": info["iters"], "cg_iters": info["tcg"]}
        if verbose:
            print(f"k={k+1:3d} p={p:3d} sigma={sigma:9.3e} eta_p={res['eta_p']:.2e} "
                  f"eta_d={res['eta_d']:.2e} eta_g={res['eta_g']:.2e} dobj={res['dual_obj']:.10f} "
                  f"rtr={info['iters']} tcg={info['tcg']} |R|={info['gnorm']:.2e}")
        if res["eta_max"] <= prm.tol:
            status = "converged"
            row["escape_delta"] = 0
            row["time_s"] = time.perf_counter() - t0
            trace.append(row)
            break
        Vs = escape_directions(res["lam"], res["V"], prm.eig_neg_tol, prm.escape_max)
        if Vs is not None and Y.shape[1] + Vs.shape[1] > n:  # p never exceeds n (S has rank <= n)
            Vs = Vs[:, : n - Y.shape[1]] if Y.shape[1] < n else None
        # escape gate (reading R36): X^{k+1} certifies the subproblem (Prop 4.3) only at a
        # stationary point; an inner solve far above its tolerance keeps the rank unchanged
        gated = prm.escape_gate > 0 and info["gnorm"] > prm.escape_gate * grad_tol
        if gated:
            Vs = None
        # multiplier hold (reading R40): X^{k+1} = grad Phi_k(S^{k+1}) - Diag(z) is subproblem k's
        # certificate (Lemma 3.2, Prop 4.3); while it has escape directions and
        # eta_d > hold_tau min(1, eta_p), undo step 6, keep sigma, escape and re-solve subproblem k
        hold = (prm.hold_max > 0 and prm.hold_tau > 0 and holds < prm.hold_max and Vs is not None
                and res["eta_d"] > prm.hold_tau * min(1.0, res["eta_p"]))
        # rank tolerance tied to the residual (reading R32); no reduction in an iteration that
        # escapes (reading R34: the escape columns of the previous iteration are O(sqrt(|lambda|/sigma))
        # and a relative tolerance would remove them before they grow)
        if Vs is None and not gated:
            Y = rank_reduce(Y, min(prm.rank_tol, max(1e-8, 0.01 * math.sqrt(res["eta_max"]))))
        if Vs is not None:
            delta = Vs.shape[1]
            pr = Y.shape[1]
            Y = np.hstack([Y, np.zeros((n, delta))])
            U = np.hstack([np.zeros((n, pr)), Vs])
        else:
            U = None
        totals["p_max"] = max(totals["p_max"], Y.shape[1])
        if hold:
            T = T_prev
            holds += 1
            row["escape_delta"] = -delta  # negative: the multiplier was held
            row["time_s"] = time.perf_counter() - t0
            trace.append(row)
            continue
        holds = 0
        sigma_new = sigma_update(sigma, float(np.linalg.norm(Rp)), b_norm, grad_paper, prm)
        if prm.sigma_boost > 0 and res["eta_d"] <= prm.sigma_boost * res["eta_p"]:
            sigma_new = min(prm.gamma * sigma, prm.sigma_max)  # reading R41
        row["escape_delta"] = delta
        row["time_s"] = time.perf_counter() - t0
        trace.append(row)
        sigma = sigma_new
        eta_prev = res["eta_max"]
    return {"status": status, "y": y, "Y": Y if status == "converged" else Y, "T": T,
            "z": res["z"], "X": res["X"], "eta_p": res["eta_p"], "eta_d": res["eta_d"],
            "eta_g": res["eta_g"], "eta_max": res["eta_max"], "dual_obj": res["dual_obj"],
            "primal_obj": res["primal_obj"], "trace": trace, "outer_iters": len(trace),
            "seconds": time.perf_counter() - t0, **totals}
