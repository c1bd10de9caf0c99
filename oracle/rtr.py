"""Riemannian trust-region method with truncated CG (oracle).

PAPER.md:209 chooses RTR (Absil, Baker, Gallivan) run through Manopt without
stating parameters; this is the textbook method with the defaults of DESIGN.md
reading R12: Delta_bar = sqrt(n), Delta_0 = Delta_bar/8, rho' = 0.1,
kappa = 0.1, theta = 1, plus the standard rho-regularisation (reading R12).
Parity unpinned: iterates, inner iteration counts and accept/reject decisions are
trajectory quantities (P17); the properties pinned by tests are the
invariants (monotone accepted cost, ||eta|| <= Delta, Cauchy decrease, determinism).
"""
from __future__ import annotations

import math

import numpy as np

from .subproblem import inner, project, retract


class RTRParams:
    def __init__(self, n, p, max_iter=500, max_tcg=None, rho_prime=0.1, kappa=0.1, theta=1.0,
                 delta_bar=None, delta0=None, rho_reg=1e3, precond_mu=0.0):
        self.delta_bar = math.sqrt(n) if delta_bar is None else delta_bar
        self.delta0 = self.delta_bar / 8.0 if delta0 is None else delta0
        self.rho_prime = rho_prime
        self.kappa = kappa
        self.theta = theta
        self.max_iter = max_iter
        self.max_tcg = max(1, n * (p - 1)) if max_tcg is None else max_tcg
        self.rho_reg = rho_reg
        self.precond_mu = precond_mu


def gram_preconditioner(Y, mu):
    """Right preconditioner of the truncated CG (reading R35), an SPD operator on the
    tangent space at Y:  Prec(R) = P_Y(R W),  W = gbar (G + mu gbar I)^{-1},  G = Y^T Y,
    gbar = tr(G)/p.  Returns None (identity) when mu <= 0."""
    if mu <= 0:
        return None
    G = Y.T @ Y
    gbar = np.trace(G) / G.shape[0]
    W = gbar * np.linalg.inv(G + mu * gbar * np.eye(G.shape[0]))
    W = 0.5 * (W + W.T)
    return lambda R: project(Y, R @ W)


def tcg(prob, ctx, Y, g, Delta, prm: RTRParams, prec=None):
    """Steihaug-Toint truncated CG on the model m(eta) = f + <g,eta> + 1/2 <eta, H eta>, with an
    optional preconditioner prec (SPD on the tangent space; the trust region is then measured
    in the norm <eta, prec^{-1} eta>, tracked by the e_Pe / e_Pd / d_Pd recurrences).

    Returns (eta, Heta, n_inner, hit_boundary)."""
    eta = np.zeros_like(Y)
    Heta = np.zeros_like(Y)
    r = g.copy()
    r_r = inner(r, r)
    norm_r0 = math.sqrt(r_r)
    z = r if prec is None else prec(r)
    z_r = inner(z, r)
    delta = -z
    e_Pe, e_Pd, d_Pd = 0.0, 0.0, z_r
    model = 0.0
    hit = False
    j = 0
    for j in range(1, prm.max_tcg + 1):
        Hdelta = prob.hess(ctx, delta)
        d_Hd = inner(delta, Hdelta)
        alpha = z_r / d_Hd if d_Hd != 0 else math.inf
        e_Pe_new = e_Pe + 2.0 * alpha * e_Pd + alpha * alpha * d_Pd
        if d_Hd <= 0 or e_Pe_new >= Delta * Delta:
            tau = (-e_Pd + math.sqrt(e_Pd * e_Pd + d_Pd * (Delta * Delta - e_Pe))) / d_Pd
            eta = eta + tau * delta
            Heta = Heta + tau * Hdelta
            hit = True
            break
        new_eta = eta + alpha * delta
        new_Heta = Heta + alpha * Hdelta
        new_model = inner(new_eta, g) + 0.5 * inner(new_eta, new_Heta)
        if new_model >= model:  # no model decrease: keep previous eta (Manopt-style guard)
            break
        eta, Heta, model, e_Pe = new_eta, new_Heta, new_model, e_Pe_new
        r = r + alpha * Hdelta
        r_r = inner(r, r)
        if math.sqrt(r_r) <= norm_r0 * min(norm_r0 ** prm.theta, prm.kappa):
            break
        z = r if prec is None else prec(r)
        z_r_old = z_r
        z_r = inner(z, r)
        beta = z_r / z_r_old
        delta = project(Y, -z + beta * delta)
        e_Pd = beta * (e_Pd + alpha * d_Pd)
        d_Pd = z_r + beta * beta * d_Pd
    return eta, Heta, j, hit


def rtr(prob, Y, prm: RTRParams, grad_tol: float, warm_U=None, max_halvings=25, stall=0, stall_factor=100.0):
    """Minimise prob over the oblique manifold from Y. Returns (Y, info dict).

    warm_U: optional second-order descent direction (Thm 4.5); a curvilinear
    backtracking Y(t) = retract(Y, t U), t = 1, 1/2, ..., is tried first until the
    cost decreases (reading R14).
    """
    f, g, ctx = prob.costgrad(Y)
    info = {"iters": 0, "tcg": 0, "accepted": 0, "warm_t": None}
    if warm_U is not None:
        t = 1.0
        for _ in range(max_halvings):
            try:
                Yt = retract(Y, t * warm_U)
            except FloatingPointError:
                t *= 0.5
                continue
            ft, gt, ctxt = prob.costgrad(Yt)
            if ft < f:
                Y, f, g, ctx = Yt, ft, gt, ctxt
                info["warm_t"] = t
                break
            t *= 0.5
    Delta = prm.delta0
    gn = math.sqrt(inner(g, g))
    best_gn, since_best = gn, 0
    for it in range(prm.max_iter):
        if gn <= grad_tol:
            break
        # stagnation exit (reading R30): ||grad|| has not halved within `stall`
        # iterations and is within 100x of the tolerance
        if gn <= 0.5 * best_gn:
            best_gn, since_best = gn, 0
        else:
            since_best += 1
            if stall > 0 and since_best > stall and gn <= stall_factor * grad_tol:
                break
        info["iters"] += 1
        eta, Heta, nin, hit = tcg(prob, ctx, Y, g, Delta, prm, gram_preconditioner(Y, prm.precond_mu))
        info["tcg"] += nin
        try:
            Yp = retract(Y, eta)
        except FloatingPointError:
            Delta /= 4.0
            continue
        fp, gp, ctxp = prob.costgrad(Yp)
        rhonum = f - fp
        rhoden = -inner(g, eta) - 0.5 * inner(eta, Heta)
        reg = max(1.0, abs(f)) * np.finfo(float).eps * prm.rho_reg
        rhonum += reg
        rhoden += reg
        rho = rhonum / rhoden
        if not math.isfinite(fp):
            raise FloatingPointError("non-finite cost")
        if rho < 0.25:
            Delta /= 4.0
        elif rho > 0.75 and hit:
            Delta = min(2.0 * Delta, prm.delta_bar)
        if rhoden >= 0 and rho > prm.rho_prime:
            Y, f, g, ctx = Yp, fp, gp, ctxp
            gn = math.sqrt(inner(g, g))
            info["accepted"] += 1
        if Delta < 1e-300:
            break
    info["f"] = f
    info["gnorm"] = gn
    return Y, info
