"""The oblique-manifold subproblem (Sub-k) and its derivatives (oracle).

PAPER.md:199-266 (§4). Everything is dense NumPy with S = Y Y^T formed explicitly;
no expansion tricks. Two readings of the subproblem (reading R2):

* fixed-M ("north-star literal", ADMM step 3.4a with y = y^k frozen):
      f(Y) = ||Y Y^T - M||_F^2,  M = A*(y^k) - C - T/sigma,  T = X~^k + D.
  L_sigma(YY^T, y^k, X~^k) = (sigma/2) f(Y) + const.
* ALM / y-eliminated (the reading under which Prop 4.2's Hessian, is exact):
      f^(Y) = ||S + C + T/sigma||^2 - sum_a A(S + C)_a^2 / cnt_a,   S = Y Y^T,
  which is (2/sigma) min_y L_sigma(S, y, X~) + const when A(X~) = 0 (Lemma 3.1).
  Its Euclidean gradient is 4 (S - M(S)) Y with M(S) = A*(y(S)) - C - T/sigma,
  y(S) = (AA*)^{-1} A(S + C).

Scale: the ABI and this oracle work on the f scale; Psi_k = (sigma/2) f + const, so
grad Psi_k = (sigma/2) R and ||X Y|| = (sigma/4) ||R||.
"""
from __future__ import annotations

import numpy as np

from . import operators as ops


def rowdot(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    return np.sum(A * B, axis=1)


def project(Y: np.ndarray, U: np.ndarray) -> np.ndarray:
    """P_Y(U) = U - Diag(U Y^T) Y (Lemma 4.1)."""
    return U - rowdot(U, Y)[:, None] * Y


def retract(Y: np.ndarray, U: np.ndarray) -> np.ndarray:
    """Row-normalisation retraction (reading R13).

    Raises FloatingPointError when a row of Y + U has norm <= 1e-14."""
    W = Y + U
    nrm = np.linalg.norm(W, axis=1)
    if np.any(nrm <= 1e-14):
        raise FloatingPointError("degenerate retraction row")
    return W / nrm[:, None]


def inner(A: np.ndarray, B: np.ndarray) -> float:
    return float(np.sum(A * B))


# ----------------------------------------------------------------------------------
# fixed-M subproblem: f = ||YY^T - M||^2
# ----------------------------------------------------------------------------------
def fixed_cost(M: np.ndarray, Y: np.ndarray) -> float:
    S = Y @ Y.T
    return float(np.sum((S - M) ** 2))


def fixed_eval(M: np.ndarray, Y: np.ndarray, U: np.ndarray | None = None) -> dict:
    """Cost, Euclidean gradient, Riemannian gradient (and HVP along U) of f.

    E = 4 (S - M) Y  (Euclidean gradient of ||YY^T - M||^2)
    R = P_Y(E) = E - rowdot(E, Y) o Y           (grad = 2XY on the Psi scale)
    H = P_Y(4 [Z Y + (S - M) U]) - rowdot(E, Y) o U,  Z = Y U^T + U Y^T
                                                  (P:234-239 with y frozen: no projection term)
    """
    S = Y @ Y.T
    W = S - M
    out = {"f": float(np.sum(W ** 2))}
    E = 4.0 * (W @ Y)
    rho = rowdot(E, Y)
    out["E"] = E
    out["rho"] = rho
    out["R"] = E - rho[:, None] * Y
    if U is not None:
        Z = Y @ U.T + U @ Y.T
        EH = 4.0 * (Z @ Y + W @ U)
        out["H"] = project(Y, EH) - rho[:, None] * U
    return out


# ----------------------------------------------------------------------------------
# ALM (y-eliminated) subproblem
# ----------------------------------------------------------------------------------
def alm_M(T, amap, cnt, C, sigma, S):
    """M(S) = A*(y(S)) - C - T/sigma with y(S) = (AA*)^{-1} A(S + C)."""
    yS = ops.y_update(amap, cnt, S, C)
    M = ops.At(amap, yS) - T / sigma
    if C is not None:
        M = M - C
    return M, yS


def alm_cost(T, amap, cnt, C, sigma, Y) -> float:
    """f^(Y) = ||S + C + T/sigma||^2 - sum_a A(S + C)_a^2 / cnt_a, evaluated in the equivalent
    form (||x||^2 - ||P_A x||^2 = ||(I - P_A) x||^2, P_A = A*(AA*)^{-1}A orthogonal)
        f^ = ||S + C - A*(y(S))||^2 + (2/sigma) <T, S + C> + ||T||^2 / sigma^2
    whose first term is summed from its (small) entries instead of as the difference of two
    O(n^2) sums (reading R29: needed for the trust-region ratio near convergence)."""
    m = cnt.size
    S = Y @ Y.T
    SC = S if C is None else S + C
    yS = ops.A(amap, SC, m) / cnt
    R = SC - ops.At(amap, yS)
    return float(np.sum(R * R) + (2.0 / sigma) * np.sum(T * SC) + np.sum(T * T) / sigma ** 2)


def alm_eval(T, amap, cnt, C, sigma, Y, U=None) -> dict:
    """Cost, gradients and HVP of the y-eliminated subproblem (f^ scale).

    E = 4 (S - M(S)) Y
    H = P_Y(4 [Z Y + (S - M(S)) U - A*(A(Z)/cnt) Y]) - rowdot(E, Y) o U
        which is (2/sigma) x Eq. 4.7 with grad Phi evaluated at y(S).
    """
    m = cnt.size
    S = Y @ Y.T
    M, yS = alm_M(T, amap, cnt, C, sigma, S)
    W = S - M
    out = {"f": alm_cost(T, amap, cnt, C, sigma, Y), "y": yS, "M": M}
    E = 4.0 * (W @ Y)
    rho = rowdot(E, Y)
    out["E"] = E
    out["rho"] = rho
    out["R"] = E - rho[:, None] * Y
    if U is not None:
        Z = Y @ U.T + U @ Y.T
        w = ops.A(amap, Z, m) / cnt
        EH = 4.0 * (Z @ Y + W @ U - ops.At(amap, w) @ Y)
        out["H"] = project(Y, EH) - rho[:, None] * U
    return out


# ----------------------------------------------------------------------------------
# Paper-scale literal forms (for pinning the f-scale forms above)
# ----------------------------------------------------------------------------------
def L_sigma(S, y, Xt, D, C, amap, sigma) -> float:
    """Augmented Lagrangian of (DSDP'), P:101:
    L = <D, S + C> - <X~, A*(y) - S - C> + sigma/2 ||A*(y) - S - C||^2."""
    SC = S if C is None else S + C
    R = ops.At(amap, y) - SC
    return float(np.sum(D * SC) - np.sum(Xt * R) + 0.5 * sigma * np.sum(R * R))


def grad_Phi(S, y, Xt, D, C, amap, sigma):
    """nabla Phi_k(S) = X~ - sigma (A*(y) - S - C) + D (Lemma 3.2)."""
    SC = S if C is None else S + C
    return Xt - sigma * (ops.At(amap, y) - SC) + D


def paper_grad(G, Y):
    """Eq. 4.6: grad Psi = 2 X Y, X = nabla Phi - Diag(nabla Phi S)."""
    S = Y @ Y.T
    X = G - np.diag(np.diag(G @ S))
    return 2.0 * X @ Y


def paper_hess(G, Y, U, amap, cnt, sigma, projection_term=True):
    """Eq. 4.7 literally:
    H~ = 2 nabla Phi U + 2 sigma (Z - A*((AA*)^{-1} A(Z))) Y,
    Hess = H~ - Diag(H~ Y^T) Y - 2 Diag(nabla Phi S) U."""
    m = cnt.size
    S = Y @ Y.T
    Z = Y @ U.T + U @ Y.T
    P = Z - ops.At(amap, ops.A(amap, Z, m) / cnt) if projection_term else Z
    Ht = 2.0 * G @ U + 2.0 * sigma * P @ Y
    return Ht - np.diag(Ht @ Y.T)[:, None] * Y - 2.0 * np.diag(G @ S)[:, None] * U


# ----------------------------------------------------------------------------------
# Callable subproblems for the RTR driver (cache S, W, rho between cost and HVP)
# ----------------------------------------------------------------------------------
class FixedMProblem:
    """f(Y) = ||YY^T - M||^2 (fixed-M reading)."""

    def __init__(self, M):
        self.M = M
        self.n_costgrad = 0
        self.n_hvp = 0

    def costgrad(self, Y):
        self.n_costgrad += 1
        S = Y @ Y.T
        W = S - self.M
        E = 4.0 * (W @ Y)
        rho = rowdot(E, Y)
        ctx = {"Y": Y, "W": W, "rho": rho}
        return float(np.sum(W ** 2)), E - rho[:, None] * Y, ctx

    def hess(self, ctx, U):
        self.n_hvp += 1
        Y, W, rho = ctx["Y"], ctx["W"], ctx["rho"]
        Z = Y @ U.T + U @ Y.T
        EH = 4.0 * (Z @ Y + W @ U)
        return project(Y, EH) - rho[:, None] * U


class ALMProblem:
    """f^(Y) = ||S + C + T/sigma||^2 - sum_a A(S+C)_a^2/cnt_a (ALM reading)."""

    def __init__(self, T, amap, cnt, C, sigma):
        self.T, self.amap, self.cnt, self.C, self.sigma = T, amap, cnt, C, sigma
        self.m = cnt.size
        self.n_costgrad = 0
        self.n_hvp = 0

    def costgrad(self, Y):
        self.n_costgrad += 1
        S = Y @ Y.T
        SC = S if self.C is None else S + self.C
        a = ops.A(self.amap, SC, self.m)
        Rs = SC - ops.At(self.amap, a / self.cnt)  # (I - P_A)(S + C), see alm_cost
        f = float(np.sum(Rs * Rs) + (2.0 / self.sigma) * np.sum(self.T * SC) + np.sum(self.T * self.T) / self.sigma ** 2)
        M = ops.At(self.amap, a / self.cnt) - self.T / self.sigma
        if self.C is not None:
            M = M - self.C
        W = S - M
        E = 4.0 * (W @ Y)
        rho = rowdot(E, Y)
        ctx = {"Y": Y, "W": W, "rho": rho}
        return f, E - rho[:, None] * Y, ctx

    def hess(self, ctx, U):
        self.n_hvp += 1
        Y, W, rho = ctx["Y"], ctx["W"], ctx["rho"]
        Z = Y @ U.T + U @ Y.T
        w = ops.A(self.amap, Z, self.m) / self.cnt
        EH = 4.0 * (Z @ Y + W @ U - ops.At(self.amap, w) @ Y)
        return project(Y, EH) - rho[:, None] * U


def fixed_rows(M_rows: np.ndarray, rows: np.ndarray, Y: np.ndarray, U: np.ndarray | None = None) -> dict:
    """Rows `rows` of E, R (and H) of the fixed-M subproblem, for sampled checks at sizes where the
    full n x n products do not fit the oracle's budget. M_rows = M[rows, :]. Same definitions as
    fixed_eval restricted to those rows:
        E_j = 4 sum_i (S_ji - M_ji) y_i,     S_ji = <y_j, y_i>
        H_j = P_{y_j}(4 [ (Z Y)_j + ((S - M) U)_j ]) - rowdot(E, Y)_j u_j."""
    S_rows = Y[rows] @ Y.T
    W = S_rows - M_rows
    E = 4.0 * (W @ Y)
    rho = rowdot(E, Y[rows])
    out = {"E": E, "rho": rho, "R": E - rho[:, None] * Y[rows]}
    if U is not None:
        Z_rows = Y[rows] @ U.T + U[rows] @ Y.T
        EH = 4.0 * (Z_rows @ Y + W @ U)
        yr = Y[rows]
        out["H"] = EH - rowdot(EH, yr)[:, None] * yr - rho[:, None] * U[rows]
    return out


def fixed_cost_blocked(M_block_fn, Y: np.ndarray, block: int = 1024) -> float:
    """f = ||YY^T - M||^2 accumulated over row blocks; M_block_fn(i0, i1) returns M[i0:i1, :]."""
    n = Y.shape[0]
    f = 0.0
    for i0 in range(0, n, block):
        i1 = min(n, i0 + block)
        W = Y[i0:i1] @ Y.T - M_block_fn(i0, i1)
        f += float(np.sum(W * W))
    return f
