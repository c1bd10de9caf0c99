"""Multi-block (clique-chain) sparse BQP relaxation and its ManiDSDP solve (oracle).

ORACLE — test infrastructure only (see oracle/__init__.py). SURVEY.md §8(f) row f2.

PAPER.md:555-602 (§6.2, Eq. BQP-sparse, the sparse SOS relaxation and DSDP-sparse) and the
remark P:434-436 (Algorithm 2 extends to multi-block SDPs):

* cliques x_k = {x_{(q-2)(k-1)+1}, .., x_{(q-2)k+2}}, k = 1..t, d = (q-2)t + 2 variables,
  consecutive cliques share two variables;
* objective sum_k x_k^T Q_k x_k + c_k^T x_k;
* one moment block per clique with basis v(x_k) = [1, x_k, products of two clique variables]
  (graded-lex, P:466 applied per clique), n_b = 1 + q + q(q-1)/2 rows;
* one constraint (one entry of y) per square-free monomial of degree <= 4 that appears in some
  block, SHARED by all blocks in which it appears (the moment y_alpha is one number; P:593-602
  "multi-block version of (DSDP) with C = 0");
* S = A*(y) in S^+_{n_b} x .. x S^+_{n_b}, diag S = 1.

Block storage: block k owns rows k*n_b .. (k+1)*n_b - 1 of the factor Y (N = t*n_b rows, the
oblique manifold of all rows) and the n_b x n_b matrices amaps[k], T[k]; S_k = Y_k Y_k^T. Only
the diagonal blocks exist: a cross-block product y_i^T y_j is never part of the problem.

Everything below is Algorithm 2 (oracle/admm.py) with every n x n object replaced by its list
of diagonal blocks; the block-diagonal X has the union of the blocks' spectra, so eta_d and the
escape directions come from the per-block eigendecompositions (readings R37-R39 of DESIGN.md).
Monomial order of the shared constraints: graded-lex of sorted global index tuples (R18).
Uniform block size only (the paper's workload has one q for all cliques).
"""
from __future__ import annotations

import itertools
import math
import time

import numpy as np

from .admm import Params, eta_d_of, rank_reduce, sigma_update
from .rtr import RTRParams, rtr
from .subproblem import project, rowdot


# ------------------------------------------------------------------------------------------------
# relaxation data
# ------------------------------------------------------------------------------------------------
def chain_cliques(q: int, t: int):
    """0-based variable index tuples of the t cliques."""
    if q < 2 or t < 1:
        raise ValueError("need q >= 2, t >= 1")
    return [tuple(range((q - 2) * k, (q - 2) * k + q)) for k in range(t)]


def block_basis(clique):
    """v(x_k) as sorted global index tuples, graded-lex (P:466 per clique)."""
    return [()] + [(i,) for i in clique] + list(itertools.combinations(clique, 2))


def chain_monomials(q: int, t: int):
    """Union over cliques of the square-free monomials of degree <= 4 in the clique's variables,
    graded-lex over sorted global index tuples (reading R18)."""
    mons = set()
    for cl in chain_cliques(q, t):
        for k in range(5):
            mons.update(itertools.combinations(cl, k))
    return sorted(mons, key=lambda a: (len(a), a))


def relax_chain(Qs: np.ndarray, cs: np.ndarray):
    """(amaps [t, n_b, n_b] int32, cnt [m], b [m], monomials) of the sparse relaxation.

    amaps[k][i, j] = id of v_i(x_k) v_j(x_k) reduced mod (x^2 - 1) (symmetric difference);
    cnt_a = number of ordered positions, over all blocks, whose id is a (= (AA*)_aa);
    b_a = coefficient of monomial a in sum_k x_k^T Q_k x_k + c_k^T x_k reduced mod the ideal:
    b_{1} = sum_k tr Q_k, b_{x_i} = sum_{k: i in x_k} c_k,i, b_{x_i x_j} = sum_k 2 Q_k,ij."""
    t, q = Qs.shape[0], Qs.shape[1]
    cliques = chain_cliques(q, t)
    mons = chain_monomials(q, t)
    ids = {a: k for k, a in enumerate(mons)}
    nb = 1 + q + q * (q - 1) // 2
    amaps = np.empty((t, nb, nb), dtype=np.int32)
    for k, cl in enumerate(cliques):
        sets = [frozenset(a) for a in block_basis(cl)]
        for i in range(nb):
            for j in range(nb):
                amaps[k, i, j] = ids[tuple(sorted(sets[i] ^ sets[j]))]
    m = len(mons)
    cnt = np.bincount(amaps.ravel(), minlength=m).astype(np.int64)
    b = np.zeros(m)
    for k, cl in enumerate(cliques):
        b[ids[()]] += np.trace(Qs[k])
        for li, i in enumerate(cl):
            b[ids[(i,)]] += cs[k, li]
        for li, lj in itertools.combinations(range(q), 2):
            b[ids[(cl[li], cl[lj])]] += 2.0 * Qs[k, li, lj]
    return amaps, cnt, b, mons


def chain_value(Qs, cs, x) -> float:
    """sum_k x_k^T Q_k x_k + c_k^T x_k."""
    t, q = Qs.shape[0], Qs.shape[1]
    v = 0.0
    for k, cl in enumerate(chain_cliques(q, t)):
        xk = x[list(cl)]
        v += float(xk @ Qs[k] @ xk + cs[k] @ xk)
    return v


def chain_moment_vector(x, mons) -> np.ndarray:
    """mu(x)_a = prod_{i in a} x_i over the relaxation's monomials."""
    return np.array([np.prod(x[list(a)]) if a else 1.0 for a in mons])


def chain_block_factor(x, q: int, t: int) -> np.ndarray:
    """Rank-one factor of the moment blocks of a point x in {-1,1}^d: rows v(x_k)_i (N x 1)."""
    rows = []
    for cl in chain_cliques(q, t):
        rows += [np.prod(x[list(a)]) if a else 1.0 for a in block_basis(cl)]
    return np.array(rows)[:, None]


def chain_brute_force(Qs, cs):
    """min over x in {-1,1}^d of the chain objective by enumeration (d <= 22)."""
    t, q = Qs.shape[0], Qs.shape[1]
    d = (q - 2) * t + 2
    if d > 22:
        raise ValueError("brute force limited to d <= 22")
    best, arg = np.inf, None
    for bits in range(1 << d):
        x = np.array([1.0 if (bits >> k) & 1 else -1.0 for k in range(d)])
        v = chain_value(Qs, cs, x)
        if v < best:
            best, arg = v, x
    return best, arg


# ------------------------------------------------------------------------------------------------
# block operators (P:58 per block; the shared y couples the blocks)
# ------------------------------------------------------------------------------------------------
def A_blocks(amaps, Xb, m) -> np.ndarray:
    """A(X)_a = sum_k sum_{(i,j): amaps[k]_ij = a} X_k,ij."""
    return np.bincount(amaps.ravel(), weights=Xb.ravel(), minlength=m)


def At_blocks(amaps, y) -> np.ndarray:
    """A*(y)_k,ij = y[amaps[k]_ij]."""
    return y[amaps]


def block_gram(Y, V, t) -> np.ndarray:
    """[Y_k V_k^T]_k, Y_k = rows of block k."""
    nb = Y.shape[0] // t
    return np.stack([Y[k * nb:(k + 1) * nb] @ V[k * nb:(k + 1) * nb].T for k in range(t)])


def block_apply(Mb, Y) -> np.ndarray:
    """Rows of blockdiag(M_k) Y."""
    t, nb = Mb.shape[0], Mb.shape[1]
    return np.vstack([Mb[k] @ Y[k * nb:(k + 1) * nb] for k in range(t)])


class BlockALMProblem:
    """y-eliminated subproblem (reading R2) over the product of blocks:
    f^(Y) = sum_k ||S_k + C_k + T_k/sigma||^2 - sum_a A(S + C)_a^2 / cnt_a, evaluated (reading
    R29) as ||S + C - A*(y(S))||^2 + (2/sigma) <T, S + C> + ||T||^2/sigma^2, all sums over blocks.
    E = 4 blockdiag(S_k - M_k(S)) Y,  H = P_Y(4 [Z Y + (S - M(S)) U - A*(A(Z)/cnt) Y]) - rho o U
    with Z_k = Y_k U_k^T + U_k Y_k^T (the dense formulas of oracle/subproblem.py, block by block)."""

    def __init__(self, T, amaps, cnt, sigma):
        self.T, self.amaps, self.cnt, self.sigma = T, amaps, cnt, sigma
        self.t = amaps.shape[0]
        self.m = cnt.size
        self.n_costgrad = 0
        self.n_hvp = 0

    def costgrad(self, Y):
        self.n_costgrad += 1
        S = block_gram(Y, Y, self.t)
        yS = A_blocks(self.amaps, S, self.m) / self.cnt
        Rs = S - At_blocks(self.amaps, yS)
        f = float(np.sum(Rs * Rs) + (2.0 / self.sigma) * np.sum(self.T * S)
                  + np.sum(self.T * self.T) / self.sigma ** 2)
        M = At_blocks(self.amaps, yS) - self.T / self.sigma
        W = S - M
        E = 4.0 * block_apply(W, Y)
        rho = rowdot(E, Y)
        return f, E - rho[:, None] * Y, {"Y": Y, "W": W, "rho": rho, "y": yS}

    def hess(self, ctx, U):
        self.n_hvp += 1
        Y, W, rho = ctx["Y"], ctx["W"], ctx["rho"]
        Z = block_gram(Y, U, self.t)
        Z = Z + np.transpose(Z, (0, 2, 1))
        w = A_blocks(self.amaps, Z, self.m) / self.cnt
        EH = 4.0 * (block_apply(Z, Y) + block_apply(W, U) - block_apply(At_blocks(self.amaps, w), Y))
        return project(Y, EH) - rho[:, None] * U


def block_alm_eval(T, amaps, cnt, sigma, Y, U=None) -> dict:
    """f^, E, rho, R (and H along U) of BlockALMProblem as arrays (parity helper)."""
    prob = BlockALMProblem(T, amaps, cnt, sigma)
    f, R, ctx = prob.costgrad(Y)
    rho = ctx["rho"]
    out = {"f": f, "R": R, "rho": rho, "E": R + rho[:, None] * Y, "y": ctx["y"]}
    if U is not None:
        out["H"] = prob.hess(ctx, U)
    return out


# ------------------------------------------------------------------------------------------------
# Algorithm 2 over blocks
# ------------------------------------------------------------------------------------------------
def block_residues(amaps, cnt, b, y, Y, T):
    """eta_p, eta_d, eta_g (readings R6-R8) of (y, S = blockdiag(Y_k Y_k^T),
    X = blockdiag(T_k - Diag z_k)); the spectrum of X is the union of the blocks' spectra
    (reading R38). Returns per-block eigenpairs for the escape step."""
    t, nb = amaps.shape[0], amaps.shape[1]
    S = block_gram(Y, Y, t)
    R = At_blocks(amaps, y) - S
    z = rowdot(block_apply(T, Y), Y)
    lams, Vs = [], []
    for k in range(t):
        Xk = T[k] - np.diag(z[k * nb:(k + 1) * nb])
        lam, V = np.linalg.eigh(Xk)
        lams.append(lam)
        Vs.append(V)
    lam_min = min(float(l[0]) for l in lams)
    lam_max = max(float(l[-1]) for l in lams)
    eta_p = float(np.linalg.norm(R))
    eta_d = eta_d_of(lam_min, lam_max)
    dobj = float(b @ y)
    pobj = float(np.sum(z))
    eta_g = abs(dobj - pobj) / (1.0 + abs(dobj) + abs(pobj))
    return {"eta_p": eta_p, "eta_d": eta_d, "eta_g": eta_g, "eta_max": max(eta_p, eta_d, eta_g),
            "dual_obj": dobj, "primal_obj": pobj, "z": z, "lams": lams, "Vs": Vs,
            "lam_min": lam_min, "lam_max": lam_max}


def block_escape_directions(lams, Vs, eig_neg_tol, escape_max):
    """Escape directions of the block-diagonal X (Thm 4.5, on the product of the blocks'
    manifolds; reading R39): in every block, the eigenpairs with lambda < -eig_neg_tol (1 + |lambda_max|)
    (lambda_max over all blocks), most negative first; column c of the result holds the c-th such
    eigenvector of EVERY block that has one, in that block's rows (zeros elsewhere) — the blocks do not
    interact, so one new column escapes in all blocks at once. delta = min(escape_max, max_k #neg_k)
    columns; each block's vector signed so that its largest-|.| entry is positive (R25). Returns an
    N x delta array or None. For t = 1 this is oracle/admm.escape_directions."""
    t, nb = len(lams), lams[0].size
    lam_max = max(float(l[-1]) for l in lams)
    thresh = -eig_neg_tol * (1.0 + abs(lam_max))
    negs = [int(np.sum(l < thresh)) for l in lams]  # eigh: ascending
    delta = min(escape_max, max(negs))
    if delta == 0:
        return None
    out = np.zeros((t * nb, delta))
    for k in range(t):
        for c in range(min(delta, negs[k])):
            v = Vs[k][:, c].copy()
            j = int(np.argmax(np.abs(v)))
            if v[j] < 0:
                v = -v
            out[k * nb:(k + 1) * nb, c] = v
    return out


def solve_blocks(amaps, cnt, b, prm: Params, Y0: np.ndarray, verbose=False):
    """Algorithm 2 on the multi-block problem, C = 0.
    Same control flow and readings as oracle/admm.solve; the tCG preconditioner (R35) is off
    for block problems (reading R37).
    Parity unpinned: the trajectory (see oracle/admm.py)."""
    t0 = time.perf_counter()
    t, nb = amaps.shape[0], amaps.shape[1]
    N = t * nb
    m = cnt.size
    if np.any(cnt <= 0):
        raise ValueError("Assumption 2 violated: constraint with no position")
    T = At_blocks(amaps, b / cnt)  # X~^0 = 0, T = D
    y = np.zeros(m)
    sigma = prm.sigma0
    Y = Y0.copy()
    U = None
    eta_prev = 1.0
    b_norm = float(np.linalg.norm(b))
    trace = []
    status = "not_converged"
    res = None
    totals = {"rtr": 0, "tcg": 0, "costgrad": 0, "hvp": 0, "p_max": Y.shape[1]}
    for k in range(prm.max_outer):
        p = Y.shape[1]
        prob = BlockALMProblem(T, amaps, cnt, sigma)
        eps_k = max(0.1 * min(1.0, eta_prev) * prm.eps_scale, prm.eps_floor)
        grad_tol = 4.0 * eps_k / sigma
        Y, info = rtr(prob, Y, RTRParams(N, p, max_iter=prm.max_rtr, rho_reg=prm.rho_reg,
                                        max_tcg=prm.max_tcg if prm.max_tcg > 0 else None,
                                        precond_mu=0.0), grad_tol, warm_U=U,
                      stall=prm.stall_rtr, stall_factor=prm.stall_factor)
        totals["rtr"] += info["iters"]
        totals["tcg"] += info["tcg"]
        totals["costgrad"] += prob.n_costgrad
        totals["hvp"] += prob.n_hvp
        grad_paper = 0.5 * sigma * info["gnorm"]
        S = block_gram(Y, Y, t)
        y = A_blocks(amaps, S, m) / cnt  # step 5
        Rp = At_blocks(amaps, y) - S
        T = T - sigma * Rp  # step 6
        res = block_residues(amaps, cnt, b, y, Y, T)
        row = {"iter": k + 1, **{c: res[c] for c in ("eta_p", "eta_d", "eta_g", "eta_max",
                                                       "primal_obj", "dual_obj")},
               "sigma": sigma, "p": p, "inner_iters": info["iters"], "cg_iters": info["tcg"]}
        if verbose:
            print(f"k={k+1:3d} p={p:3d} sigma={sigma:9.3e} eta_p={res['eta_p']:.2e} "
                  f"eta_d={res['eta_d']:.2e} eta_g={res['eta_g']:.2e} dobj={res['dual_obj']:.10f} "
                  f"rtr={info['iters']} tcg={info['tcg']}")
        if res["eta_max"] <= prm.tol:
            status = "converged"
            row["escape_delta"] = 0
            row["time_s"] = time.perf_counter() - t0
            trace.append(row)
            break
        Vs = block_escape_directions(res["lams"], res["Vs"], prm.eig_neg_tol, prm.escape_max)
        pcap = min(128, nb)  # reading R39: p <= min(128, n_b) for block problems
        if Vs is not None and Y.shape[1] + Vs.shape[1] > pcap:
            Vs = Vs[:, : pcap - Y.shape[1]] if Y.shape[1] < pcap else None
        gated = prm.escape_gate > 0 and info["gnorm"] > prm.escape_gate * grad_tol
        if gated:
            Vs = None
        if Vs is None and not gated:
            Y = rank_reduce(Y, min(prm.rank_tol, max(1e-8, 0.01 * math.sqrt(res["eta_max"]))))
        if Vs is not None:
            pr = Y.shape[1]
            Y = np.hstack([Y, np.zeros((N, Vs.shape[1]))])
            U = np.hstack([np.zeros((N, pr)), Vs])
        else:
            U = None
        row["escape_delta"] = 0 if Vs is None else Vs.shape[1]
        totals["p_max"] = max(totals["p_max"], Y.shape[1])
        sigma = sigma_update(sigma, res["eta_p"], b_norm, grad_paper, prm)
        eta_prev = res["eta_max"]
        row["time_s"] = time.perf_counter() - t0
        trace.append(row)
    return {"status": status, "y": y, "Y": Y, "T": T, "z": res["z"], "sigma": sigma,
            "dual_obj": res["dual_obj"], "primal_obj": res["primal_obj"], "eta_p": res["eta_p"],
            "eta_d": res["eta_d"], "eta_g": res["eta_g"], "eta_max": res["eta_max"],
            "outer_iters": len(trace), "trace": trace, "totals": totals,
            "time_s": time.perf_counter() - t0}
