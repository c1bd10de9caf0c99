"""Seeded synthetic input generators shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no operators, no relaxation, no
subproblem formulas): it only draws the random data that both sides receive
(SURVEY.md §8(d) D-IN).

* ``bqp_instance(d, seed, kind)`` — the BQP data (Q, c) of BASELINE.json configs
  0-3: Q_ij ~ U[-1,1] i.i.d. for i<j mirrored, zero diagonal, c ~ U[-1,1]^d;
  ``kind="er05"`` masks Q with an Erdos-Renyi graph, edge probability 0.05.
  (The paper draws N(0,1) data with unpublished seeds; BASELINE.json
  fixes U[-1,1], which governs.)
* ``sweep_inputs(n, p)`` — the subproblem-kernel sweep of config 4: M symmetric
  with entries N(0,1)/sqrt(n), Y with unit rows, U a random tangent direction.
* ``chain_bqp_instance(q, t, seed)`` — the sparse (clique-chain) BQP of PAPER.md:555-579
  (SURVEY §8(f) row f2): t cliques of q variables, Q_k symmetric with [Q_k]_ij ~ N(0,1)
  (i <= j, mirrored), c_k ~ N(0,1)^q, as the paper draws them (no BASELINE config).
* ``initial_factor(n, p, seed)`` — the random starting point Y^0 the method
  draws (PAPER.md:321 writes Y^0 = 0, not a manifold point; reading R1),
  passed as an input to both the oracle and the GPU solver.
"""
from __future__ import annotations

import numpy as np

SEED = 20251204


def bqp_instance(d: int, seed: int = 0, kind: str = "dense"):
    """Return (Q, c): Q symmetric d x d with zero diagonal, c length d (float64)."""
    if d < 1:
        raise ValueError("d must be >= 1")
    if kind not in ("dense", "er05"):
        raise ValueError(f"unknown kind {kind!r}")
    rng = np.random.default_rng([SEED, d, seed])
    iu = np.triu_indices(d, 1)
    q = rng.uniform(-1.0, 1.0, iu[0].size)
    if kind == "er05":
        q = q * (rng.random(iu[0].size) < 0.05)
    Q = np.zeros((d, d))
    Q[iu] = q
    Q = Q + Q.T
    c = rng.uniform(-1.0, 1.0, d)
    return Q, c


def chain_bqp_instance(q: int, t: int, seed: int = 0):
    """Return (Qs [t, q, q], cs [t, q]) for the clique-chain BQP."""
    if q < 2 or t < 1:
        raise ValueError("need q >= 2, t >= 1")
    rng = np.random.default_rng([SEED, 23, q, t, seed])
    iu = np.triu_indices(q)
    Qs = np.zeros((t, q, q))
    for k in range(t):
        A = np.zeros((q, q))
        A[iu] = rng.standard_normal(iu[0].size)
        Qs[k] = A + np.triu(A, 1).T
    cs = rng.standard_normal((t, q))
    return Qs, cs


def _unit_rows(A: np.ndarray) -> np.ndarray:
    return A / np.linalg.norm(A, axis=1, keepdims=True)


def sweep_factor(n: int, p: int):
    """Y (unit rows) and a tangent direction U for the sweep, row-major (n, p)."""
    rng = np.random.default_rng([SEED, n, p])
    Y = _unit_rows(rng.standard_normal((n, p)))
    U = rng.standard_normal((n, p))
    U -= np.sum(U * Y, axis=1, keepdims=True) * Y
    return Y, U


def sweep_matrix_cpu(n: int) -> np.ndarray:
    """Dense symmetric M with M_ij = M_ji = A_ij / sqrt(n) (i <= j), A ~ N(0,1), numpy."""
    rng = np.random.default_rng([SEED, n])
    A = rng.standard_normal((n, n))
    M = np.triu(A)
    M += np.triu(A, 1).T
    M /= np.sqrt(n)
    return M


def sweep_matrix_torch(n: int, device="cuda", ld: int | None = None):
    """Same distribution generated on the device with torch's seeded generator.

    Used for the large sweep sizes (n = 16384, 32768: 2.1 / 8.6 GB) where a host
    draw plus a host->device copy would dominate the run. Returns a (n, ld) torch
    tensor whose first n columns hold M (padding columns are zero).
    """
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(SEED * 1000003 + n)
    ld = n if ld is None else ld
    out = torch.zeros((n, ld), dtype=torch.float64, device=device)
    bs = 2048
    # build the symmetric matrix in row blocks of the upper triangle, then mirror
    A = torch.randn((n, n), generator=g, dtype=torch.float64, device=device)
    A.triu_()
    A.div_(float(np.sqrt(n)))
    out[:, :n] = A
    for i0 in range(0, n, bs):
        i1 = min(n, i0 + bs)
        # lower part of rows i0:i1 = transposed strict upper part of columns i0:i1
        blk = A[:i1, i0:i1].T.clone()  # (i1-i0, i1)
        blk = torch.tril(blk, diagonal=i0 - 1)  # keep j < i strictly
        out[i0:i1, :i1] += blk
    del A
    return out


def sweep_inputs(n: int, p: int):
    """(M, Y, U) for the sweep at a size the host handles (numpy arrays)."""
    M = sweep_matrix_cpu(n)
    Y, U = sweep_factor(n, p)
    return M, Y, U


def initial_factor(n: int, p: int, seed: int = 0) -> np.ndarray:
    """Y^0: standard-normal rows normalised to unit length (n, p)."""
    rng = np.random.default_rng([SEED, 7, n, p, seed])
    return _unit_rows(rng.standard_normal((n, p)))


def random_unit_factor(n: int, p: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng([SEED, 11, n, p, seed])
    return _unit_rows(rng.standard_normal((n, p)))


def random_matrix(n: int, k: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng([SEED, 13, n, k, seed])
    return rng.standard_normal((n, k))


def random_symmetric(n: int, seed: int, scale: float = 1.0) -> np.ndarray:
    rng = np.random.default_rng([SEED, 17, n, seed])
    A = rng.standard_normal((n, n)) * scale
    return (A + A.T) / 2.0
