"""ORACLE — test infrastructure only.

A plain, slow, obviously correct CPU (NumPy float64, single-threaded BLAS)
implementation of what the ManiDSDP hot path computes, written from the paper
(PAPER.md = arXiv 2512.04406 LaTeX source; citations "P:n" are its line numbers).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything under ``oracle/``. The product path
(``paper_2512_04406_b200``) never imports it, and this package never imports the
product path: the two share no code. Shared *inputs* come from ``inputs/``.

Modules
  bqp         monomial basis, constraint index map, b, brute force
  operators   A, A*, AA*, D, y-update
  subproblem  fixed-M and y-eliminated (ALM) subproblem cost / gradient / HVP
                                                                       
  rtr         Riemannian trust region + truncated CG                 (Absil et al.)
  admm        Algorithm 2 (ManiDSDP): outer update, residues, escape, rank, sigma
                                                                       
Pinning status of every function: see DESIGN.md "Oracle pins". Parts whose parity
cannot be pinned (RTR trajectories, inner iteration counts) are marked
"parity unpinned" in their docstrings.
"""
import os as _os

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    _os.environ.setdefault(_v, "1")

try:  # pin BLAS to one thread even if numpy was imported first
    from threadpoolctl import threadpool_limits as _tpl

    _tpl(1)
except Exception:  # pragma: no cover
    pass
