"""Constraint operators of (DSDP) for an index-map operator (oracle).

PAPER.md:58 (§2): A(X) = (<A_a, X>)_a, A*(y) = sum_a y_a A_a. With A_a the 0/1
indicator of the positions whose index-map id is a, A(X)_a = sum of X over those
(ordered) positions and A*(y)_ij = y[amap_ij]. AA* = Diag(cnt) (each position has one
id), so (AA*)^{-1} is a division by cnt; Assumption 2 <=> every cnt_a >= 1.
"""
from __future__ import annotations

import numpy as np


def A(amap: np.ndarray, X: np.ndarray, m: int) -> np.ndarray:
    """A(X)_a = sum_{(i,j): amap_ij = a} X_ij."""
    return np.bincount(amap.ravel(), weights=X.ravel(), minlength=m)


def At(amap: np.ndarray, y: np.ndarray) -> np.ndarray:
    """A*(y)_ij = y[amap_ij]."""
    return y[amap]


def AAt(amap: np.ndarray, m: int) -> np.ndarray:
    """Diagonal of AA*: (AA*)_aa = <A_a, A_a> = cnt_a."""
    return np.bincount(amap.ravel(), minlength=m).astype(float)


def check_assumption2(cnt: np.ndarray) -> None:
    """Assumption 2: AA* invertible <=> no empty constraint."""
    if np.any(cnt <= 0):
        raise ValueError("Assumption 2 violated: constraint with no position")


def gram_solve(cnt: np.ndarray, v: np.ndarray) -> np.ndarray:
    """(AA*)^{-1} v."""
    return v / cnt


def D_matrix(amap: np.ndarray, cnt: np.ndarray, b: np.ndarray) -> np.ndarray:
    """D = A*((AA*)^{-1} b)."""
    return At(amap, gram_solve(cnt, b))


def y_update(amap, cnt, S, C):
    """y = (AA*)^{-1} A(S + C) (Lemma 3.1; Alg. 2 step 5)."""
    m = cnt.size
    SC = S if C is None else S + C
    return gram_solve(cnt, A(amap, SC, m))
