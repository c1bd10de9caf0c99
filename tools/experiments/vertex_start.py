"""Diagnostic (not a product path): is the second-order relaxation of the d-variable BQP instance tight, and is
finding the optimal vertex the hard part of the solve?  A one-flip tabu search finds a good x in {-1,1}^d on
the host; the solve then starts from the rank-one factor Y0 = [v(x), 0] (v(x) = the monomial vector).
If the relaxation is tight at x, the primal iterate is optimal from the start and Algorithm 2 only has to
build the multiplier X~ (the phase the d = 80 trace shows after its third outer iteration).

Usage: python tools/experiments/vertex_start.py D time_limit_s [key=value ...]
"""
import itertools
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from inputs import bqp_instance  # noqa: E402
from paper_2512_04406_b200 import abi  # noqa: E402


def tabu(Q, c, reps=60, iters=4000, seed=1):
    d = len(c)
    rng = np.random.default_rng(seed)
    best, bx = np.inf, None
    for _ in range(reps):
        x = rng.choice([-1.0, 1.0], d)
        g = Q @ x
        fx = x @ Q @ x + c @ x
        until = np.zeros(d, int)
        lb, lx = fx, x.copy()
        for it in range(iters):
            delta = -4 * x * g - 2 * c * x
            cand = np.where((until <= it) | (fx + delta < lb - 1e-12), delta, np.inf)
            i = int(np.argmin(cand))
            fx += delta[i]
            g -= 2 * x[i] * Q[:, i]
            x[i] = -x[i]
            until[i] = it + 10 + rng.integers(0, 10)
            if fx < lb - 1e-12:
                lb, lx = fx, x.copy()
        if lb < best - 1e-9:
            best, bx = lb, lx.copy()
    return best, bx


d = int(sys.argv[1])
tl = float(sys.argv[2])
kw = {}
for a in sys.argv[3:]:
    k, v = a.split("=")
    kw[k] = float(v) if "." in v or "e" in v else int(v)
Q, c = bqp_instance(d, 0, "er05" if d == 150 else "dense")
Q = np.asarray(Q, float)
c = np.asarray(c, float)
fbest, x = tabu(Q, c)
print(json.dumps({"d": d, "tabu_best": fbest}), flush=True)
v = np.concatenate([[1.0], x, [x[i] * x[j] for i, j in itertools.combinations(range(d), 2)]])
Y0 = np.zeros((len(v), 2))
Y0[:, 0] = v
ctx = abi.Context(0, None)
ctx.set_bqp(Q, c)
ctx.set_params(ctx.default_params(p0=2, time_limit_s=tl, **kw))
ctx.set_initial_factor(Y0)
t0 = time.time()
info = ctx.solve()
for r in ctx.trace():
    print(" ".join(f"{k}={v:.3e}" if isinstance(v, float) and k.startswith("eta") else f"{k}={v:.6g}"
                   for k, v in r.items()), flush=True)
print(json.dumps({"d": d, "tabu_best": fbest, "solve_s": time.time() - t0, **info}), flush=True)
