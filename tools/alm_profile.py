"""Development aid: time the y-eliminated (ALM) evaluation the solver runs inside a d = 80 solve
(n = 3241) — cost+gradient and Hessian-vector product separately — with a synchronised wall clock over
many calls, to show where solve time goes. Synthetic state: T symmetric N(0, 1/n), unit-row
Y, tangent U (the parity tests check these calls against the oracle).

Usage: python tools/alm_profile.py [d | chain:q:t] [p,p,...] [reps]
  chain:q:t times the multi-block evaluation of the clique-chain relaxation (blocks.cu)
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from inputs import bqp_instance  # noqa: E402
from paper_2512_04406_b200 import abi  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "80"
ps = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [16, 64, 128, 240]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
ctx = abi.Context(0, 0)
rng = np.random.default_rng(0)
if arg.startswith("chain"):
    from inputs import chain_bqp_instance  # noqa: E402

    _, q, t = arg.split(":")
    ctx.set_bqp_chain(*chain_bqp_instance(int(q), int(t), 0))
    d = arg
    n = ctx.sizes()[0]
    nb = ctx.block_sizes()[1]
    ld = nb + (-nb) % 64
    Tp = np.zeros((n, ld))
    for k in range(int(t)):
        B = rng.standard_normal((nb, nb)) / np.sqrt(nb)
        Tp[k * nb:(k + 1) * nb, :nb] = (B + B.T) / 2
else:
    d = int(arg)
    Q, c = bqp_instance(d, 0)
    ctx.set_bqp(Q, c)
    n = ctx.sizes()[0]
    ld = n + (-n) % 64
    T = rng.standard_normal((n, n)) / np.sqrt(n)
    T = (T + T.T) / 2
    Tp = np.zeros((n, ld))
    Tp[:, :n] = T
Td = torch.from_numpy(Tp).cuda()
for p in ps:
    Y = rng.standard_normal((n, p))
    Y /= np.linalg.norm(Y, axis=1, keepdims=True)
    U = rng.standard_normal((n, p))
    U -= np.sum(U * Y, axis=1, keepdims=True) * Y
    Yd, Ud = torch.from_numpy(Y).cuda(), torch.from_numpy(U).cuda()
    cost = torch.zeros(1, dtype=torch.float64, device="cuda")
    E, R, H = torch.empty_like(Yd), torch.empty_like(Yd), torch.empty_like(Yd)
    res = {}
    for name, flags, args in (("costgrad", abi.EVAL_COSTGRAD, (None, cost, E, R, None)),
                              ("hvp", abi.EVAL_HVP, (Ud, None, None, None, H))):
        for _ in range(3):
            ctx.alm_eval(flags, p, Td, ld, 2.0, Yd, *args)
        ctx.sync()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            ctx.alm_eval(flags, p, Td, ld, 2.0, Yd, *args)
        ctx.sync()
        res[name] = (time.perf_counter() - t0) / reps * 1e3
    # one n x n x p product = 2 n^2 p flops; the HVP does the M.U product and the projection-term
    # product (2 n^2 p each on the TMA path) plus the dense Gram tiles (2 n^2 (2p) / 2)
    print(f"d={d} n={n} p={p}: costgrad {res['costgrad']:.3f} ms, hvp {res['hvp']:.3f} ms "
          f"(2n^2p = {2 * n * n * p / 1e9:.2f} GF -> {2 * n * n * p / res['hvp'] / 1e9:.1f} TF/s per product-equivalent)",
          flush=True)
