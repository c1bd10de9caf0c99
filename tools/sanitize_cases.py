"""Small cases for compute-sanitizer (racecheck / synccheck / memcheck; one tool per gpurun call):
every kernel family of libdrsdp.so at tiny sizes — fixed-M evaluations on the TMA ring
(n = 1000, p = 16), the upper-triangle path (n = 4100, p = 8), the column-chunked generic path
(p = 100), ALM evaluations (dense Gram tiles, pair product), the operator kernels, block Lanczos,
and a d = 10 solve with and without the captured tCG graph.

Usage: compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import bqp_instance, initial_factor, random_symmetric, sweep_factor  # noqa: E402
from paper_2512_04406_b200 import abi  # noqa: E402


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


ctx = abi.Context(0, 0)
for n, p in ((1000, 16), (4100, 8), (300, 100)):
    M = dev(random_symmetric(n, 1, 1.0 / np.sqrt(n)))
    Y, U = sweep_factor(n, p)
    Yd, Ud = dev(Y), dev(U)
    cost = torch.zeros(1, dtype=torch.float64, device="cuda")
    R, H = torch.empty_like(Yd), torch.empty_like(Yd)
    ctx.set_subproblem_matrix(n, M, n)
    ctx.subproblem_eval(abi.EVAL_COSTGRAD | abi.EVAL_HVP, p, Yd, Ud, cost, None, R, H)
    ctx.sync()
    print("fixed", n, p, cost.item(), flush=True)
Q, c = bqp_instance(20, 0)
ctx.set_bqp(Q, c)
n = ctx.sizes()[0]
ld = n + (-n) % 64
T = np.zeros((n, ld))
T[:, :n] = random_symmetric(n, 2, 0.1)
Td = dev(T)
for p in (16, 80):
    Y, U = sweep_factor(n, p)
    Yd, Ud = dev(Y), dev(U)
    cost = torch.zeros(1, dtype=torch.float64, device="cuda")
    R, H = torch.empty_like(Yd), torch.empty_like(Yd)
    ctx.alm_eval(abi.EVAL_COSTGRAD | abi.EVAL_HVP, p, Td, ld, 2.0, Yd, Ud, cost, None, R, H)
    ctx.sync()
    print("alm", n, p, cost.item(), flush=True)
z = dev(np.linspace(-0.1, 0.1, n))
V = torch.zeros((n, 8), dtype=torch.float64, device="cuda")
print("lanczos", ctx.x_eigs(Td, ld, z, 8, 8, V)[2], flush=True)
for graph in (False, True):
    if not graph:
        os.environ["DRSDP_NO_GRAPH"] = "1"
    else:
        os.environ.pop("DRSDP_NO_GRAPH", None)
    Q, c = bqp_instance(10, 0)
    ctx.set_bqp(Q, c)
    n = ctx.sizes()[0]
    ctx.set_params(ctx.default_params(p0=2, precond_mu=0.05 if graph else 0.0, eig_method=2 if graph else 1))
    ctx.set_initial_factor(initial_factor(n, 2, 0))
    info = ctx.solve()
    print("solve", graph, info["status"], info["dual_obj"], flush=True)
# multi-block (clique-chain) relaxation: block evaluations and a small solve (blocks.cu)
from inputs import chain_bqp_instance  # noqa: E402

Qs, cs = chain_bqp_instance(6, 3, 0)
ctx.set_bqp_chain(Qs, cs)
n = ctx.sizes()[0]
t, nb = ctx.block_sizes()
ld = nb + (-nb) % 64
Tb = np.zeros((n, ld))
Tb[:, :nb] = 0.1 * np.random.default_rng(3).standard_normal((n, nb))
for k in range(t):
    blk = Tb[k * nb:(k + 1) * nb, :nb]
    Tb[k * nb:(k + 1) * nb, :nb] = blk + blk.T
Td = dev(Tb)
for p in (3, 20):
    Y, U = sweep_factor(n, p)
    Yd, Ud = dev(Y), dev(U)
    cost = torch.zeros(1, dtype=torch.float64, device="cuda")
    R, H = torch.empty_like(Yd), torch.empty_like(Yd)
    ctx.alm_eval(abi.EVAL_COSTGRAD | abi.EVAL_HVP, p, Td, ld, 2.0, Yd, Ud, cost, None, R, H)
    ctx.sync()
    print("block alm", n, p, cost.item(), flush=True)
ctx.set_params(ctx.default_params(p0=2))
ctx.set_initial_factor(initial_factor(n, 2, 0))
info = ctx.solve()
print("block solve", info["status"], info["dual_obj"], flush=True)
ctx.close()
print("SANITIZE_CASES_DONE")
