import sys, numpy as np, torch
sys.path.insert(0, '.')
from inputs import sweep_matrix_cpu, sweep_factor
from oracle import subproblem as sp
from paper_2512_04406_b200 import abi
ctx = abi.Context(0, 0)
for mode in ("E", "noE", "E_only_cg", "fresh"):
  for n in (4, 37, 200, 1000):
    p = 1
    if mode == "fresh":
        ctx = abi.Context(0, 0)
    M = sweep_matrix_cpu(n); Y, U = sweep_factor(n, p)
    Md = torch.tensor(M, device='cuda'); ctx.set_subproblem_matrix(n, Md, n)
    Yd = torch.tensor(Y, device='cuda'); Ud = torch.tensor(U, device='cuda')
    cost = torch.zeros(1, dtype=torch.float64, device='cuda'); R = torch.empty_like(Yd); E = torch.empty_like(Yd); H = torch.empty_like(Yd)
    if mode == "E" or mode == "fresh":
        ctx.subproblem_eval(3, p, Yd, Ud, cost, E, R, H)
    elif mode == "noE":
        ctx.subproblem_eval(3, p, Yd, Ud, cost, None, R, H)
    else:
        ctx.subproblem_eval(1, p, Yd, None, cost, E, R, None)
    torch.cuda.synchronize()
    o = sp.fixed_eval(M, Y, U)
    print(mode, n, p, cost.item(), o['f'], np.abs(R.cpu().numpy() - o['R']).max(), flush=True)
