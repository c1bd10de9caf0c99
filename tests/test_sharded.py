"""Row-sharded evaluation: the host-side decomposition and collectives with
gloo at world_size 2 on CPU (the per-block arithmetic by the oracle's row formulas, test side), and
on one GPU the library's row-block mode over two blocks against the oracle."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from inputs import random_symmetric, sweep_factor
from oracle import subproblem as sp
from paper_2512_04406_b200 import sharded


def test_row_blocks_partition():
    for n, w in ((1000, 2), (5051, 4), (300, 8), (7, 3)):
        b = sharded.row_blocks(n, w)
        assert b[0][0] == 0 and b[-1][1] == n and len(b) == w
        assert all(b[k][1] == b[k + 1][0] for k in range(w - 1))


def _worker(rank, world, port, n, p, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    M = random_symmetric(n, 5, 1.0 / np.sqrt(n))
    Y, U = sweep_factor(n, p)
    blocks = sharded.row_blocks(n, world)
    r0, r1 = blocks[rank]
    rows = np.arange(r0, r1)

    def local_cost_grad():
        o = sp.fixed_rows(M[rows], rows, Y)
        P = M[rows] @ Y
        share = -2.0 * np.sum(P * Y[rows]) + np.sum(M[rows] ** 2)
        if r0 == 0:
            G = Y.T @ Y
            share += np.sum(G * G)
        return torch.tensor([share], dtype=torch.float64), torch.from_numpy(o["R"])

    def local_hvp():
        o = sp.fixed_rows(M[rows], rows, Y, U)
        return torch.tensor([np.sum(U[rows] * o["H"])]), torch.from_numpy(o["H"])

    f, R = sharded.sharded_eval(torch, dist, local_cost_grad, n, blocks, rank)
    uh, H = sharded.sharded_eval(torch, dist, local_hvp, n, blocks, rank)
    if rank == 0:
        out_q.put((float(f[0]), R.numpy(), float(uh[0]), H.numpy()))
    dist.destroy_process_group()


def test_gloo_world2_matches_single_rank():
    n, p, world = 300, 8, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    f, R, uh, H = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    M = random_symmetric(n, 5, 1.0 / np.sqrt(n))
    Y, U = sweep_factor(n, p)
    ref = sp.fixed_eval(M, Y, U)
    assert abs(f - ref["f"]) <= 1e-12 * ref["f"]
    np.testing.assert_allclose(R, ref["R"], atol=1e-12 * np.abs(ref["E"]).max())
    np.testing.assert_allclose(H, ref["H"], atol=1e-12 * np.abs(ref["H"]).max())
    assert abs(uh - sp.inner(U, ref["H"])) <= 1e-12 * abs(uh)


@pytest.mark.gpu
@pytest.mark.parametrize("n,p,world", [(1000, 16, 2), (4100, 8, 3), (2500, 64, 4)])
def test_gpu_row_blocks_match_oracle(n, p, world):
    """The library's row-block mode (one block per would-be rank, run in turn on one GPU) summed /
    concatenated as sharded_eval does equals the oracle's full evaluation (<= 1e-10 relative)."""
    from paper_2512_04406_b200 import abi

    ctx = abi.Context(0, 0)
    M = random_symmetric(n, 6, 1.0 / np.sqrt(n))
    Y, U = sweep_factor(n, p)
    ld = n + (-n) % 32
    Yd = torch.tensor(Y, device="cuda")
    Ud = torch.tensor(U, device="cuda")
    cost_sum = 0.0
    Rs, Hs = [], []
    for r0, r1 in sharded.row_blocks(n, world):
        Mb = torch.zeros((r1 - r0, ld), dtype=torch.float64, device="cuda")
        Mb[:, :n] = torch.tensor(M[r0:r1])
        ctx.set_subproblem_rows(n, r0, r1, Mb, ld)
        cost = torch.zeros(1, dtype=torch.float64, device="cuda")
        R = torch.empty((r1 - r0, p), dtype=torch.float64, device="cuda")
        H = torch.empty_like(R)
        ctx.subproblem_eval(abi.EVAL_COSTGRAD | abi.EVAL_HVP, p, Yd, Ud, cost, None, R, H)
        ctx.sync()
        cost_sum += cost.item()
        Rs.append(R.cpu().numpy())
        Hs.append(H.cpu().numpy())
    ref = sp.fixed_eval(M, Y, U)
    G = Y.T @ Y
    scale = np.linalg.norm(4 * M @ Y) + np.linalg.norm(4 * Y @ G)
    assert abs(cost_sum - ref["f"]) <= 1e-10 * (np.sum(G * G) + np.sum(M * M))
    assert np.linalg.norm(np.vstack(Rs) - ref["R"]) <= 1e-10 * scale
    assert np.linalg.norm(np.vstack(Hs) - ref["H"]) <= 1e-10 * (scale + np.linalg.norm(4 * (Y @ U.T + U @ Y.T) @ Y))
    ctx.close()
