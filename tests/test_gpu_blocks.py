"""GPU parity of the multi-block (clique-chain) relaxation, SURVEY §8(f) row f2 (PAPER.md:555-602,
remark P:434-436), through the C ABI, against oracle/sparse_bqp.py.

Bars as in test_gpu_parity.py: index map and segments bit-exact; evaluations <= 1e-10 relative to
the summand scale; solves eta_max <= 1e-8 (recomputed by the oracle from the returned tuple) and
the objective within 1e-6 relative of the oracle's."""
import json
import os

import numpy as np
import pytest

from inputs import chain_bqp_instance, initial_factor, random_matrix, random_unit_factor
from oracle import admm
from oracle import sparse_bqp as sb
from oracle import subproblem as sp

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-10
GOLD = os.path.join(os.path.dirname(__file__), "golden", "oracle_chain_solves.json")


@pytest.fixture(scope="module")
def ctx():
    from paper_2512_04406_b200 import abi, build

    build.build()
    c = abi.Context(0, 0)
    yield c
    c.close()


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def rel(a, b, scale):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / scale)


def _segments_from_oracle(amaps, m):
    """Independent CSR over upper positions with GLOBAL rows, sorted (id, row, col)."""
    t, nb = amaps.shape[0], amaps.shape[1]
    iu, ju = np.triu_indices(nb)
    ids, keys = [], []
    for k in range(t):
        ids.append(amaps[k][iu, ju].astype(np.int64))
        keys.append(((k * nb + iu).astype(np.uint64) << np.uint64(16)) | (k * nb + ju).astype(np.uint64))
    ids, keys = np.concatenate(ids), np.concatenate(keys)
    order = np.lexsort((keys, ids))
    ptr = np.zeros(m + 1, np.int64)
    np.add.at(ptr, ids + 1, 1)
    return np.cumsum(ptr), keys[order].astype(np.uint32)


@pytest.mark.parametrize("q,t", [(4, 1), (4, 3), (5, 4), (7, 2), (20, 3)])
def test_chain_index_map_bit_exact(ctx, q, t):
    Qs, cs = chain_bqp_instance(q, t, 0)
    amaps, cnt, b, _ = sb.relax_chain(Qs, cs)
    ctx.set_bqp_chain(Qs, cs)
    tt, nb = ctx.block_sizes()
    assert (tt, nb) == (t, amaps.shape[1])
    n, m, nu = ctx.sizes()
    assert n == t * nb and m == cnt.size and nu == t * nb * (nb + 1) // 2
    amap, seg_ptr, seg_pos = ctx.export_index_map()
    np.testing.assert_array_equal(amap, amaps.reshape(t * nb, nb))
    ptr_o, pos_o = _segments_from_oracle(amaps, m)
    np.testing.assert_array_equal(seg_ptr, ptr_o)
    np.testing.assert_array_equal(seg_pos, pos_o)


def test_set_blocks_general_equals_chain(ctx):
    """drsdp_set_blocks with the oracle's maps defines the same problem as drsdp_set_bqp_chain."""
    Qs, cs = chain_bqp_instance(5, 3, 4)
    amaps, cnt, b, _ = sb.relax_chain(Qs, cs)
    ctx.set_blocks(amaps, b)
    a1, p1, s1 = ctx.export_index_map()
    ctx.set_bqp_chain(Qs, cs)
    a2, p2, s2 = ctx.export_index_map()
    assert np.array_equal(a1, a2) and np.array_equal(p1, p2) and np.array_equal(s1, s2)


def _block_state(q, t, seed, p, sigma):
    Qs, cs = chain_bqp_instance(q, t, seed)
    amaps, cnt, b, _ = sb.relax_chain(Qs, cs)
    tt, nb, m = amaps.shape[0], amaps.shape[1], cnt.size
    rng = np.random.default_rng([seed, 31, p])
    Xt = rng.standard_normal((tt, nb, nb)) * 0.3
    Xt = Xt + np.transpose(Xt, (0, 2, 1))
    Xt = Xt - sb.At_blocks(amaps, sb.A_blocks(amaps, Xt, m) / cnt)
    T = Xt + sb.At_blocks(amaps, b / cnt)
    N = tt * nb
    Y = random_unit_factor(N, p, seed + 2)
    U = sp.project(Y, random_matrix(N, p, seed + 3))
    return Qs, cs, amaps, cnt, b, T, Y, U


def _stacked(T, ld):
    t, nb = T.shape[0], T.shape[1]
    out = np.zeros((t * nb, ld))
    out[:, :nb] = T.reshape(t * nb, nb)
    return out


@pytest.mark.parametrize("q,t,p", [(4, 3, 1), (5, 4, 3), (6, 3, 16), (8, 5, 17), (20, 3, 33), (20, 4, 64), (20, 3, 100), (20, 2, 128)])
def test_block_alm_eval_parity(ctx, q, t, p):
    from paper_2512_04406_b200 import abi

    sigma = 2.5
    Qs, cs, amaps, cnt, b, T, Y, U = _block_state(q, t, 3, p, sigma)
    ctx.set_bqp_chain(Qs, cs)
    nb = amaps.shape[1]
    ld = nb + (-nb) % 64
    Td, Yd, Ud = dev(_stacked(T, ld)), dev(Y), dev(U)
    cost = torch.zeros(1, dtype=torch.float64, device="cuda")
    E, R, H = torch.empty_like(Yd), torch.empty_like(Yd), torch.empty_like(Yd)
    ctx.alm_eval(abi.EVAL_COSTGRAD | abi.EVAL_HVP, p, Td, ld, sigma, Yd, Ud, cost, E, R, H)
    torch.cuda.synchronize()
    o = sb.block_alm_eval(T, amaps, cnt, sigma, Y, U)
    S = sb.block_gram(Y, Y, t)
    M = sb.At_blocks(amaps, o["y"]) - T / sigma
    sE = np.linalg.norm(4 * sb.block_apply(M, Y)) + np.linalg.norm(4 * sb.block_apply(S, Y))
    assert abs(cost.item() - o["f"]) <= TOL * (np.sum(S * S) + np.sum((T / sigma) ** 2) + np.sum(o["y"] ** 2 * cnt))
    assert rel(E.cpu().numpy(), o["E"], sE) <= TOL
    assert rel(R.cpu().numpy(), o["R"], sE) <= TOL
    Z = sb.block_gram(Y, U, t)
    Z = Z + np.transpose(Z, (0, 2, 1))
    w = sb.A_blocks(amaps, Z, cnt.size) / cnt
    sH = sE + np.linalg.norm(4 * sb.block_apply(sb.At_blocks(amaps, w), Y))
    assert rel(H.cpu().numpy(), o["H"], sH) <= TOL


@pytest.mark.parametrize("q,t,p", [(5, 3, 4), (20, 3, 12)])
def test_block_y_and_dual_update_parity(ctx, q, t, p):
    """y = A(S)/cnt over all blocks (Alg. 2 step 5), T <- T - sigma (A*(y) - S) per block (step 6),
    z = rowdot(T Y, Y) (step 7) and the scalars [||R||, b^T y, sum z, ||T||^2]."""
    sigma = 1.7
    Qs, cs, amaps, cnt, b, T, Y, U = _block_state(q, t, 5, p, sigma)
    ctx.set_bqp_chain(Qs, cs)
    tt, nb, m = amaps.shape[0], amaps.shape[1], cnt.size
    ld = nb + (-nb) % 64
    Yd = dev(Y)
    yd = torch.zeros(m, dtype=torch.float64, device="cuda")
    ctx.y_update(p, Yd, yd)
    S = sb.block_gram(Y, Y, tt)
    y_o = sb.A_blocks(amaps, S, m) / cnt
    torch.cuda.synchronize()
    assert np.abs(yd.cpu().numpy() - y_o).max() <= 1e-13
    Td = dev(_stacked(T, ld))
    zd = torch.zeros(tt * nb, dtype=torch.float64, device="cuda")
    sc = torch.zeros(4, dtype=torch.float64, device="cuda")
    ctx.dual_update(p, Yd, dev(y_o), sigma, Td, ld, zd, sc)
    torch.cuda.synchronize()
    R = sb.At_blocks(amaps, y_o) - S
    Tn = T - sigma * R
    z = sp.rowdot(sb.block_apply(Tn, Y), Y)
    np.testing.assert_allclose(Td.cpu().numpy()[:, :nb], Tn.reshape(tt * nb, nb), rtol=0, atol=1e-12)
    np.testing.assert_allclose(zd.cpu().numpy(), z, rtol=0, atol=1e-11 * (1 + np.abs(z).max()))
    s = sc.cpu().numpy()
    assert abs(s[0] - np.linalg.norm(R)) <= 1e-11 * (1 + np.linalg.norm(R))
    assert abs(s[1] - b @ y_o) <= 1e-11 * (1 + abs(b @ y_o))
    assert abs(s[2] - z.sum()) <= 1e-10 * (1 + np.abs(z).sum())
    assert abs(s[3] - np.sum(Tn * Tn)) <= 1e-11 * np.sum(Tn * Tn)


def _gpu_chain_solve(ctx, q, t, seed, p0=2, **kw):
    Qs, cs = chain_bqp_instance(q, t, seed)
    ctx.set_bqp_chain(Qs, cs)
    n = ctx.sizes()[0]
    ctx.set_params(ctx.default_params(p0=p0, **kw))
    ctx.set_initial_factor(initial_factor(n, p0, seed))
    info = ctx.solve()
    return Qs, cs, info, ctx.solution(want_X=True)


def _check_certified(Qs, cs, info, sol, amaps, cnt, b):
    assert info["status"] == 0
    T = np.stack([sol["X"][k] for k in range(amaps.shape[0])])
    nb = amaps.shape[1]
    # T = X + Diag z per block; residues recomputed by the oracle from the returned tuple
    for k in range(amaps.shape[0]):
        T[k] = T[k] + np.diag(sol["z"][k * nb:(k + 1) * nb])
    res = sb.block_residues(amaps, cnt, b, sol["y"], sol["Y"], T)
    assert res["eta_max"] <= 1e-8, res["eta_max"]
    assert abs(res["dual_obj"] - info["dual_obj"]) <= 1e-9 * (1 + abs(info["dual_obj"]))
    return res


@pytest.mark.parametrize("q,t,seed", [(4, 3, 0), (5, 3, 1), (6, 2, 2), (10, 3, 0)])
def test_chain_solve_vs_oracle(ctx, q, t, seed):
    Qs, cs, info, sol = _gpu_chain_solve(ctx, q, t, seed)
    amaps, cnt, b, _ = sb.relax_chain(Qs, cs)
    _check_certified(Qs, cs, info, sol, amaps, cnt, b)
    N = amaps.shape[0] * amaps.shape[1]
    ref = sb.solve_blocks(amaps, cnt, b, admm.Params(p0=2), initial_factor(N, 2, seed))
    assert ref["status"] == "converged"
    assert abs(info["dual_obj"] - ref["dual_obj"]) <= 1e-6 * (1 + abs(ref["dual_obj"]))
    d = (q - 2) * t + 2
    if d <= 14:
        bf, _ = sb.chain_brute_force(Qs, cs)
        assert info["dual_obj"] <= bf + 1e-6


def test_chain_solve_q20_vs_stored_oracle(ctx):
    """q = 20 (the paper's clique size) against the stored oracle solves
    (tools/oracle_reference_solves.py --chain, oracle only)."""
    gold = json.load(open(GOLD))
    for g in gold["solves"]:
        Qs, cs, info, sol = _gpu_chain_solve(ctx, g["q"], g["t"], g["seed"])
        amaps, cnt, b, _ = sb.relax_chain(Qs, cs)
        _check_certified(Qs, cs, info, sol, amaps, cnt, b)
        assert abs(info["dual_obj"] - g["dual_obj"]) <= 1e-6 * (1 + abs(g["dual_obj"]))


def test_chain_solve_paper_size_certified(ctx):
    """q = 20, t = 20 (the smallest instance of the paper's Table 2): converged, with the
    residues recomputed by the oracle from the returned tuple and the rounding x_i = sign(y_{x_i})
    certifying the relaxation value when it is attained (b^T y <= f(x) always, weak duality)."""
    Qs, cs, info, sol = _gpu_chain_solve(ctx, 20, 20, 0)
    amaps, cnt, b, _ = sb.relax_chain(Qs, cs)
    res = _check_certified(Qs, cs, info, sol, amaps, cnt, b)
    d = 18 * 20 + 2
    x = np.sign(sol["y"][1:1 + d])
    x[x == 0] = 1.0
    fx = sb.chain_value(Qs, cs, x)
    assert info["dual_obj"] <= fx + 1e-6 * (1 + abs(fx))
    assert res["eta_max"] <= 1e-8
