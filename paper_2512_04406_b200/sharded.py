"""Row-sharded subproblem evaluation across GPUs.

M (n x n, symmetric) is split into contiguous row blocks, one per rank; Y and U (n x p) are
replicated. Per evaluation every rank runs the fused product on its block through the C-ABI row
mode (drsdp_set_subproblem_rows / drsdp_subproblem_eval: P_block = M_block Y with the row-local
epilogue of Eq. 4.6 / 4.7), then the exchange step of 8(e):
  * an all-reduce (SUM) of the block cost shares (the cost is additive over row blocks:
    f = ||G||^2 + sum_blocks (-2 sum_{i in block} <(MY)_i, y_i> + ||M_block||^2), G counted once);
  * an all-gather of the n x p output rows (R or H) so that the next direction / iterate is
    replicated again.
torch.distributed is the plumbing (NCCL on GPUs, gloo in the CPU tests); the arithmetic runs in
the library's kernels. This module only partitions rows and issues the collectives.
"""
from __future__ import annotations


def row_blocks(n: int, world: int):
    """Contiguous row blocks [r0, r1) of near-equal size (multiples of 128 rows where possible,
    the product kernel's CTA height), one per rank."""
    per = -(-n // world)
    per = -(-per // 128) * 128 if per >= 128 else per
    out = []
    for r in range(world):
        r0 = min(n, r * per)
        r1 = min(n, r0 + per)
        out.append((r0, r1))
    return out


def gather_rows(torch, dist, local, n, blocks, rank, group=None):
    """All-gather the per-rank row blocks of an (rows, p) tensor into the full (n, p) tensor
    (blocks padded to the largest block for the collective)."""
    per = max(r1 - r0 for r0, r1 in blocks)
    p = local.shape[1]
    buf = torch.zeros((per, p), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    parts = [torch.empty_like(buf) for _ in blocks]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([parts[k][: r1 - r0] for k, (r0, r1) in enumerate(blocks)], dim=0)


def sharded_eval(torch, dist, local_eval, n, blocks, rank, group=None, gather=True):
    """One row-sharded evaluation. local_eval() runs this rank's block and returns
    (cost_share (1-element tensor), rows (rows x p tensor)); returns (f, full rows or the local
    block when gather=False)."""
    cost, rows = local_eval()
    dist.all_reduce(cost, op=dist.ReduceOp.SUM, group=group)
    if not gather:
        return cost, rows
    return cost, gather_rows(torch, dist, rows, n, blocks, rank, group)
