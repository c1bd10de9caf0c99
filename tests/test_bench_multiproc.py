"""Host logic of bench.py's N > 1 path on CPU (gloo, world_size 2): every rank times its own
replica, the job time is the max over ranks (all-reduce MAX), value = all ranks' evaluations / that
time (replicas only, no data-path collective). The reference arm runs on
rank 0 only; the other ranks exit 0 without work."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port), "RANK": str(rank),
                       "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank)})
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    w, r, local = bench.dist_setup()
    t_local = 10.0 + 5.0 * rank  # rank 1 is the slow one
    t_max = bench.barrier_and_max(t_local, w, torch.device("cpu"))
    steps = 7
    value = 2.0 * steps * w / (t_max / 1e3)
    q.put((r, w, local, t_max, value))
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_and_weak_scaling_value():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [o[0] for o in out] == [0, 1] and all(o[1] == 2 for o in out)
    assert all(o[3] == 15.0 for o in out)  # every rank sees the slowest rank's time
    assert all(abs(o[4] - 2.0 * 7 * 2 / 0.015) < 1e-9 for o in out)


def test_reference_arm_nonzero_rank_exits_without_work(monkeypatch, capsys):
    import argparse

    import bench

    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")
    args = argparse.Namespace(n=64, p=4, ref_rows=8, warmup=3, steps=1, ref_budget=0.1, gpus=2)
    assert bench.run_reference(args) == 0
    assert capsys.readouterr().out == ""
