#!/usr/bin/env python
"""bench.py — the driver's benchmark contract for the ManiDSDP hot path on B200.

Workload (BASELINE.json configs[4], the configuration its metric "subproblem grad+HVP evals/s &
GB/s vs HBM roofline" is quoted on): the oblique-manifold subproblem f(Y) = ||YY^T - M||^2 with a
dense symmetric M, entries N(0,1)/sqrt(n), Y with unit rows, U a random tangent direction,
n = 32768 (M = 8.6 GB, far larger than the 126 MB L2: no flush needed), p = 16 by default.
One step = one cost+gradient+Riemannian-gradient evaluation followed by one Hessian-vector
product at the same Y (the "grad+HVP" pair of the metric), i.e. 2 subproblem evaluations.
value = evaluations/s (whole job; 2 per step). The other sweep points (n in {4096, 16384, 32768} x
p in {8, 16, 32, 64}) and full ManiDSDP solves of the dense BQPs d = 10, 40 (configs[0..1], "solve time to
KKT 1e-8") and d = 80 (the paper's largest dense size) are reported in the same JSON line under "sweep" and "solves".

Multi-GPU (--gpus N under torchrun): the benchmark runs replicas (no data-path collective, DESIGN.md
"replicas only"): every rank runs the same workload on its own GPU, no collective on the data
path; value = all ranks' evaluations / max-over-ranks time (weak scaling).

--impl reference: the oracle (oracle/, plain NumPy, single-threaded) timed on the host cores on a
bounded sample of the same workload (rows of the n x n problem; scaled to the metric's unit).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "subproblem grad+HVP evals/s & GB/s vs HBM roofline; solve time to KKT 1e-8"
UNIT = "subproblem evals/s"


def measured_peaks():
    """HBM GB/s from MEASURED_PEAKS.json (driver-written); fp64 from our own measurement
    (profiles/r01_fp64_peaks.json) because MEASURED_PEAKS.json has no fp64 figure."""
    hbm, hbm_src = 6650.0, "fallback B200_PROFILING.md"
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm, hbm_src = float(mp["hbm_gbs"]), "measured MEASURED_PEAKS.json hbm_gbs (copy)"
    except Exception:
        pass
    f64, f64_src = 37.1, "measured profiles/r01_fp64_peaks.json dmma_m8n8k4_tflops"
    try:
        pk = json.load(open(os.path.join(ROOT, "profiles", "r01_fp64_peaks.json")))
        f64 = float(pk["dmma_m8n8k4_tflops"])
    except Exception:
        pass
    return hbm, hbm_src, f64, f64_src


def work_units(n, p, kind):
    """Algorithmic bytes and flops of one evaluation (SURVEY.md §8(d) D-ALG):
    distinct M entries 8 n(n+1)/2 plus the n x p operands; 2 n^2 p flops for M.V."""
    m_bytes = 8.0 * n * (n + 1) / 2
    if kind == "matrix":
        return m_bytes, 0.0
    if kind == "costgrad":
        return m_bytes + 16.0 * n * p + 8.0 * n, 2.0 * n * n * p + 2.0 * n * p * p
    return m_bytes + 24.0 * n * p, 2.0 * n * n * p + 4.0 * n * p * p


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[k] for r in self.rows for k in range(4) if len(r) > 4 + k and r[4 + k] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def barrier_and_max(t_ms, world, device):
    if world == 1:
        return t_ms
    import torch
    import torch.distributed as dist

    x = torch.tensor([t_ms], dtype=torch.float64, device=device)
    dist.all_reduce(x, op=dist.ReduceOp.MAX)
    return float(x.item())


# ------------------------------------------------------------------------------------------------
# oracle timings (cpu_baseline and --impl reference)
# ------------------------------------------------------------------------------------------------
def oracle_sample(n, p, Mrows_fn, Y, U, rows_per_eval, budget_s=15.0):
    """Time the oracle's plain evaluation formulas (oracle.subproblem.fixed_rows: cost rows,
    E, R, and the HVP rows) on `rows_per_eval` rows of the n x n problem; returns the scaled
    full-problem evaluations/s and the sample description."""
    from oracle import subproblem as sp  # noqa: oracle is test infrastructure; cpu_baseline leg only

    rows = np.arange(rows_per_eval)
    Mr = Mrows_fn(rows)
    t0 = time.perf_counter()
    reps = 0
    while True:
        sp.fixed_rows(Mr, rows, Y)          # cost + gradient rows
        sp.fixed_rows(Mr, rows, Y, U)       # HVP rows
        reps += 1
        if time.perf_counter() - t0 > budget_s or reps >= 50:
            break
    dt = (time.perf_counter() - t0) / reps  # seconds per (costgrad + HVP) on the sample rows
    per_pair_full = dt * n / rows_per_eval
    return 2.0 / per_pair_full, (f"oracle.subproblem.fixed_rows (NumPy, 1 BLAS thread) on rows 0..{rows_per_eval - 1} of "
                                 f"the n={n}, p={p} problem, cost+grad then HVP, {reps} reps; scaled by n/{rows_per_eval}")


def cpu_model():
    """Host CPU model name (lscpu / /proc/cpuinfo) for the oracle timings."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_full_eval(n, p, M, Y, U):
    """One unsampled oracle evaluation pair (cost+grad, then HVP: oracle.subproblem.fixed_eval on the
    whole n x n problem) on 1 core; returns seconds per evaluation."""
    from oracle import subproblem as sp  # noqa: oracle is test infrastructure; cpu_baseline leg only

    t0 = time.perf_counter()
    sp.fixed_eval(M, Y)
    sp.fixed_eval(M, Y, U)
    return (time.perf_counter() - t0) / 2.0


def oracle_solves(seeds=(0, 1, 2), d=10):
    """The oracle's full Alg. 2 solves of BASELINE configs[0] (d = 10, 3 seeds) timed in-run on
    1 core (plus the stored d = 40 oracle solve, tests/golden/oracle_solves.json, reported as cached)."""
    from inputs import bqp_instance, initial_factor
    from oracle import admm, bqp  # noqa: oracle is test infrastructure; cpu_baseline leg only

    rows = []
    for seed in seeds:
        Q, c = bqp_instance(d, seed)
        amap, cnt, b = bqp.relax(Q, c)
        t0 = time.perf_counter()
        o = admm.solve(amap, cnt, b, None, admm.Params(p0=2), initial_factor(amap.shape[0], 2, seed))
        rows.append({"d": d, "seed": seed, "seconds": time.perf_counter() - t0, "status": o["status"],
                     "outer_iters": o["outer_iters"], "dual_obj": o["dual_obj"], "eta_max": o["eta_max"],
                     "cores": 1, "kind": "oracle, in-run"})
    try:
        gold = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_solves.json")))
        for v in gold["solves"]:
            if v.get("d") == 40:
                rows.append({"d": 40, "seed": v.get("seed", 0), "seconds": v.get("seconds_1core"),
                             "status": v.get("status"), "outer_iters": v.get("outer_iters"),
                             "dual_obj": v.get("dual_obj"), "cores": 1,
                             "kind": f"oracle, cached {gold.get('date')} at commit {gold.get('commit')} "
                                     "(tests/golden/oracle_solves.json, tools/oracle_reference_solves.py)"})
    except Exception:
        pass
    return rows


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def run_reference(args):
    world, rank, local = dist_setup()
    if rank != 0:
        return 0
    from inputs import sweep_factor, sweep_matrix_cpu  # noqa

    n, p = args.n, args.p
    Y, U = sweep_factor(n, p)
    rng_rows = min(args.ref_rows, n)

    # rows of M from the same generator the GPU arm uses (torch on the device if present)
    try:
        import torch

        if torch.cuda.is_available():
            from inputs import sweep_matrix_torch

            Md = sweep_matrix_torch(n)
            Mrows_fn = lambda rows: Md[torch.as_tensor(rows, device="cuda")].cpu().numpy()
        else:
            raise RuntimeError
    except Exception:
        M = sweep_matrix_cpu(n) if n <= 8192 else None
        if M is None:
            rng = np.random.default_rng([20251204, n, 99])
            Mrows_fn = lambda rows: rng.standard_normal((rows.size, n)) / np.sqrt(n)
        else:
            Mrows_fn = lambda rows: M[rows]
    vals = []
    for _ in range(args.warmup):
        oracle_sample(n, p, Mrows_fn, Y, U, rng_rows, budget_s=2.0)
    t0 = time.perf_counter()
    desc = ""
    for _ in range(args.steps):
        v, desc = oracle_sample(n, p, Mrows_fn, Y, U, rng_rows, budget_s=args.ref_budget)
        vals.append(v)
    wall = time.perf_counter() - t0
    value = float(np.median(vals))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 2000.0 / value,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_block(args),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc,
                             "host_cores": host_cores()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": wall}
    print(json.dumps(line), flush=True)
    return 0


def config_block(args):
    return {"workload": f"BASELINE.json configs[4] subproblem-kernel sweep point n={args.n}, p={args.p} "
                        "(fixed-M f = ||YY^T - M||^2, M ~ N(0,1)/sqrt(n) symmetric, unit-row Y, tangent U)",
            "n": args.n, "p": args.p, "step": "1 cost+grad+Riemannian-grad eval + 1 HVP eval (tangent U) at the same Y, one "
                    "drsdp_subproblem_eval(COSTGRAD|HVP) call (one fused pass over M for 5 <= p <= 32)",
            "l2_policy": "inputs larger than L2 (M = 8 n^2 bytes >> 126 MB) at n >= 16384; n = 4096 sweep points "
                         "flush L2 (512 MB read) before each timed launch", "parallelism": "replicas" if args.gpus > 1 else "single-gpu"}


# ------------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------------
def timed_evals(ctx, stream, torch, n, p, Md, Yd, Ud, reps, warmup, flush=None):
    """Average device ms per COSTGRAD and per HVP; with `flush` (a buffer larger than L2) the L2
    is overwritten before every timed launch so that M comes from HBM."""
    cost = torch.zeros(1, dtype=torch.float64, device="cuda")
    R = torch.empty_like(Yd)
    H = torch.empty_like(Yd)
    flush_sink = torch.zeros((), dtype=torch.float64, device="cuda")
    ctx.set_subproblem_matrix(n, Md, n)
    res = {}
    for flags, name in ((1, "costgrad"), (2, "hvp")):
        for w in range(warmup):
            ctx.subproblem_eval(1, p, Yd, None, cost, None, R, None)
            if flags == 2:
                ctx.subproblem_eval(2, p, Yd, Ud, None, None, None, H)
        tot = 0.0
        for r in range(reps):
            if flags == 2:
                ctx.subproblem_eval(1, p, Yd, None, cost, None, R, None)
            if flush is not None:
                flush_sink.copy_(flush.sum())  # read 512 MB (> L2): evicts M without dirty lines
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ctx.subproblem_eval(flags, p, Yd, Ud, cost, None, R, H if flags == 2 else None)
            b.record(stream)
            b.synchronize()
            tot += a.elapsed_time(b)
        res[name] = tot / reps
    if 5 <= p <= 32:
        # the fused one-pass call (cost+grad and HVP at the same Y): device ms per call
        for w in range(warmup):
            ctx.subproblem_eval(3, p, Yd, Ud, cost, None, R, H)
        tot = 0.0
        for r in range(reps):
            if flush is not None:
                flush_sink.copy_(flush.sum())
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ctx.subproblem_eval(3, p, Yd, Ud, cost, None, R, H)
            b.record(stream)
            b.synchronize()
            tot += a.elapsed_time(b)
        res["both"] = tot / reps
    return res


def run_gpu(args):
    import torch

    world, rank, local = dist_setup()
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    from inputs import sweep_factor, sweep_matrix_torch
    from paper_2512_04406_b200 import abi, build

    build.build()
    stream = torch.cuda.Stream(device=device)
    torch.cuda.set_stream(stream)
    ctx = abi.Context(local, stream.cuda_stream)
    hbm, hbm_src, f64, f64_src = measured_peaks()
    n, p = args.n, args.p

    # ---------------- primary: the grad+HVP step at (n, p) -------------------------------------
    Md = sweep_matrix_torch(n, device=device)
    Y, U = sweep_factor(n, p)
    Yd = torch.tensor(Y, device=device)
    Ud = torch.tensor(U, device=device)
    ctx.set_subproblem_matrix(n, Md, n)
    cost = torch.zeros(1, dtype=torch.float64, device=device)
    R = torch.empty_like(Yd)
    H = torch.empty_like(Yd)

    def step():
        # cost + gradient + Riemannian gradient and the HVP along U at the same Y: one call; for
        # 5 <= p <= 32 the library serves both from ONE pass over M (product M [Y U], EPI_BOTH)
        ctx.subproblem_eval(abi.EVAL_COSTGRAD | abi.EVAL_HVP, p, Yd, Ud, cost, None, R, H)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    launches0 = ctx.launch_count()
    ctx.profile_enable(True)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    t_ms = ev0.elapsed_time(ev1)
    launches = ctx.launch_count() - launches0
    k_ms_cg, k_n_cg = ctx.profile_read(1)
    k_ms_hv, k_n_hv = ctx.profile_read(2)
    k_ms_both, k_n_both = ctx.profile_read(4)
    ctx.profile_enable(False)
    if world > 1:
        torch.distributed.barrier()
    t_max = barrier_and_max(t_ms, world, device)
    evals = 2.0 * args.steps * world
    value = evals / (t_max / 1e3)

    # roofline of the dominant kernel (the fused product): either one EPI_BOTH launch per step
    # (cost+grad and HVP from one pass over M) or separate COSTGRAD / HVP launches
    b_cg, f_cg = work_units(n, p, "costgrad")
    b_hv, f_hv = work_units(n, p, "hvp")
    if k_n_both > 0:
        t_k = k_ms_both / k_n_both / 1e3  # s per launch
        # one pass over M for both products: the matrix bytes once, the operands of both, all flops
        bytes_l = b_cg + b_hv - work_units(n, p, "matrix")[0]
        flops_l = f_cg + f_hv
        k_ms_cg, k_ms_hv = k_ms_both, 0.0
    else:
        t_k = (k_ms_cg + k_ms_hv) / max(1, k_n_cg + k_n_hv) / 1e3
        bytes_l = (b_cg + b_hv) / 2.0
        flops_l = (f_cg + f_hv) / 2.0
    t_hbm, t_f64 = bytes_l / (hbm * 1e9), flops_l / (f64 * 1e12)
    if t_f64 >= t_hbm:
        roof = {"bound": "tensor", "achieved": flops_l / t_k / 1e12, "peak": f64, "unit": "TFLOP/s",
                "peak_source": f64_src + " (fp64 DMMA; tcgen05 has no f64 kind)"}
    else:
        roof = {"bound": "hbm", "achieved": bytes_l / t_k / 1e9, "peak": hbm, "unit": "GB/s", "peak_source": hbm_src}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = None
    # DRAM bytes per launch from the committed ncu --set full capture of this configuration
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        if tr.get("n") == n and tr.get("p") == p:
            roof["traffic"] = tr["dram_bytes_per_launch"]
            roof["traffic_source"] = tr["source"]
    except Exception:
        pass
    roof["kernel"] = ("symv_tma_kernel<PT, EPI_BOTH> (TMA ring + DMMA over M [Y U], cost/gradient and HVP row "
                      "epilogues in one pass; timing includes the V^T staging)" if k_n_both > 0 else
                      "symv_tma_kernel (TMA ring + DMMA, COSTGRAD and HVP epilogues; timing includes the V^T staging)")
    roof["evals_per_launch"] = 2 if k_n_both > 0 else 1
    roof["per_launch_ms"] = t_k * 1e3
    roof["algorithmic_bytes_per_launch"] = bytes_l
    roof["algorithmic_flops_per_launch"] = flops_l
    roof["share_of_step"] = (k_ms_cg + k_ms_hv) / t_ms
    roof["gbs_8n2_convention"] = 8.0 * n * n / t_k / 1e9

    # ---------------- e2e: the same step through the host-buffer C-ABI entry -------------------
    Yh = torch.tensor(Y).pin_memory()
    Uh = torch.tensor(U).pin_memory()
    Rh = torch.empty_like(Yh).pin_memory()
    Hh = torch.empty_like(Yh).pin_memory()
    ch = torch.zeros(1, dtype=torch.float64).pin_memory()
    lib = ctx.lib

    def e2e_step():
        rc = lib.drsdp_subproblem_eval_host(ctx.h, abi.EVAL_COSTGRAD | abi.EVAL_HVP, p, Yh.data_ptr(),
                                            Uh.data_ptr(), ch.data_ptr(), None, Rh.data_ptr(), Hh.data_ptr())
        if rc:
            raise abi.DrsdpError(rc, "e2e")

    for _ in range(max(1, args.warmup)):
        e2e_step()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    k_e2e = max(3, args.steps // 4)
    for _ in range(k_e2e):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    te = barrier_and_max(e0.elapsed_time(e1), world, device)
    e2e = {"value": 2.0 * k_e2e * world / (te / 1e3), "unit": UNIT, "h2d_bytes_per_step": 2 * 8 * n * p,
           "d2h_bytes_per_step": 8 + 2 * 8 * n * p,
           "api": "drsdp_subproblem_eval_host (pinned host Y, U in; cost, R, H out)"}
    del Yh, Uh, Rh, Hh

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_block(args),
           "roofline": roof, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
           "gbs_8n2_convention": 8.0 * n * n * evals / world / (t_max / 1e3) / 1e9}

    # ---------------- sweep (BASELINE configs[4]) --------------------------------------------
    if not args.no_sweep and rank == 0:
        sweep = []
        del Md
        torch.cuda.empty_cache()
        flush = torch.zeros(64 << 20, dtype=torch.float64, device=device)  # 512 MB > L2
        for sn in (4096, 16384, 32768):
            Ms = sweep_matrix_torch(sn, device=device)
            fl_buf = flush if sn * sn * 8 < 4 * 132644864 else None
            for sp_ in (8, 16, 32, 64):
                Ys, Us = sweep_factor(sn, sp_)
                Ysd, Usd = torch.tensor(Ys, device=device), torch.tensor(Us, device=device)
                reps = 20 if sn >= 16384 else 100
                ms = timed_evals(ctx, stream, torch, sn, sp_, Ms, Ysd, Usd, reps, 3, fl_buf)
                for kind in ("costgrad", "hvp"):
                    by, fl = work_units(sn, sp_, kind)
                    t = ms[kind] / 1e3
                    t_roof = max(8.0 * sn * sn / (hbm * 1e9), 2.0 * sn * sn * sp_ / (f64 * 1e12))
                    t_roof_alg = max(by / (hbm * 1e9), fl / (f64 * 1e12))
                    sweep.append({"n": sn, "p": sp_, "eval": kind, "us": ms[kind] * 1e3, "evals_per_s": 1.0 / t,
                                  "gbs_8n2": 8.0 * sn * sn / t / 1e9, "tflops": fl / t / 1e12,
                                  "frac_bj5_roofline": t_roof / t, "frac_alg_roofline": t_roof_alg / t})
                if "both" in ms:
                    # one call = 2 evaluations: M once, both operand sets, both evaluations' flops
                    b_cg, f_cg = work_units(sn, sp_, "costgrad")
                    b_hv, f_hv = work_units(sn, sp_, "hvp")
                    by = b_cg + b_hv - work_units(sn, sp_, "matrix")[0]
                    fl = f_cg + f_hv
                    t = ms["both"] / 1e3
                    t_roof = 2.0 * max(8.0 * sn * sn / (hbm * 1e9), 2.0 * sn * sn * sp_ / (f64 * 1e12))
                    t_roof_alg = max(by / (hbm * 1e9), fl / (f64 * 1e12))
                    sweep.append({"n": sn, "p": sp_, "eval": "costgrad+hvp (one call, one pass over M)",
                                  "us": ms["both"] * 1e3, "evals_per_s": 2.0 / t, "tflops": fl / t / 1e12,
                                  "frac_bj5_roofline": t_roof / t, "frac_alg_roofline": t_roof_alg / t})
            del Ms
            torch.cuda.empty_cache()
        del flush
        sweep_l2 = "n=4096: a 512 MB buffer is read (summed) before every timed launch (L2 flush without dirty lines)"
        out["sweep"] = sweep
        out["sweep_l2"] = sweep_l2
        out["sweep_note"] = ("frac_bj5_roofline = max(8n^2/BW, 2n^2p/F64) / t (BASELINE north star); "
                             "frac_alg_roofline uses the algorithmic bytes (distinct M entries)")

    # ---------------- full solves (configs[0], configs[1]) -----------------------------------
    if not args.no_solve and rank == 0:
        from inputs import bqp_instance, initial_factor

        solves = []
        runs = [(d, 0) for d in args.solve_d]
        if 10 in args.solve_d:  # configs[0] is quoted over 3 seeds (the oracle's in-run solves)
            runs[runs.index((10, 0)) + 1:runs.index((10, 0)) + 1] = [(10, 1), (10, 2)]
        for d, seed in runs:
            kind = "er05" if d == 150 else "dense"  # configs[3] is the Erdos-Renyi sparse BQP
            Q, c = bqp_instance(d, seed, kind)
            ctx.set_bqp(Q, c)
            nn = 1 + d + d * (d - 1) // 2
            p0 = 2 if d <= 10 else 4
            # BASELINE configs[2] / [3] (d = 100 dense, d = 150 ER) run with a short limit in the default
            # bench (status and residues at the limit; the certified d = 150 record comes from
            # tests/test_long_solves.py)
            tl = args.solve_time_limit if d < 100 else args.solve_time_limit_large
            ctx.set_params(ctx.default_params(p0=p0, time_limit_s=tl, **args.solve_params))
            ctx.set_initial_factor(initial_factor(nn, p0, seed))
            t0 = time.perf_counter()
            info = ctx.solve()
            wall = time.perf_counter() - t0
            paper = {10: 0.07, 20: 0.24, 30: 1.44, 40: 2.69, 50: 15.0, 60: 115.0, 70: 227.0, 80: 776.0}.get(d)
            solves.append({"d": d, "seed": seed, "kind": kind, "n": nn, "seconds": wall, "paper_mean_seconds": paper,
                           "paper_context": "ManiDSDP, MATLAB on an i9-10900 CPU, N(0,1) instances (P:789-798); "
                                            "context only, not the same instances",
                           "status": "converged" if info["status"] == 0 else
                           "not_converged", "time_limit_s": tl, "outer_iters": info["outer_iters"], "p_max": info["p_max"],
                           "eta_p": info["eta_p"], "eta_d": info["eta_d"], "eta_g": info["eta_g"],
                           "dual_obj": info["dual_obj"], "n_costgrad": info["n_costgrad"], "n_hvp": info["n_hvp"]})
            print(f"[bench] solve d={d} seed={seed}: {wall:.2f} s {solves[-1]['status']} outer={info['outer_iters']}",
                  file=sys.stderr, flush=True)
        out["solves"] = solves
        # clique-chain sparse BQPs (multi-block relaxation), N(0,1) data as
        # in the paper; the paper's ManiDSDP means (Tables 2-3) as context
        from inputs import chain_bqp_instance

        paper_chain = {(20, 20): 10.3, (20, 40): 48.4, (20, 60): 100.7, (20, 80): 189.0, (20, 100): 166.3,
                       (20, 120): 312.0, (10, 10): 0.18, (20, 10): 4.21, (30, 10): 62.9, (40, 10): 812.0}
        chain = []
        for q, t in args.solve_chain:
            Qs, cs = chain_bqp_instance(q, t, 0)
            ctx.set_bqp_chain(Qs, cs)
            nn = ctx.sizes()[0]
            ctx.set_params(ctx.default_params(p0=2, time_limit_s=args.solve_time_limit, **args.solve_params))
            ctx.set_initial_factor(initial_factor(nn, 2, 0))
            t0 = time.perf_counter()
            info = ctx.solve()
            wall = time.perf_counter() - t0
            chain.append({"q": q, "t": t, "seed": 0, "n_rows": nn, "n_b": ctx.block_sizes()[1], "m": ctx.sizes()[1],
                          "seconds": wall, "paper_mean_seconds": paper_chain.get((q, t)),
                          "paper_context": "ManiDSDP, MATLAB on an i9-10900 CPU, Tables 2-3 (P:582-672); context only",
                          "status": "converged" if info["status"] == 0 else "not_converged",
                          "outer_iters": info["outer_iters"], "p_max": info["p_max"], "eta_p": info["eta_p"],
                          "eta_d": info["eta_d"], "eta_g": info["eta_g"], "dual_obj": info["dual_obj"],
                          "n_costgrad": info["n_costgrad"], "n_hvp": info["n_hvp"]})
            print(f"[bench] chain q={q} t={t}: {wall:.2f} s {chain[-1]['status']} outer={info['outer_iters']} "
                  f"eta=({info['eta_p']:.1e},{info['eta_d']:.1e},{info['eta_g']:.1e})", file=sys.stderr, flush=True)
        out["chain_solves"] = chain

    # ---------------- cpu baseline (oracle, bounded sample) ------------------------------------
    if rank == 0 and not args.no_cpu_baseline:
        Mrows_src = sweep_matrix_torch(n, device=device)
        v, desc = oracle_sample(n, p, lambda rows: Mrows_src[torch.as_tensor(rows, device=device)].cpu().numpy(),
                                Y, U, min(args.ref_rows, n), budget_s=args.ref_budget)
        del Mrows_src
        out["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc,
                               "host_cores": host_cores(), "cpu_model": cpu_model()}
        if not args.no_full_oracle:
            # one unsampled oracle evaluation at n = 16384 beside the sampled baseline
            nf, pf = 16384, p
            Mf = sweep_matrix_torch(nf, device=device).cpu().numpy()
            Yf, Uf = sweep_factor(nf, pf)
            sec = oracle_full_eval(nf, pf, Mf, Yf, Uf)
            del Mf
            out["cpu_baseline"]["full_eval_n16384"] = {
                "seconds_per_eval": sec, "evals_per_s": 1.0 / sec, "n": nf, "p": pf, "cores": 1,
                "sample": "oracle.subproblem.fixed_eval on the whole n = 16384 problem (cost+grad, then HVP)"}
        out["oracle_solves"] = oracle_solves()
    if rank == 0:
        print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="gpu", choices=("gpu", "reference"))
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--p", type=int, default=16)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-full-oracle", action="store_true")
    ap.add_argument("--solve-d", type=lambda s: [int(x) for x in s.split(",") if x], default=[10, 40, 80, 100, 150])
    ap.add_argument("--solve-time-limit-large", type=float, default=60.0,
                    help="time limit of the d >= 100 solves (BASELINE configs[2], [3])")
    ap.add_argument("--solve-chain", type=lambda s: [tuple(int(v) for v in x.split(":")) for x in s.split(",") if x],
                    default=[(20, 20), (20, 120)], help="clique-chain solves q:t,... (multi-block relaxation)")
    ap.add_argument("--solve-time-limit", type=float, default=120.0)
    ap.add_argument("--solve-params", type=lambda s: {k: (float(v) if "." in v or "e" in v else int(v))
                                                      for k, v in (a.split("=") for a in s.split(",") if a)},
                    default={}, help="extra drsdp_params for the solves, e.g. precond_mu=0.01,eig_method=0")
    ap.add_argument("--ref-rows", type=int, default=256)
    ap.add_argument("--ref-budget", type=float, default=10.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
