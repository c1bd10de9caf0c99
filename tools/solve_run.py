"""Development aid: run drsdp_solve on BQP configs and print the per-iteration trace.

Usage: python tools/solve_run.py D[,D...] [time_limit_s] [p0] [key=value ...]  (extra drsdp_params)
       D may be chain:q:t (the clique-chain sparse BQP, multi-block relaxation)
"""
import json
import sys
import time

sys.path.insert(0, ".")
from inputs import bqp_instance, initial_factor  # noqa: E402
from oracle import bqp  # noqa: E402  (sizes only: n for the initial factor)
from paper_2512_04406_b200 import abi  # noqa: E402

ds = [x if x.startswith("chain") else int(x) for x in sys.argv[1].split(",")]
tl = float(sys.argv[2]) if len(sys.argv) > 2 else 300.0
ctx = abi.Context(0, None)
for d in ds:
    t0 = time.time()
    if isinstance(d, str):
        from inputs import chain_bqp_instance  # noqa: E402

        _, q, t = d.split(":")
        ctx.set_bqp_chain(*chain_bqp_instance(int(q), int(t), 0))
    else:
        kind = "er05" if d == 150 else "dense"
        Q, c = bqp_instance(d, 0, kind)
        ctx.set_bqp(Q, c)
    n = ctx.sizes()[0]
    p0 = int(sys.argv[3]) if len(sys.argv) > 3 else (2 if isinstance(d, str) or d <= 10 else 4)
    kw = {}
    for a in sys.argv[4:]:
        k, v = a.split("=")
        kw[k] = float(v) if "." in v or "e" in v else int(v)
    ctx.set_params(ctx.default_params(p0=p0, time_limit_s=tl, **kw))
    ctx.set_initial_factor(initial_factor(n, p0, 0))
    t1 = time.time()
    info = ctx.solve()
    t2 = time.time()
    for r in ctx.trace():
        print(" ".join(f"{k}={v:.3e}" if isinstance(v, float) and k.startswith("eta") else f"{k}={v:.6g}"
                       for k, v in r.items()), flush=True)
    print(json.dumps({"d": d, "n": n, "setup_s": t1 - t0, "solve_s": t2 - t1, **info}), flush=True)
