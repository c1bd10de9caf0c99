"""Quick timing of the fixed-M subproblem evaluation sweep (development aid; bench.py is the contract)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from inputs import sweep_factor, sweep_matrix_torch  # noqa: E402
from paper_2512_04406_b200 import abi  # noqa: E402

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = abi.Context(0, stream.cuda_stream)
out = []
ns = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["4096", "16384", "32768"])]
ps = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["8", "16", "32", "64"])]
for n in ns:
    Md = sweep_matrix_torch(n)
    ctx.set_subproblem_matrix(n, Md, n)
    for p in ps:
        Y, U = sweep_factor(n, p)
        Yd = torch.tensor(Y, device="cuda")
        Ud = torch.tensor(U, device="cuda")
        cost = torch.zeros(1, dtype=torch.float64, device="cuda")
        R = torch.empty_like(Yd)
        H = torch.empty_like(Yd)
        for flags, name in ((1, "costgrad"), (2, "hvp")):
            f = lambda: ctx.subproblem_eval(flags, p, Yd, Ud, cost, None, R, H if flags == 2 else None)
            ctx.subproblem_eval(1, p, Yd, Ud, cost, None, R, None)
            for _ in range(3):
                f()
            torch.cuda.synchronize()
            reps = max(3, int(2e9 / (8 * n * n)))
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                f()
            b.record()
            b.synchronize()
            ms = a.elapsed_time(b) / reps
            out.append({"n": n, "p": p, "eval": name, "us": ms * 1e3, "gbs_8n2": 8 * n * n / ms / 1e6,
                        "tflops": 2 * n * n * p / ms / 1e9})
            print(json.dumps(out[-1]), flush=True)
    del Md
    torch.cuda.empty_cache()
