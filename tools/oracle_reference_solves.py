"""Write tests/golden/oracle_solves.json: full oracle solves (Algorithm 2, oracle/admm.py, default
parameters) of the BASELINE BQP configs the oracle finishes in minutes, used by the GPU parity
tests to compare final objectives without re-running the oracle (the oracle is single-threaded
NumPy; d = 40 takes minutes). Calls only oracle/ and the shared input generators.

Usage: python tools/oracle_reference_solves.py [d=40 seeds...]
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from threadpoolctl import threadpool_limits  # noqa: E402

from inputs import bqp_instance, initial_factor  # noqa: E402
from oracle import admm, bqp  # noqa: E402


def main():
    out_path = os.path.join(ROOT, "tests", "golden", "oracle_solves.json")
    cases = [(10, s) for s in range(3)] + [(40, 0)]
    res = []
    commit = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"], capture_output=True,
                            text=True).stdout.strip()
    for d, seed in cases:
        Q, c = bqp_instance(d, seed)
        amap, cnt, b = bqp.relax(Q, c)
        p0 = 2 if d <= 10 else 4
        t0 = time.time()
        with threadpool_limits(1):
            r = admm.solve(amap, cnt, b, None, admm.Params(p0=p0), initial_factor(amap.shape[0], p0, seed))
        row = {"d": d, "seed": seed, "kind": "dense", "n": int(amap.shape[0]), "p0": p0, "status": r["status"],
               "dual_obj": r["dual_obj"], "primal_obj": r["primal_obj"], "eta_p": r["eta_p"], "eta_d": r["eta_d"],
               "eta_g": r["eta_g"], "outer_iters": r["outer_iters"], "seconds_1core": time.time() - t0}
        print(json.dumps(row), flush=True)
        res.append(row)
    json.dump({"what": "oracle (oracle/admm.py, default Params, 1 BLAS thread) full solves of BASELINE BQP configs",
               "written_by": "tools/oracle_reference_solves.py", "commit": commit,
               "date": time.strftime("%Y-%m-%d"), "solves": res}, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main()
