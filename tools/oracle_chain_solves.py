"""Write tests/golden/oracle_chain_solves.json: oracle solves (Algorithm 2 over blocks,
oracle/sparse_bqp.py, default parameters) of clique-chain sparse BQPs at the paper's clique size
q = 20, used by tests/test_gpu_blocks.py to compare final objectives without re-running
the oracle. Calls only oracle/ and the shared input generators.

Usage: python tools/oracle_chain_solves.py
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from threadpoolctl import threadpool_limits  # noqa: E402

from inputs import chain_bqp_instance, initial_factor  # noqa: E402
from oracle import admm  # noqa: E402
from oracle import sparse_bqp as sb  # noqa: E402


def main():
    out_path = os.path.join(ROOT, "tests", "golden", "oracle_chain_solves.json")
    cases = [(20, 2, 0), (20, 3, 1)]
    res = []
    commit = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"], capture_output=True,
                            text=True).stdout.strip()
    for q, t, seed in cases:
        Qs, cs = chain_bqp_instance(q, t, seed)
        amaps, cnt, b, _ = sb.relax_chain(Qs, cs)
        N = amaps.shape[0] * amaps.shape[1]
        t0 = time.time()
        with threadpool_limits(1):
            r = sb.solve_blocks(amaps, cnt, b, admm.Params(p0=2), initial_factor(N, 2, seed))
        row = {"q": q, "t": t, "seed": seed, "n_b": int(amaps.shape[1]), "m": int(cnt.size), "p0": 2,
               "status": r["status"], "dual_obj": r["dual_obj"], "primal_obj": r["primal_obj"],
               "eta_p": r["eta_p"], "eta_d": r["eta_d"], "eta_g": r["eta_g"], "outer_iters": r["outer_iters"],
               "seconds_1core": time.time() - t0}
        print(json.dumps(row), flush=True)
        res.append(row)
    json.dump({"what": "oracle (oracle/sparse_bqp.py solve_blocks, default Params, 1 BLAS thread) solves of "
                       "clique-chain sparse BQP relaxations (P:555-602)",
               "written_by": "tools/oracle_chain_solves.py", "commit": commit,
               "date": time.strftime("%Y-%m-%d"), "solves": res}, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main()
