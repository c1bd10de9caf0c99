# PT = 128 raw chunks, register-V upper-triangle kernel at p = 16, precond defaults at d = 40 / 80
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "large_p or full_size or upper_triangle or alm_eval or row_blocks or lanczos or degenerate or operator" > gpurun_out/r2b_tests.log 2>&1; tail -2 gpurun_out/r2b_tests.log
python - > gpurun_out/r2b_symm_check.log 2>&1 <<'PY'
import os, torch, numpy as np, sys
sys.path.insert(0, ".")
from paper_2512_04406_b200 import abi
from inputs import sweep_factor
ctx = abi.Context(0, 0)
n, p = 8192, 16
M = torch.randn(n, n, dtype=torch.float64, device="cuda"); M = (M + M.T) / (2 * n) ** 0.5
Y, U = sweep_factor(n, p)
Yd = torch.tensor(Y, device="cuda")
ctx.set_subproblem_matrix(n, M, n)
cost = torch.zeros(1, dtype=torch.float64, device="cuda"); R = torch.empty_like(Yd)
l0 = ctx.launch_count()
ctx.subproblem_eval(1, p, Yd, None, cost, None, R, None); ctx.sync()
print("SYMM16", os.environ.get("DRSDP_SYMM16"), "launches per costgrad", ctx.launch_count() - l0)
PY
DRSDP_SYMM16=1 python - >> gpurun_out/r2b_symm_check.log 2>&1 <<'PY'
import os, torch, numpy as np, sys
sys.path.insert(0, ".")
from paper_2512_04406_b200 import abi
from inputs import sweep_factor
ctx = abi.Context(0, 0)
n, p = 8192, 16
M = torch.randn(n, n, dtype=torch.float64, device="cuda"); M = (M + M.T) / (2 * n) ** 0.5
Y, U = sweep_factor(n, p)
Yd = torch.tensor(Y, device="cuda")
ctx.set_subproblem_matrix(n, M, n)
cost = torch.zeros(1, dtype=torch.float64, device="cuda"); R = torch.empty_like(Yd)
l0 = ctx.launch_count()
ctx.subproblem_eval(1, p, Yd, None, cost, None, R, None); ctx.sync()
print("SYMM16", os.environ.get("DRSDP_SYMM16"), "launches per costgrad", ctx.launch_count() - l0)
PY
cat gpurun_out/r2b_symm_check.log
DRSDP_SYMM16=1 python tools/quick_sweep.py 16384,32768 16 > gpurun_out/r2b_sweep_symm16.log 2>&1; cat gpurun_out/r2b_sweep_symm16.log
python tools/alm_profile.py 100 128,512 10 > gpurun_out/r2b_alm100.log 2>&1; cat gpurun_out/r2b_alm100.log
run() { tag=$1; shift; DRSDP_VERBOSE=1 timeout 400 python tools/solve_run.py "$@" > gpurun_out/r2b_$tag.log 2> gpurun_out/r2b_$tag.err; tail -1 gpurun_out/r2b_$tag.log | cut -c1-300; }
run H40 40 300 4 precond_mu=0.1
run H80 80 300 4 precond_mu=0.1
run H80d 80 300 4 precond_mu=0.1 eig_method=1
