# d = 100 solves: small initial sigma, escape gate (reading R36), no stall exit; Gram-preconditioned tCG
mkdir -p gpurun_out
run() { tag=$1; shift; DRSDP_VERBOSE=1 timeout 720 python tools/solve_run.py "$@" > gpurun_out/r2_$tag.log 2> gpurun_out/r2_$tag.err; tail -1 gpurun_out/r2_$tag.log | cut -c1-420; }
run F1 100 600 4 precond_mu=0.1 sigma0=0.1
run F2 100 600 4 precond_mu=0.1 sigma0=0.1 escape_gate=10.0
run F3 100 600 4 precond_mu=0.1 escape_gate=10.0
run F4 100 600 4 precond_mu=0.1 stall_rtr=0
