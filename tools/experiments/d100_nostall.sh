# inner solves without the stagnation exit (stall_rtr = 0) and the Gram preconditioner: d = 40 / 80 cost,
# then d = 100 with larger escape steps
mkdir -p gpurun_out
run() { tag=$1; shift; DRSDP_VERBOSE=1 timeout 1700 python tools/solve_run.py "$@" > gpurun_out/r2_$tag.log 2> gpurun_out/r2_$tag.err; tail -1 gpurun_out/r2_$tag.log | cut -c1-420; }
run G3 40 300 4 precond_mu=0.1 stall_rtr=0
run G2 80 300 4 precond_mu=0.1 stall_rtr=0
run G1 100 1500 4 precond_mu=0.1 stall_rtr=0 escape_max=32
