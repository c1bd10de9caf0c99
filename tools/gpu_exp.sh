mkdir -p gpurun_out
run() { tag=$1; shift; timeout 200 python tools/solve_run.py 40 150 4 "$@" > gpurun_out/exp_$tag.log 2>&1; echo "$tag $*: $(tail -1 gpurun_out/exp_$tag.log | cut -c1-330)"; }
run B stall_rtr=10
run C stall_rtr=10 rho_reg=10.0
run D stall_rtr=10 escape_max=8
run E stall_rtr=10 escape_max=8 rho_reg=10.0
run F stall_rtr=10 eps_scale=0.1
run G stall_rtr=10 escape_max=8 eig_neg_tol=1e-8
