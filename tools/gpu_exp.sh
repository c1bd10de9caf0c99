mkdir -p gpurun_out
run() { tag=$1; d=$2; tl=$3; shift; shift; shift; timeout $((tl+60)) python tools/solve_run.py $d $tl 4 "$@" > gpurun_out/exp_$tag.log 2>&1; echo "$tag d=$d $*: $(tail -1 gpurun_out/exp_$tag.log | cut -c1-300)"; }
run J10 10 60 escape_max=8 rank_tol=1e-4 stall_rtr=5
run J20 20 60 escape_max=8 rank_tol=1e-4 stall_rtr=5
run J3 40 100 escape_max=8 rank_tol=1e-6 stall_rtr=5
run J4 40 100 escape_max=8 rank_tol=1e-4 stall_rtr=10
run J5 40 100 escape_max=3 rank_tol=1e-4 stall_rtr=5
run J6 40 100 escape_max=8 rank_tol=1e-4 max_rtr=20
run J100 100 500 escape_max=8 rank_tol=1e-4 stall_rtr=5
