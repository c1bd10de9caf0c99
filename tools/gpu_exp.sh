mkdir -p gpurun_out
run() { tag=$1; d=$2; tl=$3; p0=$4; shift 4; DRSDP_VERBOSE=1 timeout $((tl+120)) python tools/solve_run.py $d $tl $p0 "$@" > gpurun_out/exp_$tag.log 2> gpurun_out/exp_$tag.err; echo "$tag d=$d p0=$p0 $*: $(grep '"d"' gpurun_out/exp_$tag.log | cut -c1-260)"; }
run V1 100 540 8 escape_max=8 rank_tol=1e-3 stall_rtr=30 max_tcg=200 sigma_min=1.0
run V2 100 540 8 escape_max=16 rank_tol=1e-3 stall_rtr=30 max_tcg=200 sigma_min=1.0 sigma0=2.0
