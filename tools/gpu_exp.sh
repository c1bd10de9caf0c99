mkdir -p gpurun_out
run() { tag=$1; d=$2; tl=$3; p0=$4; shift 4; DRSDP_VERBOSE=1 timeout $((tl+90)) python tools/solve_run.py $d $tl $p0 "$@" > gpurun_out/exp_$tag.log 2> gpurun_out/exp_$tag.err; echo "$tag d=$d p0=$p0 $*: $(grep '"d"' gpurun_out/exp_$tag.log | cut -c1-260)"; }
timeout 200 ncu --graph-profiling node --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_d40g.csv python tools/solve_run.py 40 2 > gpurun_out/ncu_d40g.log 2>&1; tail -1 gpurun_out/ncu_d40g.log
run Q1 100 420 16 escape_max=32 sigma_min=1.0
run Q2 100 420 32 escape_max=64 sigma_min=1.0 sigma0=4.0
