mkdir -p gpurun_out
run() { tag=$1; d=$2; tl=$3; p0=$4; shift 4; DRSDP_VERBOSE=1 timeout $((tl+90)) python tools/solve_run.py $d $tl $p0 "$@" > gpurun_out/exp_$tag.log 2> gpurun_out/exp_$tag.err; echo "$tag d=$d p0=$p0 $*: $(grep '"d"' gpurun_out/exp_$tag.log | cut -c1-260)"; }
run P10 10 60 2
run P20 20 60 2
run P40 40 120 4
run P40s1 40 120 4 seed=1
run P100 100 420 16 escape_max=32
