mkdir -p gpurun_out
bash tools/gpu_profile.sh
run() { tag=$1; d=$2; tl=$3; p0=$4; shift 4; timeout $((tl+90)) python tools/solve_run.py $d $tl $p0 "$@" > gpurun_out/exp_$tag.log 2> gpurun_out/exp_$tag.err; echo "$tag d=$d p0=$p0 $*: $(grep '"d"' gpurun_out/exp_$tag.log | cut -c1-200)"; }
run T1 40 120 4 max_tcg=100
run T2 40 120 4 max_tcg=300
run T3 40 120 4 max_tcg=1000
