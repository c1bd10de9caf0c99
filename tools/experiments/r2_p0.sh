# d = 100 with an over-parameterised start (p0 = 640) against a fast-growing rank (escape_max = 64), both with stall_factor = 10
mkdir -p gpurun_out
run() { tag=$1; shift; DRSDP_VERBOSE=1 timeout $T python tools/solve_run.py "$@" > gpurun_out/r2P_$tag.log 2> gpurun_out/r2P_$tag.err; }
T=3100 run P640 100 3000 640 stall_factor=10.0 escape_max=16 &
T=3100 run E64 100 3000 4 stall_factor=10.0 escape_max=64 &
wait
for t in P640 E64; do echo "== $t"; tail -1 gpurun_out/r2P_$t.log | cut -c1-400; grep "k=" gpurun_out/r2P_$t.err | tail -2 | cut -c1-300; done
