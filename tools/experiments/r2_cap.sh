# DRSDP_MAX_P = 4096: parity at the new widths, then d = 100 with more escape columns per iteration
# (cold start escape_max = 32 / 64, and the tightness diagnostic from the tabu vertex with 64)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "degenerate_and_max_p or argument_and_state or (alm_eval_full_size and 70)" > gpurun_out/r2C_parity.log 2>&1; tail -3 gpurun_out/r2C_parity.log
run() { tag=$1; shift; DRSDP_VERBOSE=1 timeout $T python tools/solve_run.py "$@" > gpurun_out/r2C_$tag.log 2> gpurun_out/r2C_$tag.err; }
T=3100 run e32 100 3000 4 escape_max=32 max_outer=1000 &
T=3100 run e64 100 3000 4 escape_max=64 max_outer=1000 &
DRSDP_VERBOSE=1 timeout 1600 python tools/experiments/vertex_start.py 100 1500 escape_max=64 > gpurun_out/r2C_v64.log 2> gpurun_out/r2C_v64.err &
wait
for t in e32 e64 v64; do echo "== $t"; tail -1 gpurun_out/r2C_$t.log | cut -c1-420; grep "k=" gpurun_out/r2C_$t.err | tail -2 | cut -c1-300; done
