# d = 100 (BASELINE configs[2]): three variants run concurrently on the one GPU for up to 55 min each
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_blocks.py -x -q > gpurun_out/r2L_blocks.log 2>&1; tail -1 gpurun_out/r2L_blocks.log
timeout 300 python tools/alm_profile.py chain:20:120 16,64,128 30 2>&1 | tail -3
run() { tag=$1; shift; DRSDP_VERBOSE=1 timeout 3500 python tools/solve_run.py "$@" > gpurun_out/r2L_$tag.log 2> gpurun_out/r2L_$tag.err; }
run s10e2 100 3300 4 stall_factor=10.0 escape_max=2 &
run s3 100 3300 4 stall_factor=3.0 &
run s10t 100 3300 4 stall_factor=10.0 tau2=0.1 &
wait
for t in s10e2 s3 s10t; do echo "== $t"; tail -1 gpurun_out/r2L_$t.log | cut -c1-420; grep "\[drsdp\]" gpurun_out/r2L_$t.err | tail -2 | cut -c1-260; done
