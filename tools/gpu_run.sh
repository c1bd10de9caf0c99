mkdir -p gpurun_out
DRSDP_VERBOSE=1 timeout 3400 python tools/solve_run.py 150 3300 4 > gpurun_out/solve_r34_150_long.log 2> gpurun_out/solve_r34_150_long_v.log
tail -1 gpurun_out/solve_r34_150_long.log | cut -c1-420
